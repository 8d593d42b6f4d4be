"""Generate golden vectors by running the REAL reference (ewaldmd) here.

Run in the build container only (it imports /root/reference, which does not
exist on the GPU box):

    python tests/golden/make_golden.py [small c1 c2 c3 c4 c5]

Every case evaluates the reference's own stock path,
``ewaldmd.EwaldSolver(box, EwaldParams(...), workers, recip).evaluate(ps)``
(``ewald.py:599-655``), on inputs produced by this repository's seeded
generators (``paper_1708_01135_b200/workloads.py``), and stores energies,
forces and rho_hat (full for small systems, seeded samples for large ones)
plus a sha256 of the inputs so the tests can check that the regenerated
inputs are bit-identical.  The fixtures pin the C oracle (tests marked
``not gpu``) and the CUDA path (``-m gpu``).
"""

import hashlib
import math
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, REPO)
sys.path.insert(0, "/root/reference/pkg/src")

import ewaldmd as em  # noqa: E402  (the reference, read-only)

from paper_1708_01135_b200 import workloads as wl  # noqa: E402

WORKERS = os.cpu_count()
# sampled particles / k-vectors of the large configs (c5 was regenerated with
# EWB_GOLDEN_SAMPLE=8192)
N_SAMPLE = int(os.environ.get("EWB_GOLDEN_SAMPLE", "512"))


def input_digest(pos, q):
    h = hashlib.sha256()
    h.update(np.ascontiguousarray(pos, dtype=np.float64).tobytes())
    h.update(np.ascontiguousarray(q, dtype=np.float64).tobytes())
    return h.hexdigest()


def ref_evaluate(pos, q, L, params, m_int=None):
    box = em.SimulationBox(L)
    ps = em.create_particle_set(pos.shape[0], box)
    ps.position[:] = pos
    ps.charge[:] = q
    if m_int is None:
        rs = em.enumerate_kvectors(box, params)
    else:
        rs = em.ReciprocalSpace(box, params, m_int)
    solver = em.EwaldSolver(box, params, workers=WORKERS, recip=rs)
    t0 = time.perf_counter()
    res = solver.evaluate(ps)
    dt = time.perf_counter() - t0
    return dict(u_sr=res.u_sr, u_lr=res.u_lr, u_self=res.u_self,
                force=ps.force.copy(), rho=rs.rho.values.copy(),
                m_int=rs.m_int.astype(np.int64), coeff=rs.coeff.copy(),
                t_eval=dt, t_sr=res.t_sr, t_alg1=res.t_alg1,
                t_alg2=res.t_alg2)


def random_neutral(n, L, seed, min_sep=0.8):
    """Rejection-sampled neutral system with +-q charge pairs (own code)."""
    rng = np.random.default_rng(seed)
    pos = np.empty((n, 3))
    k = 0
    while k < n:
        c = rng.random(3) * L
        d = pos[:k] - c
        d -= L * np.floor(d / L + 0.5)
        if k and (d * d).sum(axis=1).min() < min_sep**2:
            continue
        pos[k] = c
        k += 1
    mag = rng.random(n // 2) + 0.5
    q = np.concatenate([mag, -mag])
    return pos, q


def save(name, **arrays):
    path = os.path.join(HERE, f"{name}.npz")
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)", flush=True)


def small_cases():
    cases = []
    # rock-salt 8-ion cell, tolerance-chosen parameters (r_c clamps to L/2,
    # so the reference runs its scan-all branch: engine.py:111-134)
    ps = em.init_rocksalt(1, 2.82)
    p = em.choose_parameters(ps.count, ps.box, 1e-6)
    cases.append(("rocksalt8", ps.position.copy(), ps.charge.copy(),
                  ps.box.edge_length, p, None))
    # random neutral systems with the reference's sphere k-table
    for n, L, seed, tol in ((32, 9.0, 21, 1e-6), (64, 12.0, 5, 1e-6),
                            (200, 15.0, 7, 1e-5)):
        pos, q = random_neutral(n, L, seed)
        p = em.choose_parameters(n, em.SimulationBox(L), tol)
        cases.append((f"rand{n}_s{seed}", pos, q, L, p, None))
    # cpd >= 3 stencil branch with a sphere table
    pos, q = random_neutral(600, 14.0, 11)
    p = em.EwaldParams(alpha=0.35, r_cutoff=4.6, k_cutoff=2.2, tolerance=1e-4)
    cases.append(("rand600_s11", pos, q, 14.0, p, None))
    # odd cube table and uneven charges
    pos, q = random_neutral(300, 10.0, 3)
    p = em.EwaldParams(alpha=0.5, r_cutoff=3.3, k_cutoff=3.0, tolerance=1e-4)
    cases.append(("rand300_cube5", pos, q, 10.0, p, wl.cube_half_m(5)))
    # r_cutoff > L/2: the reference's image-shell real space (ewald.py:553-576)
    pos, q = random_neutral(64, 12.0, 41)
    s_ = math.sqrt(-math.log(1e-6))
    p = em.EwaldParams(alpha=0.1, r_cutoff=s_ / math.sqrt(0.1),
                       k_cutoff=2.0 * s_ * math.sqrt(0.1), tolerance=1e-6)
    cases.append(("wide_rand64", pos, q, 12.0, p, None))
    ps8 = em.init_rocksalt(3, 2.5)
    rng = np.random.default_rng(3)
    pos8 = ps8.position + 0.1 * rng.standard_normal(ps8.position.shape)
    L8 = ps8.box.edge_length
    pos8 = pos8 - L8 * np.floor(pos8 / L8)
    base = em.choose_parameters(ps8.count, ps8.box, 1e-6)
    a = base.alpha * 0.5
    p = em.EwaldParams(alpha=a, r_cutoff=s_ / math.sqrt(a),
                       k_cutoff=2.0 * s_ * math.sqrt(a), tolerance=1e-6)
    cases.append(("wide_nacl216", pos8, ps8.charge.copy(), L8, p, None))
    for name, pos, q, L, p, m in cases:
        out = ref_evaluate(pos, q, L, p, m)
        save(name, pos=pos, q=q, L=L, alpha=p.alpha, r_cutoff=p.r_cutoff,
             k_cutoff=p.k_cutoff, tolerance=p.tolerance,
             u_sr=out["u_sr"], u_lr=out["u_lr"], u_self=out["u_self"],
             force=out["force"], rho=out["rho"], m_int=out["m_int"],
             coeff=out["coeff"])


def config_case(name):
    cfg = wl.make_config(name, seed=0)
    L = cfg["L"]
    params = em.EwaldParams(alpha=cfg["alpha_ref"], r_cutoff=cfg["r_cutoff"],
                            k_cutoff=wl.k_cutoff_for(cfg), tolerance=1e-6)
    print(f"{name}: N={cfg['pos'].shape[0]} K={cfg['m_int'].shape[0]} "
          f"alpha_cfg={cfg['alpha_cfg']} alpha_ref={cfg['alpha_ref']}",
          flush=True)
    out = ref_evaluate(cfg["pos"], cfg["q"], L, params, cfg["m_int"])
    print(f"{name}: t_eval={out['t_eval']:.2f}s u_sr={out['u_sr']!r} "
          f"u_lr={out['u_lr']!r} u_self={out['u_self']!r}", flush=True)
    n = cfg["pos"].shape[0]
    K = cfg["m_int"].shape[0]
    rng = np.random.default_rng(12345)
    f_idx = np.sort(rng.choice(n, size=min(n, N_SAMPLE), replace=False))
    k_idx = np.sort(rng.choice(K, size=min(K, N_SAMPLE), replace=False))
    f = out["force"]
    extra = {}
    if n <= 1000:
        extra = dict(force=f, rho=out["rho"], pos=cfg["pos"], q=cfg["q"])
    save(name, digest=input_digest(cfg["pos"], cfg["q"]), L=L,
         alpha=cfg["alpha_ref"], r_cutoff=cfg["r_cutoff"],
         n_max=cfg["n_max"], u_sr=out["u_sr"], u_lr=out["u_lr"],
         u_self=out["u_self"], f_idx=f_idx, f_sample=f[f_idx],
         k_idx=k_idx, rho_re_sample=out["rho"][k_idx],
         rho_im_sample=out["rho"][K + k_idx],
         f_rms=math.sqrt(float((f * f).sum()) / n),
         f_sum=f.sum(axis=0), t_eval=out["t_eval"], t_sr=out["t_sr"],
         t_alg1=out["t_alg1"], t_alg2=out["t_alg2"], workers=WORKERS,
         **extra)


def md_cases():
    """Reference ForceAssembler (Coulomb + LJ, LJ only) and a short NVE run."""
    from ewaldmd.driver import ForceAssembler
    rng = np.random.default_rng(77)
    ps = em.init_rocksalt(2, 3.5)            # N=64, L=14
    ps.position += 0.15 * rng.standard_normal(ps.position.shape)
    ps.wrap()
    pos0 = ps.position.copy()
    for tag, coul in (("md_fa_coul_lj", True), ("md_fa_lj", False)):
        cfg = em.SimConfig(n_particles=64, box_edge=14.0, tolerance=1e-6,
                           coulomb_on=coul, lj_on=True, threads=WORKERS,
                           lj=em.LJParams(epsilon_lj=1.0, sigma=2.5, r_cutoff_lj=6.25))
        ps.position[:] = pos0
        fa = ForceAssembler(ps, cfg)
        pe = fa(ps)
        save(tag, pos=pos0, q=ps.charge.copy(), L=14.0, pe=pe,
             u_coulomb=fa.last["u_coulomb"], u_lj=fa.last["u_lj"],
             force=ps.force.copy())
    # NVE trajectory
    cfg = em.SimConfig(n_particles=64, box_edge=14.0, tolerance=1e-6, dt=0.01,
                       n_steps=8, velocity_scale=0.05, threads=WORKERS, seed=1,
                       lj_on=True,
                       lj=em.LJParams(epsilon_lj=1.0, sigma=2.5, r_cutoff_lj=6.25))
    ps = em.init_rocksalt(2, 3.5)
    ps.position += 0.15 * np.random.default_rng(78).standard_normal(ps.position.shape)
    ps.wrap()
    pos0 = ps.position.copy()
    m = em.run(cfg, ps)
    save("md_run", pos0=pos0, q=ps.charge.copy(), L=14.0,
         energy_trace=np.array(m.energy_trace), pos_final=ps.position.copy(),
         vel_final=ps.velocity.copy(), alpha=m.alpha, r_cutoff=m.r_cutoff,
         max_disp=m.max_step_displacement)


def nve_acceptance_case():
    """The reference's acceptance criterion 8 run (test_acceptance.py:226-239):
    N=1728, Coulomb + LJ, dt 0.01, 1000 NVE steps; its energy trace and
    drift (the reference measures 4.19e-4 here, above the criterion's 1e-4)."""
    cfg = em.SimConfig(n_particles=1728, box_edge=30.0, tolerance=1e-6, dt=0.01,
                       n_steps=1000, velocity_scale=0.05, threads=WORKERS, seed=8,
                       coulomb_on=True, lj_on=True)
    m = em.run(cfg)
    save("md_nve1000", energy_trace=np.array(m.energy_trace), drift=m.drift,
         max_disp=m.max_step_displacement)


if __name__ == "__main__":
    which = sys.argv[1:] or ["small", "c1", "c2", "c3", "c4", "c5"]
    for w in which:
        if w == "small":
            small_cases()
        elif w == "md":
            md_cases()
        elif w == "nve":
            nve_acceptance_case()
        else:
            config_case(w)
