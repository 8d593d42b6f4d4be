"""The tensor-core structure factor (k1_tc.cuh: int8 tcgen05 MMA on six
48-bit fixed-point slices) against the oracle and against the FP64-pipe
kernel on the same inputs: ragged particle counts, zero and wide-range
charges, sparse / permuted / +-m_x k-sets and several a-chunks.

Tolerance: the reference's rho bound, 1e-12 * max|rho| (test_ewald.py:184-190);
the scheme itself is ~1e-15 (see k1_tc.cuh)."""

import numpy as np
import pytest

from conftest import f_rms, random_neutral, rel

pytestmark = pytest.mark.gpu

RHO_TOL = 1e-12


@pytest.fixture(scope="module")
def ew():
    import paper_1708_01135_b200 as ew
    return ew


@pytest.fixture(scope="module")
def orc():
    from oracle import oracle as orc
    return orc


def _rho(ew, pos, q, L, m, tc):
    box = ew.SimulationBox(L)
    ps = ew.create_particle_set(pos.shape[0], box)
    ps.position[:] = pos
    ps.charge[:] = q
    params = ew.EwaldParams(0.5, min(4.0, 0.49 * L), 5.0, 1e-6)
    rs = ew.ReciprocalSpace(box, params, m)
    h = ew.ewald._handle_for(rs)
    h.set_tensor_cores(tc)
    ew.compute_rho_hat(ps, rs)
    return rs.rho.values.copy()


def _check(ew, orc, pos, q, L, m):
    ref = orc.rho_hat(pos, q, L, m)
    scale = max(np.abs(ref).max(), 1e-300)
    got = _rho(ew, pos, q, L, m, True)
    assert np.abs(got - ref).max() <= RHO_TOL * scale
    fp = _rho(ew, pos, q, L, m, False)
    assert np.abs(got - fp).max() <= RHO_TOL * scale


@pytest.mark.parametrize("n", [1, 3, 63, 64, 65, 200, 1000])
def test_ragged_particle_counts(ew, orc, n):
    rng = np.random.default_rng(n)
    L = 9.0
    pos = rng.random((n, 3)) * L
    q = rng.standard_normal(n)
    from paper_1708_01135_b200 import workloads as wl
    _check(ew, orc, pos, q, L, wl.cube_half_m(6))


def test_zero_and_wide_range_charges(ew, orc):
    rng = np.random.default_rng(7)
    n, L = 500, 10.0
    pos = rng.random((n, 3)) * L
    q = rng.standard_normal(n) * np.exp(rng.uniform(-7, 2, n))
    q[::7] = 0.0
    from paper_1708_01135_b200 import workloads as wl
    _check(ew, orc, pos, q, L, wl.cube_half_m(7))


def test_all_zero_charges(ew):
    from paper_1708_01135_b200 import workloads as wl
    rng = np.random.default_rng(1)
    got = _rho(ew, rng.random((100, 3)) * 8.0, np.zeros(100), 8.0, wl.cube_half_m(4), True)
    assert np.all(got == 0.0)


def test_sparse_full_sphere_kset_with_both_signs(ew, orc):
    """A permuted random subset of the full sphere: +-m_x pairs, unpaired
    columns, gaps in m_y runs."""
    rng = np.random.default_rng(3)
    r = np.arange(-9, 10)
    mx, my, mz = np.meshgrid(r, r, r, indexing="ij")
    m = np.stack([mx.ravel(), my.ravel(), mz.ravel()], axis=1)
    m = m[(m ** 2).sum(1) <= 81]
    m = m[np.any(m != 0, axis=1)]
    m = m[rng.random(m.shape[0]) < 0.6]
    m = m[rng.permutation(m.shape[0])]
    pos, q = random_neutral(300, 11.0, seed=2)
    _check(ew, orc, pos, q, 11.0, m)


def test_many_a_chunks(ew, orc):
    """|m_x| up to 130: several 80-column a-chunks."""
    m = np.array([[a, b, c] for a in range(0, 131) for b in (-1, 0, 2) for c in (0, 1)
                  if (a, b, c) != (0, 0, 0)])
    pos, q = random_neutral(256, 12.0, seed=5)
    _check(ew, orc, pos, q, 12.0, m)


def test_energies_forces_tc_vs_fp64_pipe(ew):
    from paper_1708_01135_b200 import workloads as wl
    cfg = wl.make_config("c4")
    p = ew.EwaldParams(cfg["alpha_ref"], cfg["r_cutoff"], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg["box"], p, cfg["m_int"])
    out = {}
    for tc in (True, False):
        ps = ew.create_particle_set(cfg["pos"].shape[0], cfg["box"])
        ps.position[:] = cfg["pos"]
        ps.charge[:] = cfg["q"]
        s = ew.EwaldSolver(cfg["box"], p, recip=rs)
        s.handle.set_tensor_cores(tc)
        out[tc] = (s.evaluate(ps), ps.force.copy())
    (r1, f1), (r0, f0) = out[True], out[False]
    assert rel(r1.u_lr, r0.u_lr) <= 1e-12
    assert np.abs(f1 - f0).max() <= 1e-11 * f_rms(f0)


def test_overlap_and_modes_agree(ew):
    """Two-stream overlap vs sequential (bitwise: same kernels, same order per
    stream), and the auto / forced / FP64 reciprocal modes (tolerance)."""
    from paper_1708_01135_b200 import workloads as wl
    cfg = wl.make_config("c2")
    p = ew.EwaldParams(cfg["alpha_ref"], cfg["r_cutoff"], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg["box"], p, cfg["m_int"])

    def run(overlap=True, mode="auto"):
        ps = ew.create_particle_set(cfg["pos"].shape[0], cfg["box"])
        ps.position[:] = cfg["pos"]
        ps.charge[:] = cfg["q"]
        s = ew.EwaldSolver(cfg["box"], p, recip=rs)
        s.handle.set_overlap(overlap)
        s.handle.set_tensor_cores(mode)
        res = [s.evaluate(ps) for _ in range(3)][-1]  # eager, capture, replay
        return res, ps.force.copy(), rs.rho.values.copy()

    r1, f1, rho1 = run(True)
    r0, f0, rho0 = run(False)
    assert (r1.u_sr, r1.u_lr, r1.u_self) == (r0.u_sr, r0.u_lr, r0.u_self)
    assert np.array_equal(rho1, rho0)
    assert np.abs(f1 - f0).max() <= 1e-13 * f_rms(f0)  # real-space atomics order
    r2, f2, _ = run(True, False)
    assert rel(r2.u_lr, r1.u_lr) <= 1e-12
    assert np.abs(f2 - f1).max() <= 1e-11 * f_rms(f1)


def test_rho_storage_is_written_in_place(ew):
    from paper_1708_01135_b200 import workloads as wl
    cfg = wl.make_config("c1")
    p = ew.EwaldParams(cfg["alpha_ref"], cfg["r_cutoff"], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg["box"], p, cfg["m_int"])
    buf = rs.rho.values
    ps = ew.create_particle_set(cfg["pos"].shape[0], cfg["box"])
    ps.position[:] = cfg["pos"]
    ps.charge[:] = cfg["q"]
    ew.EwaldSolver(cfg["box"], p, recip=rs).evaluate(ps)
    assert rs.rho.values is buf and np.abs(buf).max() > 0.0
    # a caller-replaced (e.g. read-only or foreign) array still receives rho
    ro = np.zeros(buf.shape)
    rs.rho.values = ro
    ew.compute_rho_hat(ps, rs)
    assert rs.rho.values is ro and np.array_equal(ro, buf)


def test_skewed_charges_and_tiny_tables(ew, orc):
    """One charge 1e4 times the others (the fixed-point scale is max|q|), a
    single k-vector, and a one-particle system, all on the tensor cores."""
    rng = np.random.default_rng(11)
    n, L = 300, 10.0
    pos = rng.random((n, 3)) * L
    q = rng.standard_normal(n) * 1e-2
    q[17] = 100.0
    q -= q.mean()
    from paper_1708_01135_b200 import workloads as wl
    _check(ew, orc, pos, q, L, wl.cube_half_m(6))
    _check(ew, orc, pos, q, L, np.array([[1, 0, 0]]))
    _check(ew, orc, pos[:1], np.array([1.0]), L, wl.cube_half_m(3))


def test_forces_on_skewed_charges_tc_vs_fp64(ew):
    rng = np.random.default_rng(5)
    n, L = 400, 11.0
    pos, q = random_neutral(n, L, seed=9)
    q = q * np.exp(rng.uniform(-4, 1, n))
    q -= q.mean()
    box = ew.SimulationBox(L)
    p = ew.EwaldParams(0.4, 4.5, 6.0, 1e-6)
    from paper_1708_01135_b200 import workloads as wl
    rs = ew.ReciprocalSpace(box, p, wl.cube_half_m(9))
    out = {}
    for tc in (True, False):
        ps = ew.create_particle_set(n, box)
        ps.position[:] = pos
        ps.charge[:] = q
        s = ew.EwaldSolver(box, p, recip=rs)
        s.handle.set_tensor_cores(tc)
        out[tc] = (s.evaluate(ps), ps.force.copy())
    (r1, f1), (r0, f0) = out[True], out[False]
    assert rel(r1.u_lr, r0.u_lr) <= 1e-12
    # the reference's own Alg. 2 bound (test_ewald.py:230-239): 1e-12 max|F|
    assert np.abs(f1 - f0).max() <= 1e-12 * np.abs(f0).max()
