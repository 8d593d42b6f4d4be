"""The multi-GPU path on the product device stages: distributed.ShardedEwald
(row ownership, halo exchange by grouped send/receive, S(k) all-reduce,
reverse force exchange, owned-row all-gather) with W ranks spawned on the
one GPU of the test box and gloo for the collectives (they go through host
memory, so no kernel of one rank waits on another's), against the
reference's golden vectors of c2-c5.  world 8 on c4 exercises the two-hop
halo (a slab of 2.4 cell layers under a 3-layer stencil)."""

import os
import socket

import numpy as np
import pytest

from conftest import golden, rel

pytestmark = pytest.mark.gpu


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, name, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1708_01135_b200 as ew
        from paper_1708_01135_b200 import _lib
        from paper_1708_01135_b200 import workloads as wl
        from paper_1708_01135_b200.distributed import DeviceStages, ShardedEwald
        cfg = wl.make_config(name, seed=0)
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        params = ew.EwaldParams(cfg["alpha_ref"], cfg["r_cutoff"], wl.k_cutoff_for(cfg), 1e-6)
        rs = ew.ReciprocalSpace(cfg["box"], params, cfg["m_int"])
        h = _lib.Handle(0)
        h.set_system(cfg["L"], params.alpha, params.r_cutoff)
        h.set_kspace(rs.m_int, rs.coeff)
        pos = torch.from_numpy(cfg["pos"]).to(dev)
        q = torch.from_numpy(cfg["q"]).to(dev)
        n = q.shape[0]
        f = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        rho = torch.zeros(2 * rs.n_stored, dtype=torch.float64, device=dev)
        sh = ShardedEwald(DeviceStages(h), dev)
        u = sh.evaluate(pos, q, f, rho_out=rho)
        torch.cuda.synchronize()
        sl = sh.slab
        n_own = int(sl.owned_mask(DeviceStages(h).rows(pos).long()).sum())
        g = golden(name)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=np.array(u),
                 f_sample=f.cpu().numpy()[g["f_idx"]],
                 rho=rho.cpu().numpy(), n_own=np.array(n_own), n=np.array(n),
                 f_rms=np.array(float(torch.sqrt((f * f).sum() / n))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,world,peer", [("c2", 2, "0"), ("c3", 2, "0"), ("c4", 4, "0"),
                                             ("c4", 8, "0"), ("c5", 2, "0"), ("c2", 2, "1"),
                                             ("c4", 4, "1")])
def test_sharded_device_stages_match_golden(tmp_path, monkeypatch, name, world, peer):
    """peer = "1": the S(k) reduction fused into the finalising kernel, which
    reads the other ranks' partials through CUDA IPC (the ranks are
    processes; here they share the one GPU)."""
    monkeypatch.setenv("EWALDB200_PEER_FINALIZE", peer)
    import torch.multiprocessing as mp
    g = golden(name)
    port = _free_port()
    mp.spawn(_worker, args=(world, port, name, str(tmp_path)), nprocs=world, join=True)
    fr = float(g["f_rms"])
    k = g["k_idx"]
    owned = 0
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npz")
        owned += int(got["n_own"])
        u_sr, u_lr, u_self = got["u"]
        assert rel(u_sr, float(g["u_sr"])) <= 1e-10
        assert rel(u_lr, float(g["u_lr"])) <= 1e-10
        assert rel(u_self, float(g["u_self"])) <= 1e-10
        assert np.abs(got["f_sample"] - g["f_sample"]).max() <= 1e-9 * fr
        assert abs(float(got["f_rms"]) - fr) <= 1e-9 * fr
        K = got["rho"].shape[0] // 2
        rmax = max(np.abs(g["rho_re_sample"]).max(), np.abs(g["rho_im_sample"]).max())
        assert np.abs(got["rho"][k] - g["rho_re_sample"]).max() <= 1e-12 * rmax
        assert np.abs(got["rho"][K + k] - g["rho_im_sample"]).max() <= 1e-12 * rmax
    assert owned == int(got["n"])  # every particle owned by exactly one rank


@pytest.mark.parametrize("name,workers", [("c2", 2), ("c4", 3), ("c3", 4)])
def test_solver_workers_shards_over_devices(monkeypatch, name, workers):
    """EwaldSolver(box, params, workers=W) -- the reference signature, W read
    as the GPU count -- runs the W-rank slab decomposition inside the
    caller's process (one host thread per rank; on this one-GPU box the ranks
    share device 0) and must match the reference's golden vectors."""
    import paper_1708_01135_b200 as ew
    from paper_1708_01135_b200 import workloads as wl
    monkeypatch.setenv("EWALDB200_SHARE_DEVICES", "1")
    cfg = wl.make_config(name, seed=0)
    g = golden(name)
    box = ew.SimulationBox(cfg["L"])
    ps = ew.create_particle_set(cfg["pos"].shape[0], box)
    ps.position[:] = cfg["pos"]
    ps.charge[:] = cfg["q"]
    params = ew.EwaldParams(cfg["alpha_ref"], cfg["r_cutoff"], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(box, params, cfg["m_int"])
    solver = ew.EwaldSolver(box, params, workers=workers, recip=rs)
    assert solver._multi is not None and solver._multi.world == workers
    for rep in range(2):           # second call: reused slabs and handles
        ps.force[:] = 0.0
        res = solver.evaluate(ps)
        assert rel(res.u_sr, float(g["u_sr"])) <= 1e-10
        assert rel(res.u_lr, float(g["u_lr"])) <= 1e-10
        assert rel(res.u_self, float(g["u_self"])) <= 1e-10
        fr = float(g["f_rms"])
        assert np.abs(ps.force[g["f_idx"]] - g["f_sample"]).max() <= 1e-9 * fr
        k = g["k_idx"]
        K = rs.n_stored
        rmax = max(np.abs(g["rho_re_sample"]).max(), np.abs(g["rho_im_sample"]).max())
        assert np.abs(rs.rho.values[k] - g["rho_re_sample"]).max() <= 1e-12 * rmax
        assert np.abs(rs.rho.values[K + k] - g["rho_im_sample"]).max() <= 1e-12 * rmax
    solver._multi.close()


def test_solver_workers_errors_leave_forces(monkeypatch):
    """A coincident pair in one rank's slab: every rank raises together and
    the caller's force array is untouched."""
    import paper_1708_01135_b200 as ew
    from paper_1708_01135_b200 import workloads as wl
    monkeypatch.setenv("EWALDB200_SHARE_DEVICES", "1")
    cfg = wl.make_config("c2", seed=0)
    box = ew.SimulationBox(cfg["L"])
    ps = ew.create_particle_set(cfg["pos"].shape[0], box)
    ps.position[:] = cfg["pos"]
    ps.position[7] = ps.position[8]
    ps.charge[:] = cfg["q"]
    ps.force[:] = 1.25
    params = ew.EwaldParams(cfg["alpha_ref"], cfg["r_cutoff"], wl.k_cutoff_for(cfg), 1e-6)
    solver = ew.EwaldSolver(box, params, workers=2,
                            recip=ew.ReciprocalSpace(box, params, cfg["m_int"]))
    with pytest.raises(ew.CoincidentParticlesError):
        solver.evaluate(ps)
    assert np.all(ps.force == 1.25)
    solver._multi.close()


def test_solver_workers_wide_cutoff_stays_single_gpu(monkeypatch):
    """r_c > L/2 (the image-shell path, N <= 4096) runs on one GPU even when
    workers asks for more; results are the reference's."""
    import paper_1708_01135_b200 as ew
    monkeypatch.setenv("EWALDB200_SHARE_DEVICES", "1")
    g = golden("wide_rand64")
    box = ew.SimulationBox(float(g["L"]))
    ps = ew.create_particle_set(g["pos"].shape[0], box)
    ps.position[:] = g["pos"]
    ps.charge[:] = g["q"]
    params = ew.EwaldParams(float(g["alpha"]), float(g["r_cutoff"]), float(g["k_cutoff"]),
                            float(g["tolerance"]))
    solver = ew.EwaldSolver(box, params, workers=2, recip=ew.ReciprocalSpace(box, params, g["m_int"]))
    assert solver._multi is None
    res = solver.evaluate(ps)
    assert rel(res.u_sr, float(g["u_sr"])) <= 1e-10
    assert rel(res.u_lr, float(g["u_lr"])) <= 1e-10


def test_peer_finalize_equals_allreduce_then_finalize():
    """ewb_dev_kspace_finalize_peer (the S(k) reduction read from the ranks'
    buffers inside the finalising kernel) gives bitwise the rho and u_lr of
    summing the partials first and finalising them."""
    import torch
    import paper_1708_01135_b200 as ew
    from paper_1708_01135_b200 import _lib
    from paper_1708_01135_b200 import workloads as wl
    cfg = wl.make_config("c2", seed=0)
    dev = torch.device("cuda", 0)
    params = ew.EwaldParams(cfg["alpha_ref"], cfg["r_cutoff"], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg["box"], params, cfg["m_int"])
    h = _lib.Handle(0)
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    h.set_system(cfg["L"], params.alpha, params.r_cutoff)
    h.set_kspace(rs.m_int, rs.coeff)
    pos = torch.from_numpy(cfg["pos"]).to(dev)
    q = torch.from_numpy(cfg["q"]).to(dev)
    n = q.shape[0]
    ns = h.dev_slot_doubles()
    parts = [torch.empty(ns, dtype=torch.float64, device=dev) for _ in range(3)]
    cuts = [0, n // 3, (2 * n) // 3, n]
    with torch.cuda.stream(st):
        h.dev_load(pos.data_ptr(), q.data_ptr(), n)
        for r in range(3):
            h.dev_rho_partial(cuts[r], cuts[r + 1], parts[r].data_ptr())
        summed = parts[0].clone()
        summed += parts[1]
        summed += parts[2]
        rho_a = torch.empty(2 * rs.n_stored, dtype=torch.float64, device=dev)
        rho_b = torch.empty_like(rho_a)
        u_a = h.dev_kspace_finalize(summed.data_ptr(), rho_a.data_ptr())
        h.dev_kspace_finalize_peer([p.data_ptr() for p in parts], rho_b.data_ptr())
        e = torch.zeros(3, dtype=torch.float64, device=dev)
        h.dev_energies(e.data_ptr())
    torch.cuda.synchronize()
    assert torch.equal(rho_a, rho_b)
    assert e[1].item() == u_a


def _worker_err(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1708_01135_b200 as ew
        from paper_1708_01135_b200 import _lib
        from paper_1708_01135_b200 import workloads as wl
        from paper_1708_01135_b200.distributed import DeviceStages, ShardedEwald
        cfg = wl.make_config("c2", seed=0)
        dev = torch.device("cuda", 0)
        torch.cuda.set_device(dev)
        params = ew.EwaldParams(cfg["alpha_ref"], cfg["r_cutoff"], wl.k_cutoff_for(cfg), 1e-6)
        rs = ew.ReciprocalSpace(cfg["box"], params, cfg["m_int"])
        h = _lib.Handle(0)
        h.set_system(cfg["L"], params.alpha, params.r_cutoff)
        h.set_kspace(rs.m_int, rs.coeff)
        pos = cfg["pos"].copy()
        pos[11] = pos[12]                   # a coincident pair in one rank's slab
        pd = torch.from_numpy(pos).to(dev)
        q = torch.from_numpy(cfg["q"]).to(dev)
        f = torch.full((q.shape[0], 3), 0.5, dtype=torch.float64, device=dev)
        what = "none"
        try:
            ShardedEwald(DeviceStages(h), dev).evaluate(pd, q, f)
        except ew.CoincidentParticlesError:
            what = "coincident"
        untouched = bool(torch.all(f == 0.5).item())
        np.savez(os.path.join(out_dir, f"err{rank}.npz"), what=np.array(what),
                 untouched=np.array(untouched))
    finally:
        dist.destroy_process_group()


def test_sharded_error_raised_on_every_rank(tmp_path):
    """A coincident pair in one rank's rows: the device error flag travels
    with the energies, so EVERY rank raises CoincidentParticlesError and no
    rank writes its force array."""
    import torch.multiprocessing as mp
    world = 3
    mp.spawn(_worker_err, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        got = np.load(tmp_path / f"err{r}.npz")
        assert str(got["what"]) == "coincident"
        assert bool(got["untouched"])
