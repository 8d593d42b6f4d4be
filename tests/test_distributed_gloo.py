"""Multi-rank orchestration (distributed.SlabEwald / ShardedEwald) under gloo
on CPU with the oracle-backed stages: row ownership, halo exchange by grouped
send/receive, S(k) all-reduce, reverse force exchange and the owned-row
all-gather must reproduce the single-process evaluation."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from conftest import f_rms, rel


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def small_config(side=16, rc=4.0, beta=0.6, n_max=6, seed=3):
    """Rock salt side^3 (4096 charges, L=16): 4 r_c cells per edge, so 16
    rows of cells -- enough to give every rank a slab and a halo."""
    from paper_1708_01135_b200 import workloads as wl
    pos, q, L = wl.jittered_rocksalt(side, 1.0, 0.1, seed)
    return dict(pos=np.ascontiguousarray(pos), q=np.ascontiguousarray(q), L=float(L),
                alpha_ref=beta ** 2, r_cutoff=rc, m_int=wl.cube_half_m(n_max))


def _worker(rank, world, port, kind, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_stages import OracleStages
        from paper_1708_01135_b200 import workloads as wl
        from paper_1708_01135_b200.distributed import ShardedEwald
        cfg = wl.make_config("c1", seed=0) if kind == "c1" else small_config()
        st = OracleStages(cfg["L"], cfg["alpha_ref"], cfg["r_cutoff"], cfg["m_int"])
        sh = ShardedEwald(st, torch.device("cpu"))
        pos = torch.from_numpy(cfg["pos"])
        q = torch.from_numpy(cfg["q"])
        force = torch.zeros((q.shape[0], 3), dtype=torch.float64)
        rho = torch.zeros(2 * cfg["m_int"].shape[0], dtype=torch.float64)
        u = sh.evaluate(pos, q, force, rho_out=rho)
        sl = sh.slab
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=np.array(u),
                 force=force.numpy(), rho=rho.numpy(),
                 n_own=np.array(int(sl.owned_mask(st.rows(pos).long()).sum())))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind,world", [("small", 2), ("small", 3), ("small", 4), ("c1", 2)])
def test_sharded_matches_single_process(tmp_path, kind, world):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from oracle import oracle as orc
    from paper_1708_01135_b200 import workloads as wl
    port = _free_port()
    mp.spawn(_worker, args=(world, port, kind, str(tmp_path)), nprocs=world, join=True)
    cfg = wl.make_config("c1", seed=0) if kind == "c1" else small_config()
    ref = orc.evaluate(cfg["pos"], cfg["q"], cfg["L"], cfg["alpha_ref"],
                       cfg["r_cutoff"], cfg["m_int"])
    owned = 0
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npz")
        owned += int(got["n_own"])
        u_sr, u_lr, u_self = got["u"]
        assert rel(u_sr, ref["u_sr"]) <= 1e-12
        assert rel(u_lr, ref["u_lr"]) <= 1e-12
        assert rel(u_self, ref["u_self"]) <= 1e-13
        assert np.abs(got["force"] - ref["force"]).max() <= 1e-12 * f_rms(ref["force"])
        assert np.abs(got["rho"] - ref["rho"]).max() <= 1e-12 * np.abs(ref["rho"]).max()
    assert owned == cfg["q"].shape[0]  # every particle owned by exactly one rank


def test_halo_rows_half_and_full_shell():
    """Half-shell halo rows are the rows at lexicographically positive (oz, oy)
    offsets outside the slab; the full shell adds the mirror rows."""
    from paper_1708_01135_b200.distributed import halo_rows, row_bounds
    cpd, rad = 10, 2
    b = row_bounds(cpd * cpd, 4)
    assert b[0][0] == 0 and b[-1][1] == cpd * cpd
    lo, hi = b[1]
    half = set(halo_rows(lo, hi, cpd, rad, True).tolist())
    full = set(halo_rows(lo, hi, cpd, rad, False).tolist())
    assert half < full
    for r in half:
        assert not lo <= r < hi
    # brute force: the half-shell stencil of every owned row
    want = set()
    for r in range(lo, hi):
        cy, cz = r % cpd, r // cpd
        for oz in range(0, rad + 1):
            for oy in range(-rad, rad + 1):
                if oz == 0 and oy <= 0:
                    continue
                rr = (cy + oy) % cpd + cpd * ((cz + oz) % cpd)
                if not lo <= rr < hi:
                    want.add(rr)
    assert half == want


def test_shard_range_partition():
    from paper_1708_01135_b200.distributed import shard_range
    for n in (1, 7, 1000, 32768):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1


@pytest.mark.parametrize("world", [2, 3])
def test_thread_group_matches_single_process(world):
    """The in-process multi-GPU path behind EwaldSolver(workers=W): W host
    threads, one SlabEwald each, collectives through a ThreadGroup (barrier +
    rank-ordered sums), every rank's owned rows written into ONE force
    array.  Oracle-backed stages on CPU."""
    import sys
    import threading
    sys.path.insert(0, os.path.dirname(__file__))
    from cpu_stages import OracleStages
    from oracle import oracle as orc
    from paper_1708_01135_b200.distributed import SlabEwald, ThreadComm, ThreadGroup
    cfg = small_config()
    n = cfg["q"].shape[0]
    grp = ThreadGroup(world, timeout=120)
    force = np.zeros((n, 3))
    out = [None] * world

    def rank(r):
        st = OracleStages(cfg["L"], cfg["alpha_ref"], cfg["r_cutoff"], cfg["m_int"])
        sl = SlabEwald(st, torch.device("cpu"), n, comm=ThreadComm(grp, r, "cpu"))
        pos, q = torch.from_numpy(cfg["pos"]), torch.from_numpy(cfg["q"])
        mine = torch.nonzero(sl.owned_mask(st.rows(pos).long())).flatten()
        f_own = torch.zeros((mine.shape[0], 3), dtype=torch.float64)
        u = sl.evaluate_local(pos[mine].contiguous(), q[mine].contiguous(), f_own)
        out[r] = (u, mine.numpy(), f_own.numpy())

    ts = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert all(o is not None for o in out), "a rank failed"
    for _, idx, fo in out:
        force[idx] += fo
    assert sum(o[1].shape[0] for o in out) == n
    ref = orc.evaluate(cfg["pos"], cfg["q"], cfg["L"], cfg["alpha_ref"],
                       cfg["r_cutoff"], cfg["m_int"])
    for u_sr, u_lr, u_self in (o[0] for o in out):
        assert rel(u_sr, ref["u_sr"]) <= 1e-12
        assert rel(u_lr, ref["u_lr"]) <= 1e-12
        assert rel(u_self, ref["u_self"]) <= 1e-13
    assert np.abs(force - ref["force"]).max() <= 1e-12 * f_rms(ref["force"])


def test_thread_group_failure_releases_peers():
    """A rank that fails before a collective aborts the group: its peers get
    BrokenBarrierError instead of waiting forever."""
    import threading
    from paper_1708_01135_b200.distributed import ThreadComm, ThreadGroup
    grp = ThreadGroup(2, timeout=60)
    seen = []

    def ok():
        try:
            ThreadComm(grp, 0, "cpu").allreduce_(torch.ones(3))
        except threading.BrokenBarrierError:
            seen.append("broken")

    t = threading.Thread(target=ok)
    t.start()
    grp.abort()
    t.join(timeout=30)
    assert not t.is_alive() and seen == ["broken"]
