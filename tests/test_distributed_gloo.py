"""Multi-rank orchestration (distributed.ShardedEwald) under gloo, world 2,
on CPU: particle-sharded S(k) partials + all-reduce, z-slab real space,
force all-reduce must reproduce the single-process evaluation."""

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


def _worker(rank, world, port, name, out_dir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from cpu_stages import OracleStages
        from paper_1708_01135_b200 import workloads as wl
        from paper_1708_01135_b200.distributed import ShardedEwald
        cfg = wl.make_config(name, seed=0)
        st = OracleStages(cfg["L"], cfg["alpha_ref"], cfg["r_cutoff"], cfg["m_int"])
        sh = ShardedEwald(st, torch.device("cpu"))
        pos = torch.from_numpy(cfg["pos"])
        q = torch.from_numpy(cfg["q"])
        force = torch.zeros((q.shape[0], 3), dtype=torch.float64)
        rho = torch.zeros(2 * cfg["m_int"].shape[0], dtype=torch.float64)
        u = sh.evaluate(pos, q, force, rho_out=rho)
        np.savez(os.path.join(out_dir, f"rank{rank}.npz"), u=np.array(u),
                 force=force.numpy(), rho=rho.numpy())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_matches_single_process(tmp_path, world):
    import sys
    sys.path.insert(0, os.path.dirname(__file__))
    from oracle import oracle as orc
    from paper_1708_01135_b200 import workloads as wl
    port = _free_port()
    mp.spawn(_worker, args=(world, port, "c1", str(tmp_path)), nprocs=world, join=True)
    cfg = wl.make_config("c1", seed=0)
    ref = orc.evaluate(cfg["pos"], cfg["q"], cfg["L"], cfg["alpha_ref"],
                       cfg["r_cutoff"], cfg["m_int"])
    for r in range(world):
        got = np.load(tmp_path / f"rank{r}.npz")
        u_sr, u_lr, u_self = got["u"]
        assert rel(u_sr, ref["u_sr"]) <= 1e-12
        assert rel(u_lr, ref["u_lr"]) <= 1e-12
        assert rel(u_self, ref["u_self"]) <= 1e-14
        assert np.abs(got["force"] - ref["force"]).max() <= 1e-12 * f_rms(ref["force"])
        assert np.abs(got["rho"] - ref["rho"]).max() <= 1e-12 * np.abs(ref["rho"]).max()


def test_shard_range_partition():
    from paper_1708_01135_b200.distributed import shard_range
    for n in (1, 7, 1000, 32768):
        for w in (1, 2, 3, 8):
            rs = [shard_range(n, r, w) for r in range(w)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(w - 1))
            sizes = [b - a for a, b in rs]
            assert max(sizes) - min(sizes) <= 1
