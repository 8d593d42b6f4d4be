"""A/B: distributed.ShardedEwald on one GPU (world 1: the multi-GPU step
minus the collectives) with the real-space slab on a side stream vs in
sequence; min wall time of 30 steps per config."""
import sys
import time
sys.path.insert(0, '.')
import torch
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import _lib
from paper_1708_01135_b200 import workloads as wl
from paper_1708_01135_b200.distributed import DeviceStages, ShardedEwald
dev = torch.device('cuda', 0)
for name in sys.argv[1:]:
    cfg = wl.make_config(name)
    p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
    pos = torch.from_numpy(cfg['pos']).to(dev)
    q = torch.from_numpy(cfg['q']).to(dev)
    n = q.shape[0]
    st = torch.cuda.Stream()
    for ov in (False, True):
        h = _lib.Handle(0)
        h.set_stream(st.cuda_stream)
        h.set_system(cfg['L'], p.alpha, p.r_cutoff)
        h.set_kspace(rs.m_int, rs.coeff)
        sh = ShardedEwald(DeviceStages(h), dev, overlap=ov)
        f = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        ts = []
        with torch.cuda.stream(st):
            for it in range(35):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                u = sh.evaluate(pos, q, f)
                ts.append(time.perf_counter() - t0)
        print(f"{name} overlap={ov} step {1e3 * min(ts[5:]):.3f} ms  u={u}", flush=True)
