"""Real-space time of one z-slab (the per-rank share of a multi-GPU step)
on one GPU: ewb_dev_real_space(part, nparts) for every part, max over parts
(CUDA events, min of 20), and the check that the slabs sum to the whole."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import _lib
from paper_1708_01135_b200 import workloads as wl
dev = torch.device('cuda', 0)
for name in sys.argv[1:]:
    cfg = wl.make_config(name)
    p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
    pos = torch.from_numpy(cfg['pos']).to(dev)
    q = torch.from_numpy(cfg['q']).to(dev)
    n = q.shape[0]
    st = torch.cuda.Stream()
    h = _lib.Handle(0)
    h.set_stream(st.cuda_stream)
    h.set_system(cfg['L'], p.alpha, p.r_cutoff)
    h.set_kspace(rs.m_int, rs.coeff)
    f = torch.zeros((n, 3), dtype=torch.float64, device=dev)
    with torch.cuda.stream(st):
        h.dev_load(pos.data_ptr(), q.data_ptr(), n)
        for nparts in (1, 2, 4, 8):
            worst, usum = 0.0, 0.0
            for part in range(nparts):
                best = 1e9
                for _ in range(20):
                    e0 = torch.cuda.Event(enable_timing=True)
                    e1 = torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    u = h.dev_real_space(part, nparts, f.data_ptr())
                    e1.record(st)
                    st.synchronize()
                    best = min(best, e0.elapsed_time(e1))
                worst = max(worst, best)
                usum += u
            print(f"{name} nparts={nparts} max slab {worst:.3f} ms  u_sr={usum!r}", flush=True)
