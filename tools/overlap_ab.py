"""A/B: reciprocal space on its own stream (overlap) vs sequential; whole
evaluation time (CUDA events around ewb_dev_evaluate), min of 30."""
import sys
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import _lib
from paper_1708_01135_b200 import workloads as wl
for name in sys.argv[1:]:
    cfg = wl.make_config(name)
    p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
    dev = torch.device('cuda', 0)
    pos = torch.from_numpy(cfg['pos']).to(dev)
    q = torch.from_numpy(cfg['q']).to(dev)
    n = q.shape[0]
    res = {}
    for ov in (False, True):
        h = _lib.Handle(0)
        st = torch.cuda.Stream()
        h.set_stream(st.cuda_stream)
        h.set_system(cfg['L'], p.alpha, p.r_cutoff)
        h.set_kspace(rs.m_int, rs.coeff)
        h.set_overlap(ov)
        f = torch.zeros((n, 3), dtype=torch.float64, device=dev)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ts = []
        for it in range(35):
            f.zero_()
            torch.cuda.synchronize()
            e0.record(st)
            en, tm = h.dev_evaluate(pos.data_ptr(), q.data_ptr(), n, f.data_ptr(), None, timings=True)
            e1.record(st)
            torch.cuda.synchronize()
            if it >= 5:
                ts.append(e0.elapsed_time(e1))
        res[ov] = (min(ts), en, f.cpu().numpy(), tm)
        print(f"{name} overlap={ov} eval {min(ts):.3f} ms  stages {[round(1e3*x,3) for x in tm]}", flush=True)
    fr = np.sqrt((res[False][2] ** 2).sum() / n)
    print(f"{name} dF/Frms {np.abs(res[True][2]-res[False][2]).max()/fr:.2e} dE {np.abs(np.array(res[True][1])-np.array(res[False][1])).max():.2e}")
