"""Device-resident evaluation time (ewb_dev_evaluate, two streams, graphs),
min and median of R steps after warm-up, per config -- for A/B of builds
(EWALDB200_LIB).  usage: python tools/step_time.py c2 c4 ..."""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1708_01135_b200 as ew  # noqa: E402
from paper_1708_01135_b200 import _lib  # noqa: E402
from paper_1708_01135_b200 import workloads as wl  # noqa: E402

dev = torch.device('cuda', 0)
for name in sys.argv[1:]:
    cfg = wl.make_config(name)
    p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
    h = _lib.Handle(0)
    st = torch.cuda.Stream()
    h.set_stream(st.cuda_stream)
    h.set_system(cfg['L'], p.alpha, p.r_cutoff)
    h.set_kspace(rs.m_int, rs.coeff)
    pos = torch.from_numpy(cfg['pos']).to(dev)
    q = torch.from_numpy(cfg['q']).to(dev)
    n = q.shape[0]
    f = torch.zeros((n, 3), dtype=torch.float64, device=dev)
    l2 = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 30 if n < 500000 else 8
    ts = []
    for it in range(reps + 3):
        l2.add_(1.0)
        torch.cuda.synchronize()
        e0.record(st)
        en, _ = h.dev_evaluate(pos.data_ptr(), q.data_ptr(), n, f.data_ptr(), None)
        e1.record(st)
        torch.cuda.synchronize()
        if it >= 3:
            ts.append(e0.elapsed_time(e1))
    print(f"{name}: step min {min(ts):.4f} median {np.median(ts):.4f} ms  u = {sum(en)!r}", flush=True)
