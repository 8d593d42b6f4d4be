"""Host-side cost of the multi-GPU orchestration at world 1: ShardedEwald
(stage API, Python, no collectives) against the single-call device pipeline
(ewb_dev_evaluate), per config.  usage: python tools/sharded_overhead.py c2"""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1708_01135_b200 as ew  # noqa: E402
from paper_1708_01135_b200 import _lib  # noqa: E402
from paper_1708_01135_b200 import workloads as wl  # noqa: E402
from paper_1708_01135_b200.distributed import DeviceStages, ShardedEwald  # noqa: E402

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
    sh = ShardedEwald(DeviceStages(h), dev)

    def t_of(fn, reps=30):
        ts = []
        for it in range(reps + 3):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            fn()
            torch.cuda.synchronize()
            if it >= 3:
                ts.append(time.perf_counter() - t0)
        return 1e3 * float(np.median(ts))
    with torch.cuda.stream(st):
        t_sh = t_of(lambda: sh.evaluate(pos, q, f))
    h.set_stream(st.cuda_stream)
    t_dev = t_of(lambda: h.dev_evaluate(pos.data_ptr(), q.data_ptr(), n, f.data_ptr(), None))
    print(f"{name}: ShardedEwald (world 1) {t_sh:.3f} ms, ewb_dev_evaluate {t_dev:.3f} ms (wall)",
          flush=True)
