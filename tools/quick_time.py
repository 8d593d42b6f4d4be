import sys, time, numpy as np
sys.path.insert(0, '.')
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import workloads as wl
for name in sys.argv[1:]:
    cfg = wl.make_config(name)
    box = cfg['box']; ps = ew.create_particle_set(cfg['pos'].shape[0], box)
    ps.position[:] = cfg['pos']; ps.charge[:] = cfg['q']
    p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(box, p, cfg['m_int'])
    s = ew.EwaldSolver(box, p, recip=rs)
    print(name, s.handle.kspace_info(), flush=True)
    for it in range(4):
        t0 = time.perf_counter(); r = s.evaluate(ps); t1 = time.perf_counter()
        print(f"{name} wall {1e3*(t1-t0):.3f} ms  t_cell {1e3*r.t_cell:.3f} t_sr {1e3*r.t_sr:.3f} alg1 {1e3*r.t_alg1:.3f} alg2 {1e3*r.t_alg2:.3f} ms  E={r.total!r}", flush=True)
