"""Time the structure factor and the full evaluation for several k-column
segment caps (register footprint vs per-item setup overhead)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import workloads as wl
name = sys.argv[1]
caps = [int(x) for x in sys.argv[2].split(',')]
cfg = wl.make_config(name)
ps = ew.create_particle_set(cfg['pos'].shape[0], cfg['box'])
ps.position[:] = cfg['pos']; ps.charge[:] = cfg['q']
p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
s = ew.EwaldSolver(cfg['box'], p, recip=rs)
for mc in caps:
    s.handle.set_max_segment(mc); s.handle.set_kspace(rs.m_int, rs.coeff)
    info = s.handle.kspace_info()
    best = None
    for _ in range(3):
        r = s.evaluate(ps)
        if best is None or r.t_alg1 + r.t_alg2 < best.t_alg1 + best.t_alg2: best = r
    print(f"{name} mcap {mc:2d} M {info['M']:2d} items {info['n_items']:6d} alg1 {1e3*best.t_alg1:8.3f} alg2 {1e3*best.t_alg2:8.3f} ms  u_lr {best.u_lr!r}", flush=True)
