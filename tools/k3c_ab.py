"""A/B: force gather with C*S in the constant bank vs shared memory."""
import sys
sys.path.insert(0, '.')
import numpy as np
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import workloads as wl
for name in sys.argv[1:]:
    cfg = wl.make_config(name)
    p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
    out = {}
    for on in (False, True):
        ps = ew.create_particle_set(cfg['pos'].shape[0], cfg['box'])
        ps.position[:] = cfg['pos']; ps.charge[:] = cfg['q']
        s = ew.EwaldSolver(cfg['box'], p, recip=rs)
        s.handle.set_const_gather(on)
        best = None
        for _ in range(3):
            ps.force[:] = 0.0
            r = s.evaluate(ps)
            best = r if best is None or r.t_alg2 < best.t_alg2 else best
        out[on] = (best, ps.force.copy())
        print(f"{name} const={on} alg2 {1e3*best.t_alg2:.3f} ms", flush=True)
    fr = np.sqrt((out[False][1]**2).sum() / cfg['pos'].shape[0])
    print(f"{name} max dF/F_rms {np.abs(out[True][1]-out[False][1]).max()/fr:.2e}", flush=True)
