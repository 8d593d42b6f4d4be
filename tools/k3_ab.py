"""A/B timing of reciprocal-stage variants (EWALDB200_LIB selects the .so):
min-of-R sequential alg1/alg2 stage times per config, plus u_lr and a force
checksum (variants that only reorganise work must agree bitwise)."""
import sys
import numpy as np
sys.path.insert(0, '.')
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import workloads as wl
reps = 12
for name in sys.argv[1:]:
    cfg = wl.make_config(name)
    p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
    ps = ew.create_particle_set(cfg['pos'].shape[0], cfg['box'])
    ps.position[:] = cfg['pos']; ps.charge[:] = cfg['q']
    s = ew.EwaldSolver(cfg["box"], p, recip=rs)
    s.handle.set_overlap(False)
    ts = []
    for _ in range(reps if name != 'c5' else 4):
        ps.force[:] = 0.0
        r = s.evaluate(ps)
        ts.append((r.t_sr, r.t_alg1, r.t_alg2))
    t = [min(x[i] for x in ts) * 1e3 for i in range(3)]
    print(f"{name} sr {t[0]:.3f} alg1 {t[1]:.3f} alg2 {t[2]:.3f} ms  u_lr {r.u_lr!r} fsum {np.abs(ps.force).sum()!r}", flush=True)
