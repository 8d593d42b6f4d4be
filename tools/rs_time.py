"""min-of-R real-space stage time (t_sr) per config through the public API."""
import sys
sys.path.insert(0, '.')
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import workloads as wl
for name in sys.argv[1:]:
    cfg = wl.make_config(name)
    p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
    ps = ew.create_particle_set(cfg['pos'].shape[0], cfg['box'])
    ps.position[:] = cfg['pos']; ps.charge[:] = cfg['q']
    s = ew.EwaldSolver(cfg["box"], p, recip=rs)
    s.handle.set_overlap(False)
    ts = []
    for _ in range(20):
        r = s.evaluate(ps)
        ts.append((r.t_sr, r.t_alg1, r.t_alg2))
    t = [min(x[i] for x in ts) * 1e3 for i in range(3)]
    print(f"{name} sr {t[0]:.3f} alg1 {t[1]:.3f} alg2 {t[2]:.3f} ms  u_sr {r.u_sr!r}", flush=True)
