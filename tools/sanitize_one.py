"""One evaluation of a config through the public API (for compute-sanitizer)."""
import sys
sys.path.insert(0, '.')
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import workloads as wl
cfg = wl.make_config(sys.argv[1] if len(sys.argv) > 1 else 'c2')
p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
ps = ew.create_particle_set(cfg['pos'].shape[0], cfg['box'])
ps.position[:] = cfg['pos']; ps.charge[:] = cfg['q']
s = ew.EwaldSolver(cfg["box"], p, recip=rs)
s.handle.set_graphs(False)
s.handle.set_overlap(False)
if len(sys.argv) > 2:
    s.handle.set_max_split(int(sys.argv[2]))
r = s.evaluate(ps)
print(r, s.handle.last_pair_count())
