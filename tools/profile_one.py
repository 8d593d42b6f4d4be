"""Small driver for ncu: N evaluations of one config through the public API.
usage: python tools/profile_one.py CONFIG [REPS] [fp64]   (fp64: reciprocal
sums on the FP64-pipe kernels, ewb_set_tensor_cores(0))"""
import sys
sys.path.insert(0, '.')
import paper_1708_01135_b200 as ew  # noqa: E402
from paper_1708_01135_b200 import workloads as wl  # noqa: E402
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
cfg = wl.make_config(name)
ps = ew.create_particle_set(cfg['pos'].shape[0], cfg['box'])
ps.position[:] = cfg['pos']
ps.charge[:] = cfg['q']
p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
s = ew.EwaldSolver(cfg['box'], p, recip=ew.ReciprocalSpace(cfg['box'], p, cfg['m_int']))
if len(sys.argv) > 3 and sys.argv[3] == 'fp64':
    s.handle.set_tensor_cores(False)
for _ in range(reps):
    r = s.evaluate(ps)
print(name, r)
