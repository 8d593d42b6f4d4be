"""Where the end-to-end time goes on c2: EwaldSolver.evaluate (public API,
pinned host arrays) vs the bare C-ABI call vs the device time."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import torch
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import workloads as wl
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
cfg = wl.make_config(name)
n = cfg['pos'].shape[0]
p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
ps = ew.create_particle_set(n, cfg['box'])
ps.position = torch.from_numpy(cfg['pos']).pin_memory().numpy()
ps.charge = torch.from_numpy(cfg['q']).pin_memory().numpy()
ps.force = torch.zeros((n, 3), dtype=torch.float64).pin_memory().numpy()
s = ew.EwaldSolver(cfg['box'], p, recip=rs)
rho_pin = torch.zeros(2 * rs.n_stored, dtype=torch.float64).pin_memory().numpy()
rho_page = np.zeros(2 * rs.n_stored)
def t(f, r=50):
    for _ in range(5):
        f()
    ts = []
    for _ in range(r):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return 1e3 * np.median(ts), 1e3 * min(ts)
print("evaluate (public API)   median/min ms", t(lambda: s.evaluate(ps)))
h = s.handle
print("C-ABI, rho pinned       ", t(lambda: h.evaluate(ps.position, ps.charge, ps.force, rho_pin)))
print("C-ABI, rho pageable     ", t(lambda: h.evaluate(ps.position, ps.charge, ps.force, rho_page)))
print("C-ABI, no rho           ", t(lambda: h.evaluate(ps.position, ps.charge, ps.force, None)))
r = s.evaluate(ps)
print("device stages ms", r.t_cell * 1e3, r.t_sr * 1e3, r.t_alg1 * 1e3, r.t_alg2 * 1e3)
