"""Tensor-core structure factor vs the FP64-pipe kernel and the goldens:
rho_hat, u_lr and forces, plus timings of Alg. 1 (t_alg1)."""
import sys
import time
sys.path.insert(0, '.')
import numpy as np
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import workloads as wl


def run(name):
    cfg = wl.make_config(name)
    p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
    res = {}
    for tc in (False, True):
        ps = ew.create_particle_set(cfg['pos'].shape[0], cfg['box'])
        ps.position[:] = cfg['pos']; ps.charge[:] = cfg['q']
        s = ew.EwaldSolver(cfg['box'], p, recip=rs)
        s.handle.set_tensor_cores(tc)
        best = None
        for _ in range(4):
            ps.force[:] = 0.0
            r = s.evaluate(ps)
            best = r if best is None or r.t_alg1 < best.t_alg1 else best
        f = ps.force.copy()
        h = ew.ewald._handle_for(rs)
        h.set_tensor_cores(tc)
        ew.compute_rho_hat(ps, rs)
        res[tc] = (best, f, rs.rho.values.copy())
        print(f"{name} tc={tc} alg1 {1e3*best.t_alg1:.3f} ms  alg2 {1e3*best.t_alg2:.3f} "
              f"sr {1e3*best.t_sr:.3f} u_lr {best.u_lr!r}", flush=True)
    (b0, f0, r0), (b1, f1, r1) = res[False], res[True]
    fr = np.sqrt((f0 ** 2).sum() / f0.shape[0])
    print(f"{name} rel u_lr {abs(b1.u_lr-b0.u_lr)/abs(b0.u_lr):.2e}  max dF/Frms "
          f"{np.abs(f1-f0).max()/fr:.2e}  max|drho|/max|rho| {np.abs(r1-r0).max()/np.abs(r0).max():.2e}",
          flush=True)


for name in sys.argv[1:]:
    run(name)
