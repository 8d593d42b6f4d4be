"""Time the structure factor for several K1 pair-segment caps."""
import sys
sys.path.insert(0, '.')
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import workloads as wl
for name in sys.argv[2:]:
    cfg = wl.make_config(name)
    ps = ew.create_particle_set(cfg['pos'].shape[0], cfg['box'])
    ps.position[:] = cfg['pos']; ps.charge[:] = cfg['q']
    p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
    rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
    s = ew.EwaldSolver(cfg['box'], p, recip=rs)
    for mc in [int(x) for x in sys.argv[1].split(',')]:
        s.handle.set_max_pair_segment(mc); s.handle.set_kspace(rs.m_int, rs.coeff)
        info = s.handle.kspace_info()
        best = min((s.evaluate(ps) for _ in range(3)), key=lambda r: r.t_alg1)
        print(f"{name} mcap1 {mc:2d} M1 {info['M1']:2d} pitems {info['n_pair_items']:6d} alg1 {1e3*best.t_alg1:8.3f} ms u_lr {best.u_lr!r}", flush=True)
