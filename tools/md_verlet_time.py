"""DeviceMD step time with Verlet pair lists (skin > 0) against rebuilding
every step (skin 0, the reference's rule): rock salt side^3 at unit spacing,
r_c 6 (alpha from choose_parameters at 1e-6), Coulomb + LJ, velocity scale 0.5.
usage: python tools/md_verlet_time.py SIDE [SKIN ...]"""
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_1708_01135_b200 import md  # noqa: E402

side = int(sys.argv[1]) if len(sys.argv) > 1 else 32
skins = [float(x) for x in sys.argv[2:]] or [0.0, 0.3, 0.6]
for skin in skins:
    cfg = md.SimConfig(n_particles=side ** 3, box_edge=float(side), tolerance=1e-6,
                       r_cutoff=6.0, dt=0.005, n_steps=30, velocity_scale=0.5,
                       seed=3, lj_on=True, lj=md.LJParams(0.05, 0.8, 2.0))
    cells = md.rocksalt_cells_for(cfg.n_particles)
    ps = md.init_rocksalt(cells, cfg.box_edge / (2 * cells))
    m = md.run(cfg, ps, skin=skin)
    print(f"side {side} skin {skin}: median step {1e3 * m.median_step_wall(5):.3f} ms, "
          f"t_sr {1e3 * m.median_component('t_sr', 5):.3f} ms, verlet {m.verlet}, "
          f"max step disp {m.max_step_displacement:.4f}, E drift {m.drift:.2e}", flush=True)
