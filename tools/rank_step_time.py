"""Per-rank device time of the domain-decomposed step (distributed.SlabEwald),
simulated on one GPU without the collectives: for every rank r of W, load
its own particles + its half-shell halo rows, run the pair kernel over its
own rows, its S(k) partial, the full-K finalisation and its reciprocal
forces + self energy, in sequence (CUDA events, min of R repetitions).
Prints the slowest rank's stage times per W: the step time of W GPUs is
that plus the collectives (halo send/receive, the S(k) all-reduce, the
reverse exchange, the 4-double energy all-reduce).

usage: python tools/rank_step_time.py CONFIG [W ...]"""
import sys

import numpy as np
import torch

sys.path.insert(0, '.')
import paper_1708_01135_b200 as ew  # noqa: E402
from paper_1708_01135_b200 import _lib  # noqa: E402
from paper_1708_01135_b200 import workloads as wl  # noqa: E402
from paper_1708_01135_b200.distributed import DeviceStages, halo_rows, row_bounds  # noqa: E402

dev = torch.device('cuda', 0)
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
worlds = [int(x) for x in sys.argv[2:]] or [1, 2, 4, 8]
cfg = wl.make_config(name)
p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
pos = torch.from_numpy(cfg['pos']).to(dev)
q = torch.from_numpy(cfg['q']).to(dev)
n = q.shape[0]
st = torch.cuda.Stream()
h = _lib.Handle(0)
h.set_system(cfg['L'], p.alpha, p.r_cutoff)
h.set_kspace(rs.m_int, rs.coeff)
stages = DeviceStages(h)
stages.set_geometry_n(n)
g = stages.geometry()
slots = torch.empty(h.dev_slot_doubles(), dtype=torch.float64, device=dev)
reps = 3 if n > 500000 else 10
with torch.cuda.stream(st):
    rows = stages.rows(pos).long()
for W in worlds:
    worst, worst_r = None, -1
    for r, (lo, hi) in enumerate(row_bounds(g['n_rows'], W)):
        own = torch.nonzero((rows >= lo) & (rows < hi)).flatten()
        halo = torch.from_numpy(halo_rows(lo, hi, g['cpd'], g['rad'], True)).to(dev)
        need = torch.zeros(g['n_rows'], dtype=torch.bool, device=dev)
        if W > 1 and halo.numel():
            need[halo] = True
        hidx = torch.nonzero(need[rows]).flatten()
        lp = torch.cat([pos[own], pos[hidx]]).contiguous()
        lq = torch.cat([q[own], q[hidx]]).contiguous()
        n_own = own.numel()
        f = torch.zeros((lq.numel(), 3), dtype=torch.float64, device=dev)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        best = None
        with torch.cuda.stream(st):
            h.set_stream(st.cuda_stream)
            for _ in range(reps):
                torch.cuda.synchronize()
                ev[0].record(st)
                h.dev_load(lp.data_ptr(), lq.data_ptr(), lq.numel())
                h.dev_real_space_rows_async(lo, hi, f.data_ptr())
                ev[1].record(st)
                h.dev_rho_partial(0, n_own, slots.data_ptr())
                ev[2].record(st)
                h.dev_kspace_finalize_async(slots.data_ptr(), None)
                h.dev_recip_forces(0, n_own, f.data_ptr())
                h.dev_self_energy_range_async(0, n_own)
                ev[3].record(st)
                h.dev_check()
                t = [ev[k].elapsed_time(ev[k + 1]) for k in range(3)]
                if best is None or sum(t) < sum(best):
                    best = t
        if worst is None or sum(best) > sum(worst):
            worst, worst_r = best, r
            halo_n = hidx.numel()
    print(f"{name} W={W}: slowest rank {worst_r} (halo {halo_n} particles): "
          f"load+real {worst[0]:.3f}  S(k) partial {worst[1]:.3f}  "
          f"finalize+forces+self {worst[2]:.3f}  total {sum(worst):.3f} ms", flush=True)
