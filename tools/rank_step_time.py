"""Per-rank device time of the multi-GPU step, simulated on one GPU: the
stages of distributed.ShardedEwald for rank 0 of W (particle shard 0 of W
for S(k) and forces, real-space part 0 of W, the full-K finalisation),
without the collectives.  Prints ms per stage group and the total
(CUDA events around the stage calls, min of 20)."""
import sys
sys.path.insert(0, '.')
import torch
import paper_1708_01135_b200 as ew
from paper_1708_01135_b200 import _lib
from paper_1708_01135_b200 import workloads as wl
from paper_1708_01135_b200.distributed import shard_range
dev = torch.device('cuda', 0)
name = sys.argv[1] if len(sys.argv) > 1 else 'c2'
cfg = wl.make_config(name)
p = ew.EwaldParams(cfg['alpha_ref'], cfg['r_cutoff'], wl.k_cutoff_for(cfg), 1e-6)
rs = ew.ReciprocalSpace(cfg['box'], p, cfg['m_int'])
pos = torch.from_numpy(cfg['pos']).to(dev)
q = torch.from_numpy(cfg['q']).to(dev)
n = q.shape[0]
st = torch.cuda.Stream()
h = _lib.Handle(0)
h.set_stream(st.cuda_stream)
h.set_system(cfg['L'], p.alpha, p.r_cutoff)
h.set_kspace(rs.m_int, rs.coeff)
f = torch.zeros((n, 3), dtype=torch.float64, device=dev)
slots = torch.empty(h.dev_slot_doubles(), dtype=torch.float64, device=dev)
for W in (1, 2, 4, 8):
    i0, i1 = shard_range(n, 0, W)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    best = None
    with torch.cuda.stream(st):
        for _ in range(20):
            torch.cuda.synchronize()
            ev[0].record(st)
            h.dev_load(pos.data_ptr(), q.data_ptr(), n)
            h.dev_real_space_async(0, W, f.data_ptr())
            ev[1].record(st)
            h.dev_rho_partial(i0, i1, slots.data_ptr())
            ev[2].record(st)
            h.dev_kspace_finalize_async(slots.data_ptr())
            h.dev_recip_forces(i0, i1, f.data_ptr())
            h.dev_self_energy_async()
            ev[3].record(st)
            h.dev_check()
            t = [ev[k].elapsed_time(ev[k + 1]) for k in range(3)]
            if best is None or sum(t) < sum(best):
                best = t
    print(f"{name} W={W}: load+real {best[0]:.3f}  S(k) partial {best[1]:.3f}  "
          f"finalize+forces+self {best[2]:.3f}  total {sum(best):.3f} ms", flush=True)
