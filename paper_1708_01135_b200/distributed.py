"""Multi-GPU Ewald evaluation: one process per GPU over torch.distributed.

The reference parallelises with worker threads over contiguous particle
blocks and reduces per-worker copies of rho_hat in worker order
(engine.py:75-91, 247-254); the paper does the same across MPI ranks with a
global reduction of rho_hat.  Here each rank owns:

* reciprocal space: a contiguous particle shard [i0, i1) -- it computes the
  partial S(k) of its shard, the partials are summed by ONE all-reduce
  (NCCL over NVLink; the only data-path collective), and it gathers the
  reciprocal forces of its own shard from the complete S(k);
* real space: a z-slab of the cell grid (``ewb_dev_real_space(part,
  nparts)``); positions are replicated on every rank (the caller hands the
  full configuration, as the reference API does), so no halo exchange is
  needed and the ordered-pair write-to-centre convention (engine.py:10-14)
  means no force communication inside the pair loop;
* the per-rank force contributions and the rank's real-space energy travel
  in ONE all-reduce buffer [F (3N) | u_sr | u_lr | u_self] (u_lr and u_self
  are complete on every rank and enter from rank 0 only), so every rank
  returns the full force array (drop-in semantics).  The step enqueues all
  device work and collectives without a host synchronisation; the single
  synchronisation at the end reads the energies and the deferred device
  error flag (coincident particles, unwrapped positions).
* on CUDA the rank's real-space slab runs on a side stream concurrently with
  the reciprocal chain (S(k) partial, its all-reduce, finalisation); the
  streams join before the reciprocal forces, which add into the same
  buffer.  The stages use disjoint scratch (as in the single-GPU overlap).

``stages`` is the device-stage interface (``DeviceStages`` wraps the C-ABI);
tests inject a CPU stand-in to run this orchestration under ``gloo``.
"""

import torch
import torch.distributed as dist


def shard_range(n, rank, world):
    """Contiguous block of rank (engine.py:75-82 block_bounds)."""
    base, rem = divmod(n, world)
    i0 = rank * base + min(rank, rem)
    return i0, i0 + base + (1 if rank < rem else 0)


class DeviceStages:
    """C-ABI device stages on torch CUDA tensors (product path)."""

    def __init__(self, handle):
        self.h = handle

    def set_stream(self, stream):
        self.h.set_stream(stream.cuda_stream)

    def slot_size(self):
        return self.h.dev_slot_doubles()

    def load(self, pos, q):
        self.h.dev_load(pos.data_ptr(), q.data_ptr(), q.shape[0])

    def real_space(self, part, nparts, force):
        return self.h.dev_real_space(part, nparts, force.data_ptr())

    def real_space_async(self, part, nparts, force):
        self.h.dev_real_space_async(part, nparts, force.data_ptr())

    def finalize_async(self, slots, rho_out=None):
        self.h.dev_kspace_finalize_async(
            slots.data_ptr(), None if rho_out is None else rho_out.data_ptr())

    def self_energy_async(self):
        self.h.dev_self_energy_async()

    def energies(self, out3):
        """device slots (u_sr, u_lr, u_self) -> out3 (device tensor, 3)"""
        self.h.dev_energies(out3.data_ptr())

    def check(self):
        self.h.dev_check()

    def rho_partial(self, i0, i1, slots):
        self.h.dev_rho_partial(i0, i1, slots.data_ptr())

    def finalize(self, slots, rho_out=None):
        return self.h.dev_kspace_finalize(
            slots.data_ptr(), None if rho_out is None else rho_out.data_ptr())

    def recip_forces(self, i0, i1, force):
        self.h.dev_recip_forces(i0, i1, force.data_ptr())

    def self_energy(self):
        return self.h.dev_self_energy()


class ShardedEwald:
    """Particle-sharded Ewald evaluation across the ranks of a group."""

    def __init__(self, stages, device, group=None, overlap=True):
        self.st = stages
        self.device = device
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        self._slots = None
        cuda = torch.device(device).type == "cuda"
        self._side = torch.cuda.Stream(device=device) if overlap and cuda else None
        self._main = torch.cuda.Stream(device=device) if overlap and cuda else None

    def _allreduce(self, t):
        if self.world > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)

    def evaluate(self, pos, q, force, rho_out=None):
        """force (N,3) += Coulomb force on every rank; returns
        (u_sr, u_lr, u_self) -- identical on every rank."""
        if self._side is None:
            return self._evaluate(pos, q, force, rho_out, None)
        # the device stages and the collectives run on an explicit stream
        # (the caller's, unless it is the legacy default stream, which the
        # non-blocking side stream would not order against)
        cur = torch.cuda.current_stream(self.device)
        main = self._main if cur.cuda_stream == 0 else cur
        if main is not cur:
            main.wait_stream(cur)
        with torch.cuda.stream(main):
            self.st.set_stream(main)
            out = self._evaluate(pos, q, force, rho_out, main)
        if main is not cur:
            cur.wait_stream(main)
        return out

    def _evaluate(self, pos, q, force, rho_out, main):
        n = q.shape[0]
        ns = self.st.slot_size()
        if self._slots is None or self._slots.numel() != ns:
            self._slots = torch.empty(ns, dtype=torch.float64, device=self.device)
        i0, i1 = shard_range(n, self.rank, self.world)
        if self.world > 1:
            buf = torch.zeros(3 * n + 3, dtype=torch.float64, device=self.device)
            contrib, en = buf[:3 * n].view(n, 3), buf[3 * n:]
        else:
            contrib, en = force, torch.empty(3, dtype=torch.float64, device=self.device)
        self.st.load(pos, q)
        if main is not None:                   # real space beside the reciprocal chain
            self._side.wait_stream(main)
            self.st.set_stream(self._side)
            self.st.real_space_async(self.rank, self.world, contrib)
            self.st.set_stream(main)
        self.st.rho_partial(i0, i1, self._slots)
        self._allreduce(self._slots)           # S(k) = sum over shards
        self.st.finalize_async(self._slots, rho_out)
        if main is not None:
            main.wait_stream(self._side)       # both add into contrib
        else:
            self.st.real_space_async(self.rank, self.world, contrib)
        self.st.recip_forces(i0, i1, contrib)
        self.st.self_energy_async()
        self.st.energies(en)
        if self.world > 1:
            if self.rank != 0:
                en[1:].zero_()                 # complete on every rank: count once
            self._allreduce(buf)               # forces + energies, one collective
            force += contrib
        self.st.check()
        u_sr, u_lr, u_self = en.tolist()
        return u_sr, u_lr, u_self
