"""Multi-GPU Ewald evaluation: one process per GPU over torch.distributed.

The paper decomposes the domain over MPI ranks, exchanges halos for the
real-space loop and reduces rho_hat globally; the
reference shards particles over worker threads and reduces per-worker copies
of rho_hat in worker order (engine.py:75-91, 247-254).  Here every rank owns
the particles of a contiguous range of rows of cells (a row is the line of
cells (cy, cz) along x, numbered cy + cpd cz, so a row range is a z-slab with
at most two partial layers; every rank bins on the grid of the global
particle count, ewb_set_geometry_n):

* halo exchange: a rank needs the particles of the rows its centres' stencil
  reaches beyond its own rows -- with the half shell only the rows at
  lexicographically positive (oz, oy) offsets, i.e. the slab above it (two or
  more hops when a slab is thinner than the stencil, e.g. c4 on 8 GPUs).  Each
  rank sends (x, y, z, q) of its particles in every peer's halo rows by
  grouped point-to-point sends/receives (batch_isend_irecv: ncclSend/ncclRecv
  over NVLink); the counts travel first in one all-gather.
* real space: the pair kernel runs over own + halo particles with centres
  restricted to the own rows (ewb_dev_real_space_rows).  The half shell puts
  F_j = -F_i also on halo partners; those forces go back to their owners by
  the reverse exchange, so every pair is evaluated exactly once in the job.
* reciprocal space: each rank's S(k) partial over its own particles (the
  tensor-core GEMM), ONE all-reduce of the partials (the only collective on
  the data path besides the halo exchanges) -- overlapped with the real-space
  pair kernel, which runs on a side stream -- then every rank finalises S(k)
  and gathers the reciprocal forces of its own particles.
* energies: [u_sr, u_lr, u_self, device error flag] in one small all-reduce
  (u_lr counted on rank 0 only); the error flag (coincident particles,
  unwrapped positions) is reduced with them, so every rank raises the same
  exception together and no caller force array is touched.

``SlabEwald.evaluate_local`` is the domain-decomposed interface (each rank
holds only its own particles; halos by point-to-point exchange, as above).
``ShardedEwald`` is the drop-in over the reference API, where every rank
holds the full configuration (``SlabEwald.evaluate_replicated``): a rank
takes its own rows' particles and its halo straight from that configuration
(no point-to-point traffic at all), and the forces of every rank's own + halo
particles come back by ONE all-gather, summed into the full array on every
rank (the halo partners' forces included; no 3N all-reduce).

``stages`` is the device-stage interface (``DeviceStages`` wraps the C-ABI);
the tests inject a CPU stand-in (tests/cpu_stages.py) to run this
orchestration under ``gloo`` without a GPU.
"""

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .core import error


def shard_range(n, rank, world):
    """Contiguous block of rank (engine.py:75-82 block_bounds)."""
    base, rem = divmod(n, world)
    i0 = rank * base + min(rank, rem)
    return i0, i0 + base + (1 if rank < rem else 0)


def row_bounds(n_rows, world):
    """Rows [lo, hi) of every rank: an even split of the rows of cells."""
    return [(n_rows * r // world, n_rows * (r + 1) // world) for r in range(world)]


def halo_rows(lo, hi, cpd, rad, half):
    """Rows outside [lo, hi) that the stencil of the rows [lo, hi) reaches:
    with the half shell only the offsets (oz, oy) > (0, 0) lexicographically
    (the pair kernel's own rule), else the full (2 rad + 1)^2 stencil."""
    if hi <= lo:
        return np.zeros(0, dtype=np.int64)
    r = np.arange(lo, hi)
    cy, cz = r % cpd, r // cpd
    out = []
    for oz in range(-rad, rad + 1):
        for oy in range(-rad, rad + 1):
            if oz == 0 and oy == 0:
                continue
            if half and (oz < 0 or (oz == 0 and oy < 0)):
                continue
            out.append((cy + oy) % cpd + cpd * ((cz + oz) % cpd))
    rows = np.unique(np.concatenate(out))
    return rows[(rows < lo) | (rows >= hi)]


class DeviceStages:
    """C-ABI device stages on torch CUDA tensors (product path)."""

    def __init__(self, handle):
        self.h = handle

    @property
    def half_shell(self):
        return not getattr(self.h, "deterministic", False)

    def set_stream(self, stream):
        if stream is None:
            self.h.use_own_stream()
        else:
            self.h.set_stream(stream.cuda_stream)

    def slot_size(self):
        return self.h.dev_slot_doubles()

    def set_geometry_n(self, n):
        self.h.set_geometry_n(n)

    def geometry(self):
        return self.h.rs_geometry()

    def rows(self, pos):
        """Row of cells of every particle, on torch's current stream (the
        result is consumed by torch operations)."""
        self.h.set_stream(torch.cuda.current_stream(pos.device).cuda_stream)
        out = torch.empty(pos.shape[0], dtype=torch.int32, device=pos.device)
        self.h.dev_rows(pos.data_ptr(), pos.shape[0], out.data_ptr())
        return out

    def row_order(self, pos, n_rows):
        """(particle indices grouped by row of cells, ascending within a row;
        row offsets as a host list) -- one host synchronisation."""
        self.h.set_stream(torch.cuda.current_stream(pos.device).cuda_stream)
        n = pos.shape[0]
        order = torch.empty(n, dtype=torch.int32, device=pos.device)
        start = torch.empty(n_rows + 1, dtype=torch.int32, device=pos.device)
        self.h.dev_row_order(pos.data_ptr(), n, order.data_ptr(), start.data_ptr())
        return order.long(), start.tolist()

    def load(self, pos, q):
        self.h.dev_load(pos.data_ptr(), q.data_ptr(), q.shape[0])

    def real_space_rows(self, lo, hi, force):
        self.h.dev_real_space_rows_async(lo, hi, force.data_ptr())

    def rho_partial(self, i0, i1, slots):
        self.h.dev_rho_partial(i0, i1, slots if isinstance(slots, int) else slots.data_ptr())

    def ipc_slots(self):
        return self.h.ipc_slots()

    def ipc_open(self, handle64):
        return self.h.ipc_open(handle64)

    def finalize(self, slots, rho_out=None):
        self.h.dev_kspace_finalize_async(
            slots.data_ptr(), None if rho_out is None else rho_out.data_ptr())

    def finalize_peer(self, slot_ptrs, rho_out=None):
        """S(k) = sum of the ranks' partial slots read from peer memory, and
        its finalisation, in one kernel (ewb_dev_kspace_finalize_peer)."""
        self.h.dev_kspace_finalize_peer(slot_ptrs,
                                        None if rho_out is None else rho_out.data_ptr())

    def recip_forces(self, i0, i1, force):
        self.h.dev_recip_forces(i0, i1, force.data_ptr())

    def self_energy_range(self, i0, i1):
        self.h.dev_self_energy_range_async(i0, i1)

    def energies(self, out4):
        """device slots (u_sr, u_lr, u_self) and the error flag -> out4"""
        self.h.dev_energies(out4.data_ptr())
        self.h.dev_status(out4[3:].data_ptr())


class _Comm:
    """Collectives of one process group; gloo stages through host memory."""

    def __init__(self, group, device):
        self.group = group
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.world = dist.get_world_size(group) if dist.is_initialized() else 1
        backend = dist.get_backend(group) if dist.is_initialized() else "none"
        self.host = backend != "nccl"
        self.dev = torch.device("cpu") if self.host else torch.device(device)

    def _to(self, t):
        return t.to(self.dev) if t.device != self.dev else t

    # ---- S(k) reduction fused into the finalisation over CUDA IPC (opt-in:
    # EWALDB200_PEER_FINALIZE=1).  The ranks export their partial buffers once;
    # per step two host barriers bracket the kernel that reads every rank's
    # partial over NVLink (instead of one asynchronous NCCL all-reduce).
    def fused(self, st):
        import os
        return (self.world > 1 and hasattr(st, "ipc_slots") and hasattr(st, "finalize_peer")
                and os.environ.get("EWALDB200_PEER_FINALIZE", "0") == "1")

    def slot_ptr(self, st):
        ptr, handle = st.ipc_slots()
        if getattr(self, "_ipc_mine", None) != ptr:
            mine = torch.frombuffer(bytearray(handle), dtype=torch.uint8)
            allh = [torch.empty(64, dtype=torch.uint8) for _ in range(self.world)]
            if self.host:
                dist.all_gather(allh, mine, group=self.group)
            else:
                dev_h = [a.to(self.dev) for a in allh]
                dist.all_gather(dev_h, mine.to(self.dev), group=self.group)
                allh = [a.cpu() for a in dev_h]
            self._ipc_ptrs = [ptr if r == self.rank else st.ipc_open(bytes(allh[r].tolist()))
                              for r in range(self.world)]
            self._ipc_mine = ptr
        return ptr

    def peer_finalize(self, st, ptr, rho_out):
        torch.cuda.current_stream().synchronize()   # my partial is complete
        dist.barrier(group=self.group)               # ... and every rank's
        st.finalize_peer(self._ipc_ptrs, rho_out)
        torch.cuda.current_stream().synchronize()
        dist.barrier(group=self.group)               # peers done reading mine

    def allreduce_(self, t):
        if self.world == 1:
            return t
        x = self._to(t)
        dist.all_reduce(x, op=dist.ReduceOp.SUM, group=self.group)
        if x is not t:
            t.copy_(x)
        return t

    def counts(self, c):
        """c[p] = rows this rank sends to peer p -> M[src][dst] of all ranks."""
        if self.world == 1:
            return np.array([c])
        mine = self._to(torch.tensor(c, dtype=torch.int64))
        allc = [torch.empty_like(mine) for _ in range(self.world)]
        dist.all_gather(allc, mine, group=self.group)
        return np.stack([a.cpu().numpy() for a in allc])

    def exchange(self, send, recv_counts, width, dtype, device):
        """Grouped point-to-point: send[p] (rows, width) to peer p, receive
        recv_counts[p] rows from p.  Returns the received blocks by peer."""
        ops, recv = [], [None] * self.world
        bufs = {}
        for p in range(self.world):
            if p == self.rank:
                continue
            if recv_counts[p] > 0:
                bufs[p] = torch.empty((int(recv_counts[p]), width), dtype=dtype, device=self.dev)
                ops.append(dist.P2POp(dist.irecv, bufs[p], p, self.group))
            if send[p] is not None and send[p].shape[0] > 0:
                ops.append(dist.P2POp(dist.isend, self._to(send[p]).contiguous(), p, self.group))
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()
        for p, b in bufs.items():
            recv[p] = b.to(device) if b.device != torch.device(device) else b
        return recv

    def all_gather_rows(self, t, counts, width, need=True):
        """Every rank's t (counts[r] rows) -> list of blocks by rank (need:
        whether this rank uses them; NCCL receives them either way)."""
        if self.world == 1:
            return [t]
        m = int(max(counts))
        pad = torch.zeros((m, width), dtype=t.dtype, device=self.dev)
        pad[:t.shape[0]] = self._to(t)
        out = [torch.empty_like(pad) for _ in range(self.world)]
        dist.all_gather(out, pad, group=self.group)
        return [o[:int(c)].to(t.device) for o, c in zip(out, counts)]


class ThreadGroup:
    """W ranks driven by W host threads of ONE process (one GPU each): the
    multi-GPU path behind the reference API's ``workers`` argument, where a
    single caller thread owns the particle arrays (engine.py:256-277 fans the
    same call out to worker threads).  Collectives meet at a barrier; device
    tensors are posted after their producing stream has drained and read by
    peer copies (NVLink), summed in rank order so every rank gets bitwise the
    same result."""

    def __init__(self, world, timeout=600.0):
        import threading
        self.world = int(world)
        self.barrier = threading.Barrier(self.world, timeout=timeout)
        self.slots = [None] * self.world

    def abort(self):
        self.barrier.abort()


class ThreadComm:
    """The _Comm interface over a ThreadGroup (rank = this thread's index)."""

    host = False

    def __init__(self, group, rank, device):
        self.g = group
        self.rank, self.world = int(rank), group.world
        self.dev = torch.device(device)

    def _sync(self):
        if self.dev.type == "cuda":
            torch.cuda.current_stream(self.dev).synchronize()

    def _post(self, obj):
        """Publish obj, wait for every rank's, return all of them."""
        self._sync()
        self.g.slots[self.rank] = obj
        self.g.barrier.wait()
        return list(self.g.slots)

    def _done(self):
        self._sync()                      # peer reads finished before reuse
        self.g.barrier.wait()

    def allreduce_(self, t):
        if self.world == 1:
            return t
        allv = self._post(t)
        acc = allv[0].to(t.device, copy=True)
        for r in range(1, self.world):
            acc += allv[r].to(t.device)
        self._done()
        t.copy_(acc)
        return t

    def counts(self, c):
        allc = self._post(list(c))
        self._done()
        return np.array(allc)

    def exchange(self, send, recv_counts, width, dtype, device):
        allv = self._post(send)
        recv = [None] * self.world
        for p in range(self.world):
            if p != self.rank and recv_counts[p] > 0:
                recv[p] = allv[p][self.rank].to(device)
        self._done()
        return recv

    def all_gather_rows(self, t, counts, width, need=True):
        allv = self._post(t)
        out = [a.to(t.device) for a in allv] if need else []
        self._done()
        return out

    def fused(self, st):
        return hasattr(st, "finalize_peer")

    def slot_ptr(self, st):
        return None                               # the rank's own slot tensor

    def peer_finalize(self, st, ptr, rho_out):
        """The S(k) all-reduce fused into the finalisation: once every
        rank's partial is complete, each rank's kernel reads all of them
        through peer pointers (NVLink); the closing barrier keeps the
        buffers alive until every rank's kernel is done."""
        allv = self._post(ptr)
        st.finalize_peer(list(allv), rho_out)
        self._done()


def _raise_device_error(flag):
    flag = int(flag)
    if flag & _lib.ERR_UNWRAPPED:
        raise ValueError("positions must be wrapped into [0, L) before binning")
    if flag & _lib.ERR_COINCIDENT:
        raise error("CoincidentParticlesError", "coincident particles in Coulomb kernel")


class SlabEwald:
    """Domain-decomposed Ewald evaluation: each rank owns the particles of
    its rows of cells (see the module docstring)."""

    def __init__(self, stages, device, n_global, group=None, overlap=True, comm=None):
        self.st = stages
        self.device = torch.device(device)
        self.comm = _Comm(group, device) if comm is None else comm
        self.rank, self.world = self.comm.rank, self.comm.world
        self.n_global = int(n_global)
        stages.set_geometry_n(self.n_global)
        g = stages.geometry()
        self.cpd, self.rad, self.n_rows, self.fold = g["cpd"], g["rad"], g["n_rows"], g["fold"]
        self.bounds = row_bounds(self.n_rows, self.world)
        self.lo, self.hi = self.bounds[self.rank]
        half = stages.half_shell
        need = np.zeros((self.world, self.n_rows), dtype=bool)
        for s, (lo, hi) in enumerate(self.bounds):
            if self.fold:        # one row: its owner scans everything
                continue
            need[s, halo_rows(lo, hi, self.cpd, self.rad, half)] = True
        self.need = torch.from_numpy(need).to(self.device)
        # each rank's halo rows as runs [a, b) of consecutive rows
        self._halo_runs = []
        for r in range(self.world):
            rr = np.nonzero(need[r])[0]
            runs = []
            for v in rr.tolist():
                if runs and runs[-1][1] == v:
                    runs[-1][1] = v + 1
                else:
                    runs.append([v, v + 1])
            self._halo_runs.append([tuple(x) for x in runs])
        self._slots = None
        cuda = self.device.type == "cuda"
        self._main = torch.cuda.Stream(device=self.device) if cuda else None
        self._side = torch.cuda.Stream(device=self.device) if cuda and overlap else None

    def owned_mask(self, rows, rank=None):
        lo, hi = self.bounds[self.rank if rank is None else rank]
        return (rows >= lo) & (rows < hi)

    def evaluate_local(self, pos, q, force, rho_out=None):
        """pos (n_own, 3), q (n_own,): this rank's particles (all in its rows);
        force (n_own, 3) += their Coulomb force.  Returns the job's
        (u_sr, u_lr, u_self), identical on every rank."""
        if self._main is None:
            return self._evaluate(pos, q, force, rho_out)
        cur = torch.cuda.current_stream(self.device)
        self._main.wait_stream(cur)
        try:
            with torch.cuda.stream(self._main):
                self.st.set_stream(self._main)
                out = self._evaluate(pos, q, force, rho_out)
        finally:
            self.st.set_stream(None)       # back to the handle's own stream
            cur.wait_stream(self._main)
        return out

    def _compute(self, lpos, lq, n_own, rho_out):
        """The rank's device work on its loaded particles (own first, then
        halo): real space of its rows on the side stream, S(k) partial + the
        all-reduce, finalisation, reciprocal forces and self energy of the own
        particles.  Returns (forces of own + halo particles, energies [u_sr,
        u_lr (rank 0 only), u_self, device error flag]) before the energy
        all-reduce."""
        st, comm, dev = self.st, self.comm, self.device
        n_loc = lq.shape[0]
        flocal = torch.zeros((n_loc, 3), dtype=torch.float64, device=dev)
        ns = st.slot_size()
        if self._slots is None or self._slots.numel() != ns:
            self._slots = torch.empty(ns, dtype=torch.float64, device=dev)
        en = torch.zeros(4, dtype=torch.float64, device=dev)
        st.load(lpos, lq)
        # ---- real space of my rows beside the reciprocal chain
        if self._side is not None:
            self._side.wait_stream(self._main)
            st.set_stream(self._side)
            st.real_space_rows(self.lo, self.hi, flocal)
            st.set_stream(self._main)
        else:
            st.real_space_rows(self.lo, self.hi, flocal)
        if comm.fused(st):
            # every rank's finalising kernel sums the partials from peer memory
            ptr = comm.slot_ptr(st)
            if ptr is None:
                ptr = self._slots.data_ptr()
            st.rho_partial(0, n_own, ptr)
            comm.peer_finalize(st, ptr, rho_out)
        else:
            st.rho_partial(0, n_own, self._slots)
            comm.allreduce_(self._slots)      # S(k) = sum of the ranks' partials
            st.finalize(self._slots, rho_out)
        if self._side is not None:
            # the reciprocal forces into their own buffer, so the force GEMM
            # runs while the pair kernel is still busy on the side stream
            frec = torch.zeros((n_own, 3), dtype=torch.float64, device=dev)
            st.recip_forces(0, n_own, frec)
            st.self_energy_range(0, n_own)
            self._main.wait_stream(self._side)
            flocal[:n_own] += frec
        else:
            st.recip_forces(0, n_own, flocal)
            st.self_energy_range(0, n_own)
        st.energies(en)
        if self.rank != 0:
            en[1] = 0.0                        # u_lr is complete on every rank
        return flocal, en

    def evaluate_replicated(self, pos, q, force, rho_out=None, apply=True):
        """Every rank holds the FULL configuration (the reference API): it
        takes its own rows' particles and its halo straight from it (no
        point-to-point exchange), and the forces of every rank's own + halo
        particles return by ONE all-gather, summed into the full array on
        every rank (halo partner forces included).  Two host
        synchronisations size the per-rank lists; the collectives are the
        S(k) all-reduce, the 4-double energy all-reduce and the all-gather."""
        if self._main is None:
            return self._replicated(pos, q, force, rho_out, apply)
        cur = torch.cuda.current_stream(self.device)
        self._main.wait_stream(cur)
        try:
            with torch.cuda.stream(self._main):
                self.st.set_stream(self._main)
                out = self._replicated(pos, q, force, rho_out, apply)
        finally:
            self.st.set_stream(None)
            cur.wait_stream(self._main)
        return out

    def _replicated(self, pos, q, force, rho_out, apply=True):
        st, comm, W = self.st, self.comm, self.world
        # particles grouped by row (one stable sort, one synchronisation):
        # every rank's own rows and halo rows are slices of `order`
        order, rstart = st.row_order(pos, self.n_rows)
        lists, sizes, n_owns = [], [], []
        for r, (lo, hi) in enumerate(self.bounds):
            sl = [order[rstart[lo]:rstart[hi]]]
            for a, b in self._halo_runs[r]:
                sl.append(order[rstart[a]:rstart[b]])
            lists.append(sl)
            n_owns.append(rstart[hi] - rstart[lo])
            sizes.append(sum(int(rstart[b] - rstart[a]) for a, b in self._halo_runs[r]) + n_owns[-1])
        mine = lists[self.rank]
        lidx = torch.cat(mine) if len(mine) > 1 else mine[0]
        flocal, en = self._compute(pos[lidx].contiguous(), q[lidx].contiguous(),
                                   n_owns[self.rank], rho_out)
        comm.allreduce_(en)                    # energies + error flags of all ranks
        u_sr, u_lr, u_self, err = en.tolist()
        if err:
            _raise_device_error(err)           # every rank, before any force is written
        blocks = comm.all_gather_rows(flocal, sizes, 3, need=apply)
        if not apply:                          # another rank writes the caller's forces
            return u_sr, u_lr, u_self
        idx = torch.cat([t for sl in lists for t in sl])
        force.index_add_(0, idx.to(force.device),
                         torch.cat(blocks).to(force.device) if len(blocks) > 1 else blocks[0])
        return u_sr, u_lr, u_self

    def _evaluate(self, pos, q, force, rho_out):
        st, comm, dev = self.st, self.comm, self.device
        n_own = q.shape[0]
        rows = st.rows(pos).long()
        # ---- halo exchange: (x, y, z, q) of my particles in every peer's halo
        # (one nonzero over all peers: its (peer, particle) pairs come out
        # peer-major, one host synchronisation for the whole selection)
        need = self.need[:, rows]
        need[self.rank] = False
        nz = torch.nonzero(need)
        cnt = torch.bincount(nz[:, 0], minlength=self.world).tolist() if nz.numel() else \
            [0] * self.world
        send_idx, send = [None] * self.world, [None] * self.world
        off = 0
        xq = torch.cat([pos, q[:, None]], dim=1)
        for p in range(self.world):
            if p != self.rank:
                send_idx[p] = nz[off:off + cnt[p], 1]
                send[p] = xq[send_idx[p]]
            off += cnt[p]
        M = comm.counts(cnt)
        recv_counts = M[:, self.rank]
        recv = comm.exchange(send, recv_counts, 4, torch.float64, dev)
        halo = [r for r in recv if r is not None]
        if halo:
            h = torch.cat(halo)
            lpos = torch.cat([pos, h[:, :3]]).contiguous()
            lq = torch.cat([q, h[:, 3]]).contiguous()
        else:
            lpos, lq = pos.contiguous(), q.contiguous()
        flocal, en = self._compute(lpos, lq, n_own, rho_out)
        # ---- reverse exchange: halo partners' forces back to their owners
        back = [None] * self.world
        off = n_own
        for p in range(self.world):
            c = int(recv_counts[p]) if p != self.rank else 0
            if c:
                back[p] = flocal[off:off + c]
                off += c
        got = comm.exchange(back, cnt, 3, torch.float64, dev)
        comm.allreduce_(en)                    # energies + error flags of all ranks
        u_sr, u_lr, u_self, err = en.tolist()
        if err:
            _raise_device_error(err)
        force += flocal[:n_own]
        for p in range(self.world):
            if got[p] is not None and got[p].shape[0]:
                force.index_add_(0, send_idx[p], got[p])
        return u_sr, u_lr, u_self


class ShardedEwald:
    """Drop-in multi-GPU evaluation over the reference API: every rank holds
    the full configuration and returns the full force array."""

    def __init__(self, stages, device, group=None, overlap=True):
        self.st = stages
        self.device = torch.device(device)
        self.group = group
        self.overlap = overlap
        self.slab = None

    def evaluate(self, pos, q, force, rho_out=None):
        """force (N,3) += Coulomb force on every rank; returns
        (u_sr, u_lr, u_self) -- identical on every rank."""
        n = q.shape[0]
        if self.slab is None or self.slab.n_global != n:
            self.slab = SlabEwald(self.st, self.device, n, self.group, self.overlap)
        return self.slab.evaluate_replicated(pos, q, force, rho_out=rho_out)


def _resolve_devices(workers):
    """The reference's ``workers`` read as a GPU count: None ->
    $EWALDB200_WORKERS or 1, 0 -> every visible GPU, W -> min(W, visible GPUs)
    ranks on devices 0..W-1 (a reference caller may pass its CPU thread count).
    With $EWALDB200_SHARE_DEVICES=1 all W ranks run, round-robin over the
    visible GPUs: ranks sharing a device stay correct (no kernel of one rank
    waits on another's; the collectives meet on the host) -- the multi-rank
    tests on a one-GPU box use this."""
    import os
    if workers is None:
        workers = int(os.environ.get("EWALDB200_WORKERS", "1"))
    n_dev = torch.cuda.device_count() if torch.cuda.is_available() else 0
    workers = int(workers)
    if workers == 0:
        workers = max(n_dev, 1)
    if workers < 1:
        raise ValueError(f"workers must be >= 0, got {workers}")
    if n_dev == 0:
        raise _lib.DeviceError("no CUDA device visible (this package has no CPU path)")
    if os.environ.get("EWALDB200_SHARE_DEVICES", "0") != "1":
        workers = min(workers, n_dev)
    return [r % n_dev for r in range(workers)]


class MultiDeviceEwald:
    """``EwaldSolver(box, params, workers=W)`` with W > 1: W GPUs driven by W
    host threads of the caller's process, each rank a SlabEwald over its rows
    of cells with a ThreadGroup for the collectives.  Every rank reads the
    caller's full configuration (the reference API hands it over whole) and
    takes its own rows and its halo from it (evaluate_replicated: S(k)
    all-reduce, one all-gather of own + halo forces, summed by rank 0 into
    the caller's array)."""

    def __init__(self, L, alpha, r_cutoff, m_int, coeff, devices, overlap=True):
        from concurrent.futures import ThreadPoolExecutor
        self.devices = [torch.device("cuda", int(d)) for d in devices]
        self.world = len(self.devices)
        self.overlap = overlap
        self.n_stored = int(np.asarray(m_int).shape[0])
        self.pool = ThreadPoolExecutor(self.world, thread_name_prefix="ewb-rank")

        def make(r):
            torch.cuda.set_device(self.devices[r])
            h = _lib.Handle(self.devices[r].index)
            h.set_system(L, alpha, r_cutoff)
            h.set_kspace(m_int, coeff)
            return h
        self.handles = list(self.pool.map(make, range(self.world)))
        # peer access between the ranks' GPUs: the fused S(k) reduction reads
        # the other ranks' partials over NVLink
        for r, h in enumerate(self.handles):
            for d in {dv.index for dv in self.devices}:
                h.enable_peer_access(d)
        self.stages = [DeviceStages(h) for h in self.handles]
        self.slabs = [None] * self.world

    def close(self):
        self.pool.shutdown(wait=True)

    def _rank(self, r, grp, pos, q, want_rho):
        dev = self.devices[r]
        torch.cuda.set_device(dev)
        try:
            st, n = self.stages[r], q.shape[0]
            comm = ThreadComm(grp, r, dev)
            sl = self.slabs[r]
            if sl is None or sl.n_global != n:
                sl = self.slabs[r] = SlabEwald(st, dev, n, overlap=self.overlap, comm=comm)
            sl.comm = comm
            tp = torch.from_numpy(pos).to(dev)
            tq = torch.from_numpy(q).to(dev)
            # rank 0 sums every rank's own + halo forces (one all-gather)
            f = torch.zeros((n, 3), dtype=torch.float64, device=dev) if r == 0 else None
            rho = (torch.empty(2 * self.n_stored, dtype=torch.float64, device=dev)
                   if want_rho else None)
            u = sl.evaluate_replicated(tp, tq, f, rho_out=rho, apply=r == 0)
            return (u, None if f is None else f.cpu().numpy(),
                    None if rho is None else rho.cpu().numpy())
        except BaseException:
            grp.abort()                    # release peers waiting at a barrier
            raise

    def evaluate(self, pos, q, force, rho_out=None):
        """Host arrays: pos (N,3), q (N,) -> force (N,3) += on the caller's
        array, rho_out (2K,) overwritten if given; returns (u_sr, u_lr,
        u_self).  All ranks raise the same device error together, before
        any caller array is written."""
        grp = ThreadGroup(self.world)
        futs = [self.pool.submit(self._rank, r, grp, pos, q, rho_out is not None and r == 0)
                for r in range(self.world)]
        errs, res = [], []
        for f in futs:
            try:
                res.append(f.result())
            except BaseException as e:       # noqa: BLE001 -- re-raised below
                errs.append(e)
        if errs:
            import threading
            real = [e for e in errs if not isinstance(e, threading.BrokenBarrierError)]
            raise (real or errs)[0]
        force += res[0][1]
        if rho_out is not None:
            rho_out[:] = res[0][2]
        return res[0][0]
