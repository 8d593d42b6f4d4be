"""CPU stand-in for the device stages (TEST INFRASTRUCTURE ONLY).

Implements the stage interface of ``distributed.DeviceStages`` with the
oracle so that the multi-GPU orchestration (``distributed.SlabEwald`` /
``ShardedEwald``: row ownership, halo exchange, S(k) all-reduce, reverse
force exchange, owned-row all-gather) can be exercised under ``gloo`` on
CPU.  The "slot" buffer here is simply the caller-order rho (2K doubles).
Real space is the oracle's write-to-centre evaluation of the given centre
rows over the loaded (own + halo) particles, i.e. a full shell, so the
orchestration fetches the full-stencil halo for it.
"""

import math

import numpy as np
import torch

from oracle import oracle as orc


class OracleStages:
    half_shell = False

    def __init__(self, L, alpha, r_cutoff, m_int):
        self.L, self.alpha, self.rc = float(L), float(alpha), float(r_cutoff)
        self.m = np.ascontiguousarray(m_int, dtype=np.int64)
        self.coeff = orc.kspace_coeff(self.m, self.L, self.alpha)
        self.S = None
        self.cpd = max(1, int(math.floor(self.L / self.rc)))
        self.fold = self.cpd < 3

    def slot_size(self):
        return 2 * self.m.shape[0]

    def set_geometry_n(self, n):
        pass

    def geometry(self):
        c = 1 if self.fold else self.cpd
        return {"cpd": c, "rad": 1, "n_rows": c * c, "fold": int(self.fold)}

    def rows(self, pos):
        p = pos.detach().cpu().numpy()
        if self.fold:
            return torch.zeros(p.shape[0], dtype=torch.int32)
        e = self.L / self.cpd
        cy = np.clip(np.floor(p[:, 1] / e).astype(np.int64), 0, self.cpd - 1)
        cz = np.clip(np.floor(p[:, 2] / e).astype(np.int64), 0, self.cpd - 1)
        return torch.from_numpy((cy + self.cpd * cz).astype(np.int32))

    def row_order(self, pos, n_rows):
        rows = self.rows(pos).numpy()
        order = np.argsort(rows, kind="stable")
        start = np.concatenate([[0], np.cumsum(np.bincount(rows, minlength=n_rows))])
        return torch.from_numpy(order.astype(np.int64)), start.tolist()

    def load(self, pos, q):
        self.pos = pos.detach().cpu().numpy().astype(np.float64)
        self.q = q.detach().cpu().numpy().astype(np.float64)

    def real_space_rows(self, lo, hi, force):
        rows = self.rows(torch.from_numpy(self.pos)).numpy()
        sel = np.nonzero((rows >= lo) & (rows < hi))[0]
        self._u_sr = 0.0
        if sel.size == 0:
            return
        f = np.zeros_like(self.pos)
        u, f = orc.short_range(self.pos, self.q, self.L, self.rc, self.alpha,
                               sel=sel, force=f, threads=1)
        force += torch.from_numpy(f)
        self._u_sr = u

    def rho_partial(self, i0, i1, slots):
        if i1 > i0:
            r = orc.rho_hat(self.pos[i0:i1], self.q[i0:i1], self.L, self.m, threads=1)
        else:
            r = np.zeros(self.slot_size())
        slots.copy_(torch.from_numpy(r))

    def finalize(self, slots, rho_out=None):
        self.S = slots.detach().cpu().numpy().copy()
        K = self.m.shape[0]
        if rho_out is not None:
            rho_out.copy_(torch.from_numpy(self.S))
        self._u_lr = float(np.sum(self.coeff * (self.S[:K] ** 2 + self.S[K:] ** 2)))

    def recip_forces(self, i0, i1, force):
        if i1 <= i0:
            return
        f = np.zeros((i1 - i0, 3))
        orc.long_range(self.pos[i0:i1], self.q[i0:i1], self.L, self.m, self.coeff,
                       self.S, force=f, threads=1)
        force[i0:i1] += torch.from_numpy(f)

    def self_energy_range(self, i0, i1):
        self._u_self = orc.self_energy(self.q[i0:i1], self.alpha) if i1 > i0 else 0.0

    def energies(self, out4):
        out4.copy_(torch.tensor([self._u_sr, self._u_lr, self._u_self, 0.0],
                                dtype=torch.float64))

    def set_stream(self, stream):
        pass
