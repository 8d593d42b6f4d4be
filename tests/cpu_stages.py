"""CPU stand-in for the device stages (TEST INFRASTRUCTURE ONLY).

Implements the stage interface of ``distributed.DeviceStages`` with the
oracle so that ``distributed.ShardedEwald`` -- the multi-GPU orchestration
(particle shards, S(k) all-reduce, real-space z-slabs, force all-reduce) --
can be exercised under ``gloo`` on CPU.  The "slot" buffer here is simply the
caller-order rho (2K doubles); the orchestration treats it as opaque.
"""

import math

import numpy as np
import torch

from oracle import oracle as orc


class OracleStages:
    def __init__(self, L, alpha, r_cutoff, m_int):
        self.L, self.alpha, self.rc = float(L), float(alpha), float(r_cutoff)
        self.m = np.ascontiguousarray(m_int, dtype=np.int64)
        self.coeff = orc.kspace_coeff(self.m, self.L, self.alpha)
        self.S = None

    def slot_size(self):
        return 2 * self.m.shape[0]

    def load(self, pos, q):
        self.pos = pos.detach().cpu().numpy().astype(np.float64)
        self.q = q.detach().cpu().numpy().astype(np.float64)

    def real_space(self, part, nparts, force):
        cpd = int(math.floor(self.L / self.rc))
        cz = np.clip(np.floor(self.pos[:, 2] / (self.L / cpd)).astype(np.int64), 0, cpd - 1)
        zl, zh = cpd * part // nparts, cpd * (part + 1) // nparts
        sel = np.nonzero((cz >= zl) & (cz < zh))[0]
        f = np.zeros_like(self.pos)
        if sel.size == 0:
            return 0.0
        u, f = orc.short_range(self.pos, self.q, self.L, self.rc, self.alpha,
                               sel=sel, force=f, threads=1)
        force += torch.from_numpy(f)
        return u

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
        return float(np.sum(self.coeff * (self.S[:K] ** 2 + self.S[K:] ** 2)))

    def recip_forces(self, i0, i1, force):
        if i1 <= i0:
            return
        f = np.zeros((i1 - i0, 3))
        orc.long_range(self.pos[i0:i1], self.q[i0:i1], self.L, self.m, self.coeff,
                       self.S, force=f, threads=1)
        force[i0:i1] += torch.from_numpy(f)

    def self_energy(self):
        return orc.self_energy(self.q, self.alpha)

    # asynchronous interface (energies kept until energies())
    def real_space_async(self, part, nparts, force):
        self._u_sr = self.real_space(part, nparts, force)

    def finalize_async(self, slots, rho_out=None):
        self._u_lr = self.finalize(slots, rho_out)

    def self_energy_async(self):
        self._u_self = self.self_energy()

    def energies(self, out3):
        out3.copy_(torch.tensor([self._u_sr, self._u_lr, self._u_self], dtype=torch.float64))

    def check(self):
        pass
