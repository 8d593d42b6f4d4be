"""Device-resident MD step around the Ewald path.

Mirrors the reference driver's force assembly and NVE integrator
(``/root/reference/pkg/src/ewaldmd/driver.py`` and ``potentials.py``):

* ``LJParams``, ``lj_pair_energy``, ``lj_pair_force``, ``wca_cutoff``
  (potentials.py:21-30, 88-102) -- host scalar maths;
* ``SimConfig`` (driver.py:18-40), ``rocksalt_cells_for`` / ``init_rocksalt``
  (:43-78), ``initial_velocities`` (:193-201), ``kinetic_energy``
  (:129-131), ``RunMetrics`` (:156-190);
* ``ForceAssembler`` (:81-126): zero forces, Ewald on the device, and the
  energy-shifted 12-6 LJ term FUSED into the real-space pair kernel (one
  traversal at max(r_c, r_c,LJ), each term with its own exact cutoff
  predicate) instead of a second pair loop with its own cell list;
* ``velocity_verlet_step`` (:134-153) on host arrays (reference semantics:
  any force assembler, the kick/drift/wrap done by device kernels);
* ``DeviceMD`` / ``run`` (:204-246): positions, velocities, masses and
  forces stay in HBM across steps; per step only the two energy scalars
  (and the maximum displacement) come back to the host.

All arithmetic runs in ``libewaldb200.so``; torch is used only to own device
memory.  The integrator kernels evaluate exactly the reference's expressions
(``v += 0.5*dt*F*inv_m``, ``r += dt*v``, wrap) without FMA contraction.
"""

import ctypes
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .core import SimulationBox, error, create_particle_set, require_neutral
from .ewald import EwaldSolver, choose_parameters

DEFAULT_SIGMA = 2.5
DEFAULT_EPSILON = 1.0
BENCH_SPACING = 2.5


@dataclass(frozen=True)
class LJParams:
    """Shifted 12-6 parameters (potentials.py:21-30)."""

    epsilon_lj: float = DEFAULT_EPSILON
    sigma: float = DEFAULT_SIGMA
    r_cutoff_lj: float = 2.5 * DEFAULT_SIGMA

    def energy_shift(self):
        s6 = (self.sigma / self.r_cutoff_lj) ** 6
        return 4.0 * self.epsilon_lj * (s6 * s6 - s6)

    def consts(self):
        """The reference kernel constants (potentials.py:74-79)."""
        return (self.sigma**2, 4.0 * self.epsilon_lj, self.energy_shift(),
                24.0 * self.epsilon_lj)


def lj_pair_energy(r, params):
    s6 = (params.sigma / r) ** 6
    return 4.0 * params.epsilon_lj * (s6 * s6 - s6) - params.energy_shift()


def lj_pair_force(r, params):
    s6 = (params.sigma / r) ** 6
    return 24.0 * params.epsilon_lj * (2.0 * s6 * s6 - s6) / r


def wca_cutoff(sigma=DEFAULT_SIGMA):
    return 2.0 ** (1.0 / 6.0) * sigma


@dataclass
class SimConfig:
    n_particles: int = 1728
    box_edge: float = 30.0
    tolerance: float = 1e-6
    alpha: float | None = None
    r_cutoff: float | None = None
    dt: float = 0.005
    n_steps: int = 10
    velocity_scale: float = 0.0
    threads: int = 1
    seed: int = 0
    coulomb_on: bool = True
    lj_on: bool = True
    lj: LJParams = field(default_factory=LJParams)

    def __post_init__(self):
        if self.n_steps < 0:
            raise ValueError(f"n_steps must be >= 0, got {self.n_steps}")
        if self.dt <= 0.0:
            raise ValueError(f"dt must be positive, got {self.dt}")


def rocksalt_cells_for(n):
    c = round((n ** (1.0 / 3.0)) / 2.0)
    if c < 1 or (2 * c) ** 3 != n:
        raise error(
            "LatticeError",
            f"N = {n} is not (2c)^3 for integer c; no alternating rock-salt "
            f"lattice closes at this count")
    return c


def init_rocksalt(cells_per_dim, spacing):
    """Alternating +-1 charges on a simple cubic lattice (driver.py:54-78)."""
    cells_per_dim = int(cells_per_dim)
    if cells_per_dim < 1:
        raise error("LatticeError", f"cells_per_dim must be >= 1, got {cells_per_dim}")
    side = 2 * cells_per_dim
    ps = create_particle_set(side**3, SimulationBox(side * spacing))
    idx = np.arange(side)
    ix, iy, iz = np.meshgrid(idx, idx, idx, indexing="ij")
    ps.position[:, 0] = ix.ravel() * spacing
    ps.position[:, 1] = iy.ravel() * spacing
    ps.position[:, 2] = iz.ravel() * spacing
    ps.charge[:] = np.where((ix + iy + iz).ravel() % 2 == 0, 1.0, -1.0)
    return ps


def initial_velocities(ps, scale, seed):
    if scale <= 0.0:
        ps.velocity[:] = 0.0
        return
    rng = np.random.default_rng(seed)
    ps.velocity[:] = scale * rng.standard_normal((ps.count, 3))
    ps.velocity -= (ps.mass @ ps.velocity) / ps.mass.sum()


def kinetic_energy(ps):
    return 0.5 * float(ps.mass @ np.einsum("ij,ij->i", ps.velocity, ps.velocity))


def _device_handle_for(box, config, params):
    """A handle configured with the Coulomb and LJ switches of config."""
    if config.coulomb_on:
        solver = EwaldSolver(box, params, workers=config.threads)
        h = solver.handle
    else:
        solver = None
        h = _lib.Handle()
        h.set_system(box.edge_length, 1.0, config.lj.r_cutoff_lj)
        h.set_coulomb(False)
    if config.lj_on:
        s2, e4, shift, e24 = config.lj.consts()
        h.set_lj(True, s2, e4, shift, e24, config.lj.r_cutoff_lj)
    return solver, h


class ForceAssembler:
    """Zero forces, then Coulomb (Ewald) and LJ in one device evaluation.

    Same construction and call contract as the reference (driver.py:81-126);
    ``last`` carries u_coulomb, u_lj and the component times.  The LJ term
    is fused into the real-space kernel, so its time is part of t_sr and
    t_lj is reported as 0.
    """

    def __init__(self, ps, config):
        self.config = config
        self.box = ps.box
        self.params = None
        if config.coulomb_on:
            self.params = choose_parameters(
                ps.count, ps.box, config.tolerance, alpha=config.alpha,
                r_cutoff=config.r_cutoff)
        if not (config.coulomb_on or config.lj_on):
            self.solver, self.handle = None, None
        else:
            self.solver, self.handle = _device_handle_for(ps.box, config, self.params)
        self.last = None

    def __call__(self, ps):
        ps.force[:] = 0.0
        u_c, u_lj = 0.0, 0.0
        t = {"t_sr": 0.0, "t_alg1": 0.0, "t_alg2": 0.0, "t_lj": 0.0}
        if self.solver is not None:
            res = self.solver.evaluate(ps)
            u_c = res.total
            t.update(t_sr=res.t_sr, t_alg1=res.t_alg1, t_alg2=res.t_alg2)
            if self.config.lj_on:
                u_lj = float(self.handle.last_energies()[3])
        elif self.handle is not None:
            pos = _lib.f64c(ps.position, (ps.count, 3))
            q = _lib.f64c(ps.charge, (ps.count,))
            f = ps.force
            _, tm = self.handle.evaluate(pos, q, f)
            u_lj = float(self.handle.last_energies()[3])
            t.update(t_sr=float(tm[1]))
        self.last = {"u_coulomb": u_c, "u_lj": u_lj, **t}
        return u_c + u_lj


_MD_HANDLE = None


def _md_handle(box):
    global _MD_HANDLE
    if _MD_HANDLE is None:
        _MD_HANDLE = _lib.Handle()
    _MD_HANDLE.set_system(box.edge_length, 1.0, 0.5 * box.edge_length)
    return _MD_HANDLE


def velocity_verlet_step(ps, dt, force_assembler, timings=None):
    """One NVE velocity-Verlet update of host arrays (driver.py:134-153).

    Works with any force assembler (the reference's contract); the kick,
    drift and wrap run on the device.  For trajectories that stay in HBM
    use DeviceMD.
    """
    import torch

    h = _md_handle(ps.box)
    dev = torch.device("cuda", h.device)
    # copies and kernels on one explicit stream the handle is bound to, and
    # a synchronisation before every host read (the handle's kernels and
    # torch's copies are otherwise unordered)
    stream = _md_stream(dev)
    h.set_stream(stream.cuda_stream)
    t0 = time.perf_counter()
    n = ps.count
    with torch.cuda.stream(stream):
        pos = torch.from_numpy(np.ascontiguousarray(ps.position)).to(dev, non_blocking=False)
        vel = torch.from_numpy(np.ascontiguousarray(ps.velocity)).to(dev, non_blocking=False)
        frc = torch.from_numpy(np.ascontiguousarray(ps.force)).to(dev, non_blocking=False)
        mass = torch.from_numpy(np.ascontiguousarray(ps.mass)).to(dev, non_blocking=False)
        h.dev_md_kick_drift(pos.data_ptr(), vel.data_ptr(), frc.data_ptr(),
                            mass.data_ptr(), n, dt)
        pos_h, vel_h = pos.cpu(), vel.cpu()
    stream.synchronize()
    ps.position[:] = pos_h.numpy()
    ps.velocity[:] = vel_h.numpy()
    t1 = time.perf_counter()
    force_assembler(ps)
    t2 = time.perf_counter()
    with torch.cuda.stream(stream):
        frc.copy_(torch.from_numpy(np.ascontiguousarray(ps.force)))
        h.dev_md_kick(vel.data_ptr(), frc.data_ptr(), mass.data_ptr(), n, dt, kick=True)
        vel_h = vel.cpu()
    stream.synchronize()
    ps.velocity[:] = vel_h.numpy()
    t3 = time.perf_counter()
    if timings is not None:
        timings["t_integrate"] = (t1 - t0) + (t3 - t2)


_MD_STREAMS = {}


def _md_stream(dev):
    import torch
    if dev not in _MD_STREAMS:
        _MD_STREAMS[dev] = torch.cuda.Stream(device=dev)
    return _MD_STREAMS[dev]


@dataclass
class RunMetrics:
    n_steps: int
    step_wall: list = field(default_factory=list)
    components: dict = field(default_factory=lambda: {
        "t_sr": [], "t_alg1": [], "t_alg2": [], "t_lj": [], "t_integrate": [],
    })
    energy_trace: list = field(default_factory=list)
    max_step_displacement: float = 0.0
    verlet: dict = field(default_factory=lambda: {"builds": 0, "reuses": 0})
    alpha: float = 0.0
    r_cutoff: float = 0.0
    n_k: int = 0

    @property
    def total_energies(self):
        return [ke + pe for ke, pe in self.energy_trace]

    @property
    def drift(self):
        e = self.total_energies
        if len(e) < 2 or e[0] == 0.0:
            return 0.0
        e0 = e[0]
        return max(abs(x - e0) for x in e) / abs(e0)

    def median_step_wall(self, warmup=2):
        timed = self.step_wall[warmup:] or self.step_wall
        return float(np.median(timed)) if timed else 0.0

    def median_component(self, key, warmup=2):
        vals = self.components[key][warmup:] or self.components[key]
        return float(np.median(vals)) if vals else 0.0


class _Charges:
    """Charge array with the ParticleSet interface require_neutral reads."""

    def __init__(self, q):
        self.charge = q
        self.count = q.shape[0]


class DeviceMD:
    """NVE dynamics with every per-particle array resident in HBM.

    Per step: kick + drift + wrap kernel, force assembly (Ewald + fused LJ,
    forces zeroed on the device), kick + kinetic-energy kernel.  Only the
    energy scalars cross to the host.  ``download(ps)`` copies the state
    back.
    """

    def __init__(self, ps, config, skin=0.0):
        import torch

        self.config = config
        self.skin = float(skin)
        self.box = ps.box
        self.n = ps.count
        self.assembler = ForceAssembler(ps, config)
        h = self.assembler.handle
        if h is None:
            h = _md_handle(ps.box)
        self.h = h
        self.dev = torch.device("cuda", h.device)
        self.stream = torch.cuda.Stream(device=self.dev)
        h.set_stream(self.stream.cuda_stream)
        # Verlet pair lists (skin > 0): the real-space lists are rebuilt only
        # when a particle has moved skin/2 since the last build; the
        # reference rebuilds its cell lists every step
        h.set_skin(self.skin)
        f64 = dict(dtype=torch.float64, device=self.dev)
        with torch.cuda.stream(self.stream):
            self.pos = torch.from_numpy(np.ascontiguousarray(ps.position)).to(**f64)
            self.vel = torch.from_numpy(np.ascontiguousarray(ps.velocity)).to(**f64)
            self.q = torch.from_numpy(np.ascontiguousarray(ps.charge)).to(**f64)
            self.mass = torch.from_numpy(np.ascontiguousarray(ps.mass)).to(**f64)
            self.force = torch.zeros((self.n, 3), **f64)
            self.prev = torch.empty_like(self.pos)
        self.stream.synchronize()
        self._q_host = _Charges(np.array(ps.charge, dtype=np.float64, copy=True))
        self.last = None
        self._neutral_checked = False

    def assemble(self):
        """Forces for the current positions; returns the potential energy."""
        import torch

        with torch.cuda.stream(self.stream):
            self.force.zero_()
        if self.assembler.handle is None:
            self.last = {"u_coulomb": 0.0, "u_lj": 0.0, "t_sr": 0.0,
                         "t_alg1": 0.0, "t_alg2": 0.0, "t_lj": 0.0}
            return 0.0
        if self.config.coulomb_on and not self._neutral_checked:
            # the reference's host expression (core.py:139-145) on the charges
            # as uploaded, so accept/reject is identical
            require_neutral(self._q_host)
            self._neutral_checked = True
        if self.skin > 0.0:
            self.h.dev_verlet_check(self.pos.data_ptr(), self.n)
        en, tm = self.h.dev_evaluate(self.pos.data_ptr(), self.q.data_ptr(), self.n,
                                     self.force.data_ptr(), None, timings=True)
        u_lj = float(self.h.last_energies()[3]) if self.config.lj_on else 0.0
        u_c = float(en.sum()) if self.config.coulomb_on else 0.0
        self.last = {"u_coulomb": u_c, "u_lj": u_lj, "t_sr": float(tm[1]),
                     "t_alg1": float(tm[2]) if self.config.coulomb_on else 0.0,
                     "t_alg2": float(tm[3]) if self.config.coulomb_on else 0.0,
                     "t_lj": 0.0}
        return u_c + u_lj

    def kinetic(self):
        return self.h.dev_md_kick(self.vel.data_ptr(), self.force.data_ptr(),
                                  self.mass.data_ptr(), self.n, 0.0, kick=False)

    def step(self, dt):
        """One velocity-Verlet step; returns (kinetic, potential, t_integrate)."""
        import torch

        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        with torch.cuda.stream(self.stream):
            self.prev.copy_(self.pos)
            ev[0].record(self.stream)
            self.h.dev_md_kick_drift(self.pos.data_ptr(), self.vel.data_ptr(),
                                     self.force.data_ptr(), self.mass.data_ptr(),
                                     self.n, dt)
            ev[1].record(self.stream)
        pe = self.assemble()
        with torch.cuda.stream(self.stream):
            ev[2].record(self.stream)
        ke = self.h.dev_md_kick(self.vel.data_ptr(), self.force.data_ptr(),
                                self.mass.data_ptr(), self.n, dt, kick=True)
        with torch.cuda.stream(self.stream):
            ev[3].record(self.stream)
        self.stream.synchronize()
        t_int = 1e-3 * (ev[0].elapsed_time(ev[1]) + ev[2].elapsed_time(ev[3]))
        return ke, pe, t_int

    def max_displacement(self):
        """max over particles/axes of min(|dr|, L - |dr|) of the last step."""
        import torch

        with torch.cuda.stream(self.stream):
            d = (self.pos - self.prev).abs()
            d = torch.minimum(d, self.box.edge_length - d)
            m = float(d.max())
        return m

    def download(self, ps):
        self.stream.synchronize()
        ps.position[:] = self.pos.cpu().numpy()
        ps.velocity[:] = self.vel.cpu().numpy()
        ps.force[:] = self.force.cpu().numpy()


def run(config, ps=None, skin=0.0):
    """NVE dynamics with the state resident on the device (driver.py:204-246);
    skin > 0 reuses Verlet pair lists across steps (DeviceMD)."""
    if ps is None:
        cells = rocksalt_cells_for(config.n_particles)
        spacing = config.box_edge / (2 * cells)
        ps = init_rocksalt(cells, spacing)
    initial_velocities(ps, config.velocity_scale, config.seed)
    md = DeviceMD(ps, config, skin=skin)
    metrics = RunMetrics(n_steps=config.n_steps)
    if md.assembler.params is not None:
        metrics.alpha = md.assembler.params.alpha
        metrics.r_cutoff = md.assembler.params.r_cutoff
        metrics.n_k = md.assembler.solver.recip.count
    pe = md.assemble()
    metrics.energy_trace.append((md.kinetic(), pe))
    for _ in range(config.n_steps):
        t0 = time.perf_counter()
        ke, pe, t_int = md.step(config.dt)
        t1 = time.perf_counter()
        metrics.step_wall.append(t1 - t0)
        last = md.last
        for key in ("t_sr", "t_alg1", "t_alg2", "t_lj"):
            metrics.components[key].append(last[key])
        # the remainder of the step (launches, scalar copies) is integrator
        # bookkeeping; device integrator time is t_int
        metrics.components["t_integrate"].append(
            max(t_int, (t1 - t0) - last["t_sr"] - last["t_alg1"] - last["t_alg2"]))
        metrics.energy_trace.append((ke, pe))
        metrics.max_step_displacement = max(metrics.max_step_displacement,
                                            md.max_displacement())
    md.download(ps)
    metrics.verlet = md.h.verlet_info() if md.skin > 0.0 else {"builds": 0, "reuses": 0}
    return metrics
