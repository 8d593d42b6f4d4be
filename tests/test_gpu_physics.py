"""Physical invariants of the GPU evaluation, mirroring the reference's own
invariant tests (test_ewald.py:279-367, test_acceptance.py criteria 2, 3 and
9): forces are minus the energy gradient (central differences), the total
energy does not depend on the splitting parameter alpha, it is invariant
under a rigid translation, and the net force vanishes.  Same systems, seeds
and bounds as the reference's tests, through the public API."""

import math

import numpy as np
import pytest

from conftest import random_neutral

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ew():
    import paper_1708_01135_b200 as ew
    return ew


def particle_set(ew, pos, q, L):
    ps = ew.create_particle_set(pos.shape[0], ew.SimulationBox(L))
    ps.position[:] = pos
    ps.charge[:] = q
    return ps


def params_for(ew, alpha, tolerance=1e-6):
    """The reference's ewald_params_for (test_ewald.py:120-124)."""
    s = math.sqrt(-math.log(tolerance))
    return ew.EwaldParams(alpha=alpha, r_cutoff=s / math.sqrt(alpha),
                          k_cutoff=2.0 * s * math.sqrt(alpha), tolerance=tolerance)


def solve(ew, ps, params):
    ps.force[:] = 0.0
    res = ew.EwaldSolver(ps.box, params).evaluate(ps)
    return res.total, ps.force.copy()


def fd_forces(ew, ps, params, h):
    """Central differences -dU/dr (the reference's oracle.finite_difference_forces:
    displaced by +-h one component at a time, rewrapped, restored exactly)."""
    solver = ew.EwaldSolver(ps.box, params)
    L = ps.box.edge_length
    pos = ps.position
    out = np.zeros((ps.count, 3))

    def energy():
        ps.force[:] = 0.0
        return solver.evaluate(ps).total
    for i in range(ps.count):
        for a in range(3):
            orig = pos[i, a]
            pos[i, a] = (orig + h) % L
            up = energy()
            pos[i, a] = (orig - h) % L
            um = energy()
            pos[i, a] = orig
            out[i, a] = -(up - um) / (2.0 * h)
    return out


def test_two_charge_force_matches_finite_difference(ew):
    """test_ewald.py:279-295: a +-1 pair at L/4."""
    pos = np.array([[2.0, 6.0, 6.0], [5.0, 6.0, 6.0]])
    ps = particle_set(ew, pos, np.array([1.0, -1.0]), 12.0)
    params = ew.choose_parameters(2, ps.box, 1e-6)
    fd = fd_forces(ew, ps, params, 1e-4)
    _, f = solve(ew, ps, params)
    scale = np.abs(fd).max()
    assert np.abs(f - fd).max() <= 1e-6 * scale


@pytest.mark.parametrize("seed", [40, 41, 42])
def test_random_forces_match_finite_difference(ew, seed):
    """test_acceptance.py criterion 2: random neutral systems."""
    pos, q = random_neutral(12, 9.0, seed=seed)
    ps = particle_set(ew, pos, q, 9.0)
    params = ew.choose_parameters(12, ps.box, 1e-6)
    fd = fd_forces(ew, ps, params, 1e-4)
    _, f = solve(ew, ps, params)
    scale = max(np.abs(fd).max(), 1e-12)
    assert np.abs(f - fd).max() <= 1e-5 * scale


def test_alpha_invariance(ew):
    """test_ewald.py:314-329: alpha x0.5 and x2 (the larger cutoff of the
    smaller alpha exceeds L/2: the image-shell real space)."""
    pos, q = random_neutral(48, 11.0, seed=31)
    ps = particle_set(ew, pos, q, 11.0)
    base = ew.choose_parameters(48, ps.box, 1e-6)
    u0, f0 = solve(ew, ps, base)
    worst = 0.0
    for factor in (0.5, 2.0):
        u1, f1 = solve(ew, ps, params_for(ew, base.alpha * factor))
        worst = max(worst, abs(u1 - u0) / abs(u0))
        rows = np.arange(ps.count)
        idx = np.argmax(np.abs(f0), axis=1)
        assert np.max(np.abs(f1[rows, idx] - f0[rows, idx]) / np.abs(f0[rows, idx])) <= 1e-4
    assert worst <= 5e-6


@pytest.mark.parametrize("name", ["small", "c2"])
def test_translation_invariance_and_net_force(ew, name):
    """test_ewald.py:346-360 (and criterion 9 at the c2 size): a rigid shift
    (rewrapped) changes U by <= 1e-10 relative; the net force is ~0."""
    if name == "small":
        pos, q = random_neutral(32, 10.0, seed=33)
        L = 10.0
        params = ew.choose_parameters(32, ew.SimulationBox(L), 1e-6)
    else:
        from paper_1708_01135_b200 import workloads as wl
        cfg = wl.make_config("c2", seed=0)
        pos, q, L = cfg["pos"], cfg["q"], cfg["L"]
        params = ew.EwaldParams(cfg["alpha_ref"], cfg["r_cutoff"], wl.k_cutoff_for(cfg), 1e-6)
    ps = particle_set(ew, pos, q, L)
    u0, f0 = solve(ew, ps, params)
    ps.position += np.array([3.7, -1.1, 0.4])
    ps.wrap()
    u1, _ = solve(ew, ps, params)
    assert abs(u1 - u0) / abs(u0) <= 1e-10
    residual = np.linalg.norm(f0.sum(axis=0))
    assert residual <= 1e-8 * np.abs(f0).max() * ps.count


def test_alpha_invariance_nacl_1728_acceptance_3(ew):
    """The reference's acceptance criterion 3 (test_acceptance.py:106-128):
    jittered rock salt 12^3 (N=1728, spacing 2.5), alpha x0.5 (r_c > L/2:
    the image-shell real space on the device) and x2: |dU|/U <= 5e-6."""
    from paper_1708_01135_b200 import md
    ps = md.init_rocksalt(6, 2.5)
    rng = np.random.default_rng(3)
    ps.position += 0.1 * rng.standard_normal(ps.position.shape)
    ps.wrap()
    base = ew.choose_parameters(ps.count, ps.box, 1e-6)

    def total(params):
        ps.force[:] = 0.0
        return ew.total_coulomb(ps, params)
    u0 = total(base)
    worst = max(abs(total(params_for(ew, base.alpha * f)) - u0) / abs(u0) for f in (0.5, 2.0))
    assert worst <= 5e-6
