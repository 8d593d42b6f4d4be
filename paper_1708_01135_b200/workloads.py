"""Seeded synthetic inputs for the five BASELINE.json configurations.

Rock-salt configs (c1, c2, c3, c5) follow the reference lattice builder
``init_rocksalt`` (``driver.py:54-78``): 2c sites per dimension at spacing a,
site index x-slowest / z-fastest (``meshgrid(indexing="ij")`` ravel), charge
+1 on even (ix+iy+iz).  Positions are then jittered with
``default_rng(seed).standard_normal((N, 3)) * sigma`` and wrapped
(``core.py:156-161``), the idiom of ``test_acceptance.py:36-41``.

The random gas (c4) is placed by hard-core random sequential adsorption
(``csrc/workloads.c``) and its N(0,1) charges are mean-shifted, quantised to
a 2**-30 grid and closed with ``q[-1] = -fsum(q[:-1])`` so that the sum is
exactly zero in every summation order (without
this the reference's 1e-12 neutrality check rejects most seeds).

alpha convention: BASELINE.json quotes the conventional beta (1/length,
``erfc(beta r)``); the reference ``EwaldParams.alpha`` is beta**2
(``ewald.py:216-218``), so ``alpha_ref = alpha_cfg**2``.
"""

import ctypes
import math
import os

import numpy as np

from .core import SimulationBox

CONFIGS = {
    "c1": dict(kind="rocksalt", side=10, spacing=1.0, sigma=0.05,
               alpha_cfg=0.711, r_cutoff=4.5, n_max=8),
    "c2": dict(kind="rocksalt", side=32, spacing=1.0, sigma=0.1,
               alpha_cfg=0.533, r_cutoff=6.0, n_max=18),
    "c3": dict(kind="rocksalt", side=64, spacing=1.0, sigma=0.1,
               alpha_cfg=0.533, r_cutoff=6.0, n_max=35),
    "c4": dict(kind="gas", n=131072, L=50.8, min_sep=0.8,
               alpha_cfg=0.4, r_cutoff=8.0, n_max=21),
    "c5": dict(kind="rocksalt", side=100, spacing=1.0, sigma=0.1,
               alpha_cfg=0.533, r_cutoff=6.0, n_max=55),
}


def rocksalt_positions(side, spacing):
    """Sites and +-1 charges of init_rocksalt(side//2, spacing)."""
    if side < 2 or side % 2:
        raise ValueError(f"rock-salt side must be even and >= 2, got {side}")
    idx = np.arange(side)
    ix, iy, iz = np.meshgrid(idx, idx, idx, indexing="ij")
    pos = np.empty((side**3, 3))
    pos[:, 0] = ix.ravel() * spacing
    pos[:, 1] = iy.ravel() * spacing
    pos[:, 2] = iz.ravel() * spacing
    q = np.where((ix + iy + iz).ravel() % 2 == 0, 1.0, -1.0)
    return pos, q


def wrap(pos, L):
    out = pos - L * np.floor(pos / L)
    return np.where(out >= L, out - L, out)


def jittered_rocksalt(side, spacing, sigma, seed):
    pos, q = rocksalt_positions(side, spacing)
    L = side * spacing
    rng = np.random.default_rng(seed)
    pos = pos + sigma * rng.standard_normal(pos.shape)
    return wrap(pos, L), q, L


_GEN = None


def _gen_lib():
    global _GEN
    if _GEN is None:
        path = os.path.join(os.path.dirname(__file__), "libewb_workloads.so")
        if not os.path.exists(path):
            raise ImportError(
                f"{path} missing: run __graft_entry__.build() first")
        lib = ctypes.CDLL(path)
        lib.ewb_gen_hardcore_gas.restype = ctypes.c_int
        lib.ewb_gen_hardcore_gas.argtypes = [
            ctypes.c_int64, ctypes.c_double, ctypes.c_double, ctypes.c_uint64,
            ctypes.c_int64, ctypes.c_void_p, ctypes.POINTER(ctypes.c_int64)]
        _GEN = lib
    return _GEN


def hardcore_gas_positions(n, L, min_sep, seed):
    pos = np.empty((n, 3))
    att = ctypes.c_int64(0)
    rc = _gen_lib().ewb_gen_hardcore_gas(
        n, L, min_sep, seed, 1000 * n, pos.ctypes.data, ctypes.byref(att))
    if rc != 0:
        raise RuntimeError(f"hard-core sampler failed (code {rc}) after "
                           f"{att.value} attempts")
    return pos


def neutral_gaussian_charges(n, seed):
    """N(0,1) charges shifted by the mean and made exactly neutral."""
    rng = np.random.default_rng(seed)
    q = rng.standard_normal(n)
    q -= q.mean()
    q = np.round(q / 2.0**-30) * 2.0**-30
    q[-1] = -math.fsum(q[:-1])
    return q


def cube_half_m(n_max):
    """Half-space integer table of the cube |m_x|,|m_y|,|m_z| <= n_max.

    Same storage order and half-space rule as the reference enumerator
    (``ewald.py:189-197``): meshgrid ij ravel (x slowest, z fastest), keep
    m_z > 0, or m_z == 0 with (m_y, m_x) lexicographically positive.
    """
    rng = np.arange(-n_max, n_max + 1)
    mx, my, mz = np.meshgrid(rng, rng, rng, indexing="ij")
    m = np.stack([mx.ravel(), my.ravel(), mz.ravel()], axis=1)
    z, y, x = m[:, 2], m[:, 1], m[:, 0]
    half = (z > 0) | ((z == 0) & (y > 0)) | ((z == 0) & (y == 0) & (x > 0))
    return m[half].astype(np.int64)


def make_config(name, seed=0):
    """Inputs and parameters of one BASELINE.json config.

    Returns a dict with pos (N,3), q (N,), L, alpha_cfg, alpha_ref (=beta^2),
    r_cutoff, n_max and m_int (cube half-space table).
    """
    cfg = dict(CONFIGS[name])
    if cfg["kind"] == "rocksalt":
        pos, q, L = jittered_rocksalt(cfg["side"], cfg["spacing"],
                                      cfg["sigma"], seed)
    else:
        L = cfg["L"]
        pos = hardcore_gas_positions(cfg["n"], L, cfg["min_sep"], seed)
        q = neutral_gaussian_charges(cfg["n"], seed)
    cfg.update(name=name, seed=seed, pos=np.ascontiguousarray(pos),
               q=np.ascontiguousarray(q), L=float(L),
               alpha_ref=cfg["alpha_cfg"] ** 2,
               m_int=cube_half_m(cfg["n_max"]))
    cfg["box"] = SimulationBox(L)
    return cfg


def k_cutoff_for(cfg):
    """Reciprocal cutoff enclosing the cube (unused once a table is given)."""
    return (2.0 * math.pi / cfg["L"]) * cfg["n_max"] * math.sqrt(3.0)
