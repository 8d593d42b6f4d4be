"""ORACLE -- TEST INFRASTRUCTURE ONLY (the checker, never the product).

ctypes wrapper over ``oracle/liboracle.so`` (built from ewald_oracle.c by
``oracle/Makefile`` or ``__graft_entry__.build()``), the CPU restatement of
the reference Ewald hot path.  Only tests/, ``__graft_entry__.smoke()`` and
bench.py's cpu-baseline / ``--impl reference`` legs may import this module.

Parity: pinned against golden vectors produced by the real reference
(``tests/golden/make_golden.py``) in ``tests/test_oracle_golden.py``.
"""

import ctypes
import math
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_INT = ctypes.c_int

_SIG = {
    "orc_rho_hat": [_P, _P, _I64, _D, _P, _I64, _INT, _P],
    "orc_long_range": [_P, _P, _I64, _D, _P, _I64, _P, _P, _INT, _P, _P],
    "orc_short_range": [_P, _P, _I64, _D, _D, _D, _INT, _P, _I64, _P, _P],
    "orc_short_range_wide": [_P, _P, _I64, _D, _D, _D, _INT, _P, _P],
}

_LIB = None


class OracleError(RuntimeError):
    def __init__(self, code, what):
        super().__init__(f"oracle {what} failed with code {code}")
        self.code = code


def lib():
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing; run `make -C oracle`")
        L = ctypes.CDLL(LIB_PATH)
        for k, a in _SIG.items():
            getattr(L, k).argtypes = a
            getattr(L, k).restype = _INT
        L.orc_num_threads.restype = _INT
        _LIB = L
    return _LIB


def host_threads():
    return int(lib().orc_num_threads())


def _p(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def _c(a, dt=np.float64):
    return np.ascontiguousarray(a, dtype=dt)


def kspace_coeff(m_int, L, alpha):
    """C_k = 4 pi/(V k^2) exp(-k^2/(4 alpha)) as ReciprocalSpace (ewald.py:157-161)."""
    kvec = (2.0 * math.pi / L) * np.asarray(m_int).astype(float)
    k2 = np.einsum("ij,ij->i", kvec, kvec)
    return (4.0 * math.pi / (L**3 * k2)) * np.exp(-k2 / (4.0 * alpha))


def rho_hat(pos, q, L, m_int, threads=None):
    pos, q, m = _c(pos), _c(q), _c(m_int, np.int64)
    K = m.shape[0]
    out = np.zeros(2 * K)
    rc = lib().orc_rho_hat(_p(pos), _p(q), q.shape[0], float(L), _p(m), K,
                           threads or host_threads(), _p(out))
    if rc:
        raise OracleError(rc, "rho_hat")
    return out


def long_range(pos, q, L, m_int, coeff, rho, force=None, threads=None):
    pos, q, m = _c(pos), _c(q), _c(m_int, np.int64)
    coeff, rho = _c(coeff), _c(rho)
    n = q.shape[0]
    f = np.zeros((n, 3)) if force is None else force
    u = ctypes.c_double(0.0)
    rc = lib().orc_long_range(_p(pos), _p(q), n, float(L), _p(m), m.shape[0],
                              _p(coeff), _p(rho), threads or host_threads(),
                              _p(f), ctypes.byref(u))
    if rc:
        raise OracleError(rc, "long_range")
    return u.value, f


def short_range(pos, q, L, r_cutoff, alpha, sel=None, force=None,
                threads=None):
    pos, q = _c(pos), _c(q)
    n = q.shape[0]
    f = np.zeros((n, 3)) if force is None else force
    s = None if sel is None else _c(sel, np.int64)
    u = ctypes.c_double(0.0)
    rc = lib().orc_short_range(_p(pos), _p(q), n, float(L), float(r_cutoff),
                               float(alpha), threads or host_threads(),
                               _p(s), 0 if s is None else s.shape[0], _p(f),
                               ctypes.byref(u))
    if rc:
        raise OracleError(rc, "short_range")
    return u.value, f


def short_range_wide(pos, q, L, r_cutoff, alpha, force=None, threads=None):
    """Image-shell real space for r_c > L/2 (ewald.py:490-576)."""
    pos, q = _c(pos), _c(q)
    n = q.shape[0]
    f = np.zeros((n, 3)) if force is None else force
    u = ctypes.c_double(0.0)
    rc = lib().orc_short_range_wide(_p(pos), _p(q), n, float(L),
                                    float(r_cutoff), float(alpha),
                                    threads or host_threads(), _p(f),
                                    ctypes.byref(u))
    if rc:
        raise OracleError(rc, "short_range_wide")
    return u.value, f


def self_energy(q, alpha):
    """-sqrt(alpha/pi) * q.q (ewald.py:482-484)."""
    q = _c(q)
    return -math.sqrt(alpha / math.pi) * float(q @ q)


def evaluate(pos, q, L, alpha, r_cutoff, m_int, coeff=None, threads=None):
    """EwaldSolver.evaluate restated (ewald.py:629-655)."""
    if coeff is None:
        coeff = kspace_coeff(m_int, L, alpha)
    f = np.zeros((np.asarray(q).shape[0], 3))
    u_self = self_energy(q, alpha)
    if r_cutoff > 0.5 * L:   # the reference's wide-cutoff branch (ewald.py:635-637)
        u_sr, _ = short_range_wide(pos, q, L, r_cutoff, alpha, force=f,
                                   threads=threads)
    else:
        u_sr, _ = short_range(pos, q, L, r_cutoff, alpha, force=f,
                              threads=threads)
    rho = rho_hat(pos, q, L, m_int, threads=threads)
    u_lr, _ = long_range(pos, q, L, m_int, coeff, rho, force=f,
                         threads=threads)
    return dict(u_sr=u_sr, u_lr=u_lr, u_self=u_self, force=f, rho=rho)
