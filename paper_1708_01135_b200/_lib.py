"""ctypes binding of libewaldb200.so (the C-ABI in include/ewald_b200.h).

There is no fallback: if the shared library is missing or no CUDA device is
usable, every entry point raises.  Status codes map onto the reference's
exception classes (core.py:14-55).
"""

import ctypes
import os

import numpy as np

from .core import error

LIB_NAME = "libewaldb200.so"
LIB_PATH = os.environ.get(
    "EWALDB200_LIB",
    os.path.join(os.path.dirname(os.path.abspath(__file__)), LIB_NAME))

EWB_OK = 0
EWB_EINVAL = 1
EWB_ECOINCIDENT = 2
EWB_ECUTOFF = 3
EWB_EUNWRAPPED = 4
EWB_ECUDA = 5
EWB_EBOX = 6
EWB_EKSPACE = 7
EWB_ESTATE = 8
EWB_ESIZE = 9

#: device error bits (ewb_dev_status)
ERR_UNWRAPPED = 1
ERR_COINCIDENT = 2

_P = ctypes.c_void_p
_I64 = ctypes.c_int64
_D = ctypes.c_double
_INT = ctypes.c_int

#: every symbol include/ewald_b200.h declares, with (restype, argtypes)
SIGNATURES = {
    "ewb_version": (_INT, []),
    "ewb_create": (_INT, [_INT, ctypes.POINTER(_P)]),
    "ewb_destroy": (None, [_P]),
    "ewb_last_error": (ctypes.c_char_p, [_P]),
    "ewb_set_stream": (_INT, [_P, ctypes.c_size_t]),
    "ewb_use_own_stream": (_INT, [_P]),
    "ewb_set_max_segment": (_INT, [_P, _INT]),
    "ewb_set_max_pair_segment": (_INT, [_P, _INT]),
    "ewb_set_stencil": (_INT, [_P, _INT]),
    "ewb_set_deterministic": (_INT, [_P, _INT]),
    "ewb_set_real_space_split": (_INT, [_P, _INT]),
    "ewb_set_graphs": (_INT, [_P, _INT]),
    "ewb_set_const_gather": (_INT, [_P, _INT]),
    "ewb_set_tensor_cores": (_INT, [_P, _INT]),
    "ewb_set_overlap": (_INT, [_P, _INT]),
    "ewb_set_system": (_INT, [_P, _D, _D, _D, _D]),
    "ewb_set_kspace": (_INT, [_P, _P, _I64, _P]),
    "ewb_kspace_info": (_INT, [_P, _P]),
    "ewb_compute_rho_hat": (_INT, [_P, _P, _P, _I64, _P]),
    "ewb_long_range": (_INT, [_P, _P, _P, _I64, _P, _P, _P]),
    "ewb_short_range": (_INT, [_P, _P, _P, _I64, _P, _P]),
    "ewb_self_energy": (_INT, [_P, _P, _I64, _P]),
    "ewb_evaluate": (_INT, [_P, _P, _P, _I64, _P, _P, _P, _P]),
    "ewb_dev_load": (_INT, [_P, _P, _P, _I64]),
    "ewb_dev_slot_doubles": (_I64, [_P]),
    "ewb_dev_rho_partial": (_INT, [_P, _I64, _I64, _P]),
    "ewb_dev_kspace_finalize": (_INT, [_P, _P, _P, _P]),
    "ewb_dev_kspace_finalize_peer": (_INT, [_P, _P, _INT, _P]),
    "ewb_enable_peer_access": (_INT, [_P, _INT]),
    "ewb_ipc_slots": (_INT, [_P, ctypes.POINTER(_P), _P]),
    "ewb_ipc_open": (_INT, [_P, _P, ctypes.POINTER(_P)]),
    "ewb_ipc_close": (_INT, [_P, _P]),
    "ewb_dev_recip_forces": (_INT, [_P, _I64, _I64, _P]),
    "ewb_dev_real_space": (_INT, [_P, _INT, _INT, _P, _P]),
    "ewb_dev_self_energy": (_INT, [_P, _P]),
    "ewb_dev_self_energy_range": (_INT, [_P, _I64, _I64, _P]),
    "ewb_set_geometry_n": (_INT, [_P, _I64]),
    "ewb_rs_geometry": (_INT, [_P, _P]),
    "ewb_dev_rows": (_INT, [_P, _P, _I64, _P]),
    "ewb_dev_row_order": (_INT, [_P, _P, _I64, _P, _P]),
    "ewb_dev_real_space_rows": (_INT, [_P, _INT, _INT, _P, _P]),
    "ewb_dev_energies": (_INT, [_P, _P]),
    "ewb_dev_check": (_INT, [_P]),
    "ewb_dev_status": (_INT, [_P, _P]),
    "ewb_dev_evaluate": (_INT, [_P, _P, _P, _I64, _P, _P, _P, _P]),
    "ewb_set_coulomb": (_INT, [_P, _INT]),
    "ewb_set_lj": (_INT, [_P, _INT, _D, _D, _D, _D, _D, _D]),
    "ewb_last_energies": (_INT, [_P, _P]),
    "ewb_dev_md_kick_drift": (_INT, [_P, _P, _P, _P, _P, _I64, _D]),
    "ewb_dev_md_kick": (_INT, [_P, _P, _P, _P, _I64, _D, _INT, _P]),
    "ewb_probe_fp64_peak": (_INT, [_P, _P]),
    "ewb_probe_i8_peak": (_INT, [_P, _P]),
    "ewb_probe_i8_shape": (_INT, [_P, _INT, _P]),
    "ewb_probe_i8_shape_ts": (_INT, [_P, _INT, _P]),
    "ewb_tc_info": (_INT, [_P, _P]),
    "ewb_last_pair_count": (_INT, [_P, _P]),
    "ewb_launch_count": (_I64, [_P]),
    "ewb_host_alloc": (_INT, [ctypes.c_size_t, ctypes.POINTER(ctypes.c_void_p)]),
    "ewb_host_free": (_INT, [_P]),
    "ewb_set_skin": (_INT, [_P, _D]),
    "ewb_dev_verlet_check": (_INT, [_P, _P, _I64, ctypes.POINTER(_INT)]),
    "ewb_verlet_info": (_INT, [_P, _P]),
    "ewb_host_register": (_INT, [_P, ctypes.c_size_t]),
    "ewb_host_unregister": (_INT, [_P]),
}

_LIB = None


def load_library():
    """Load the CUDA library; raise ImportError (loudly) if it is absent."""
    global _LIB
    if _LIB is not None:
        return _LIB
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} not found: the CUDA extension is not built "
            f"(run __graft_entry__.build()); there is no CPU fallback")
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _LIB = lib
    return lib


def _ptr(a):
    return None if a is None else ctypes.c_void_p(a.ctypes.data)


def pinned_zeros(n):
    """float64 zeros in page-locked host memory (device copies land directly);
    plain numpy memory when no CUDA device is present."""
    import weakref
    n = int(n)
    lib = load_library()
    ptr = ctypes.c_void_p()
    if n < 1 or lib.ewb_host_alloc(n * 8, ctypes.byref(ptr)) != EWB_OK or not ptr.value:
        return np.zeros(max(n, 0))
    arr = np.ctypeslib.as_array((ctypes.c_double * n).from_address(ptr.value))
    arr[:] = 0.0
    weakref.finalize(arr, lib.ewb_host_free, ctypes.c_void_p(ptr.value))
    return arr


class HostPins:
    """Caller host arrays page-locked in place while they live.

    A reference ``ParticleSet`` allocates pageable numpy arrays
    (core.py:111-115) and an MD loop hands the same arrays to every
    evaluation; copies from pageable memory are staged by the driver and
    block the host.  An array that owns its memory, is at least MIN_BYTES
    and C-contiguous is registered (cudaHostRegister) the second time it is
    seen; a finalizer unregisters it before numpy frees the memory (weakref
    callbacks run at the start of the array's deallocation).  Arrays that
    do not own their memory (views, ctypes / torch pinned buffers) are left
    alone."""

    MIN_BYTES = 1 << 18
    MAX_ENTRIES = 64

    def __init__(self):
        self._seen = {}    # (ptr, nbytes) -> weakref to the owning array
        self._pinned = set()

    def touch(self, a):
        import weakref
        if not (isinstance(a, np.ndarray) and a.base is None and a.flags.owndata
                and a.flags.c_contiguous and a.nbytes >= self.MIN_BYTES):
            return
        key = (a.ctypes.data, a.nbytes)
        if key in self._pinned:
            return
        ref = self._seen.get(key)
        if ref is None or ref() is not a:
            if len(self._seen) >= self.MAX_ENTRIES:
                self._seen = {k: r for k, r in self._seen.items() if r() is not None}
                if len(self._seen) >= self.MAX_ENTRIES:
                    return
            self._seen[key] = weakref.ref(a)
            return
        lib = load_library()
        if lib.ewb_host_register(ctypes.c_void_p(key[0]), key[1]) != EWB_OK:
            return
        self._pinned.add(key)
        del self._seen[key]
        weakref.finalize(a, HostPins._release, self, key)

    @staticmethod
    def _release(pins, key):
        pins._pinned.discard(key)
        load_library().ewb_host_unregister(ctypes.c_void_p(key[0]))


PINS = HostPins()


class DeviceError(RuntimeError):
    """CUDA failure or misuse of the device library."""


def raise_for(status, message, lib=None):
    if status == EWB_OK:
        return
    if status == EWB_ECOINCIDENT:
        raise error("CoincidentParticlesError", message)
    if status == EWB_ECUTOFF:
        raise error("CutoffTooLargeError", message)
    if status == EWB_EKSPACE:
        raise error("KSpaceEmptyError", message)
    if status == EWB_EBOX:
        raise error("BoxTooSmallError", message)
    if status == EWB_ESIZE:
        raise error("OracleSizeError", message)
    if status in (EWB_EINVAL, EWB_EUNWRAPPED):
        raise ValueError(message)
    raise DeviceError(f"libewaldb200 status {status}: {message}")


def default_device():
    return int(os.environ.get("EWALDB200_DEVICE",
                              os.environ.get("LOCAL_RANK", "0")))


def f64c(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None and a.shape != shape:
        a = a.reshape(shape)
    return a


class Handle:
    """One device context: box/parameters, k-space plan, device buffers."""

    def __init__(self, device=None):
        self.lib = load_library()
        self.device = default_device() if device is None else int(device)
        h = ctypes.c_void_p()
        st = self.lib.ewb_create(self.device, ctypes.byref(h))
        if st != EWB_OK:
            raise DeviceError(
                f"ewb_create(device={self.device}) failed with status {st}: "
                f"no usable CUDA device (this package has no CPU path)")
        self.h = h
        self.system = None
        self.kspace_key = None
        self.deterministic = False

    def __del__(self):
        h = getattr(self, "h", None)
        if h is not None and h.value:
            try:
                self.lib.ewb_destroy(h)
            except Exception:
                pass
            self.h = None

    def _check(self, st):
        if st != EWB_OK:
            msg = self.lib.ewb_last_error(self.h)
            raise_for(st, msg.decode() if msg else "", self.lib)

    # configuration -------------------------------------------------------
    def set_system(self, L, alpha, r_cutoff):
        key = (float(L), float(alpha), float(r_cutoff))
        if key != self.system:
            rc = float(r_cutoff)
            self._check(self.lib.ewb_set_system(self.h, key[0], key[1], rc,
                                                rc**2))
            self.system = key

    def set_kspace(self, m_int, coeff, key=None):
        if key is not None and key == self.kspace_key:
            return
        m = np.ascontiguousarray(m_int, dtype=np.int64).reshape(-1, 3)
        c = f64c(coeff)
        if c.shape[0] != m.shape[0]:
            raise ValueError("coeff and m_int lengths differ")
        self._check(self.lib.ewb_set_kspace(self.h, _ptr(m), m.shape[0],
                                            _ptr(c)))
        self.kspace_key = key

    def set_max_segment(self, mcap):
        self._check(self.lib.ewb_set_max_segment(self.h, int(mcap)))
        self.kspace_key = None

    def set_max_pair_segment(self, mcap1):
        self._check(self.lib.ewb_set_max_pair_segment(self.h, int(mcap1)))
        self.kspace_key = None

    def set_const_gather(self, on):
        self._check(self.lib.ewb_set_const_gather(self.h, 1 if on else 0))

    def set_tensor_cores(self, on):
        """True: tensor cores, False: FP64 kernels, "auto": by problem size."""
        mode = 2 if on == "auto" else (1 if on else 0)
        self._check(self.lib.ewb_set_tensor_cores(self.h, mode))

    def set_overlap(self, on):
        self._check(self.lib.ewb_set_overlap(self.h, 1 if on else 0))

    def set_graphs(self, on):
        self._check(self.lib.ewb_set_graphs(self.h, 1 if on else 0))

    def set_deterministic(self, on):
        self._check(self.lib.ewb_set_deterministic(self.h, 1 if on else 0))
        self.deterministic = bool(on)

    def set_real_space_split(self, mode):
        """0/False: the fused traversal + evaluation kernel (default);
        1/True: two passes -- per-unit pair lists in HBM, then their
        evaluation (the machinery of the Verlet lists, ewb_set_skin);
        2: two passes with a tiny list capacity (tests the overflow pass)."""
        self._check(self.lib.ewb_set_real_space_split(self.h, int(mode)))

    def set_skin(self, skin):
        """Verlet pair lists built at r_c + skin, reused while every particle
        stays within skin/2 of its build position (0: rebuild every call)."""
        self._check(self.lib.ewb_set_skin(self.h, float(skin)))

    def dev_verlet_check(self, d_pos, n):
        """True if the next evaluation of d_pos must rebuild the lists."""
        r = _INT(1)
        self._check(self.lib.ewb_dev_verlet_check(self.h, _P(d_pos), int(n), ctypes.byref(r)))
        return bool(r.value)

    def verlet_info(self):
        out = np.zeros(2, dtype=np.int64)
        self._check(self.lib.ewb_verlet_info(self.h, out.ctypes.data))
        return {"builds": int(out[0]), "reuses": int(out[1])}

    def set_stencil(self, rad):
        self._check(self.lib.ewb_set_stencil(self.h, int(rad)))

    def kspace_info(self):
        info = np.zeros(8, dtype=np.int64)
        self._check(self.lib.ewb_kspace_info(self.h, _ptr(info)))
        return dict(zip(("K", "n_items", "M", "n_rows", "n_tiles",
                         "max_table", "n_pair_items", "M1"), info.tolist()))

    def set_stream(self, stream_ptr):
        """Bind every later call to a CUDA stream (0: the legacy default
        stream, i.e. torch's default stream)."""
        self._check(self.lib.ewb_set_stream(self.h, int(stream_ptr)))

    def use_own_stream(self):
        """Back to the handle's own non-blocking stream."""
        self._check(self.lib.ewb_use_own_stream(self.h))

    def set_coulomb(self, on):
        self._check(self.lib.ewb_set_coulomb(self.h, 1 if on else 0))

    def set_lj(self, on, sigma2=0.0, four_eps=0.0, shift=0.0, tf_eps=0.0,
               rc_lj=0.0):
        rc_lj = float(rc_lj)
        self._check(self.lib.ewb_set_lj(self.h, 1 if on else 0, float(sigma2),
                                        float(four_eps), float(shift),
                                        float(tf_eps), rc_lj, rc_lj**2))

    def last_energies(self):
        out = np.zeros(4)
        self._check(self.lib.ewb_last_energies(self.h, _ptr(out)))
        return out

    def dev_md_kick_drift(self, d_pos, d_vel, d_force, d_mass, n, dt):
        self._check(self.lib.ewb_dev_md_kick_drift(self.h, d_pos, d_vel, d_force,
                                                   d_mass, int(n), float(dt)))

    def dev_md_kick(self, d_vel, d_force, d_mass, n, dt, kick=True):
        ke = ctypes.c_double(0.0)
        self._check(self.lib.ewb_dev_md_kick(self.h, d_vel, d_force, d_mass, int(n),
                                             float(dt), 1 if kick else 0,
                                             ctypes.byref(ke)))
        return ke.value

    def probe_fp64_peak(self):
        out = ctypes.c_double(0.0)
        self._check(self.lib.ewb_probe_fp64_peak(self.h, ctypes.byref(out)))
        return out.value

    def probe_i8_peak(self):
        out = ctypes.c_double(0.0)
        self._check(self.lib.ewb_probe_i8_peak(self.h, ctypes.byref(out)))
        return out.value

    def probe_i8_shape(self, n_mma):
        out = ctypes.c_double(0.0)
        self._check(self.lib.ewb_probe_i8_shape(self.h, int(n_mma), ctypes.byref(out)))
        return out.value

    def probe_i8_shape_ts(self, n_mma):
        out = ctypes.c_double(0.0)
        self._check(self.lib.ewb_probe_i8_shape_ts(self.h, int(n_mma), ctypes.byref(out)))
        return out.value

    def tc_info(self):
        info = np.zeros(8, dtype=np.int64)
        self._check(self.lib.ewb_tc_info(self.h, _ptr(info)))
        return dict(zip(("enabled", "k1_mtiles", "k1_npad_sum", "k3_mtiles", "k3_K",
                         "k3_pairs_per_kstep", "k1_pairs_per_kstep", "A"), info.tolist()))

    def last_pair_count(self):
        out = ctypes.c_int64(0)
        self._check(self.lib.ewb_last_pair_count(self.h, ctypes.byref(out)))
        return out.value

    def launch_count(self):
        return int(self.lib.ewb_launch_count(self.h))

    # host-pointer entry points --------------------------------------------
    def compute_rho_hat(self, pos, q, rho_out):
        n = q.shape[0]
        self._check(self.lib.ewb_compute_rho_hat(self.h, _ptr(pos), _ptr(q),
                                                 n, _ptr(rho_out)))

    def long_range(self, pos, q, rho, force):
        u = ctypes.c_double(0.0)
        self._check(self.lib.ewb_long_range(self.h, _ptr(pos), _ptr(q),
                                            q.shape[0], _ptr(rho),
                                            _ptr(force), ctypes.byref(u)))
        return u.value

    def short_range(self, pos, q, force):
        u = ctypes.c_double(0.0)
        self._check(self.lib.ewb_short_range(self.h, _ptr(pos), _ptr(q),
                                             q.shape[0], _ptr(force),
                                             ctypes.byref(u)))
        return u.value

    def self_energy(self, q):
        u = ctypes.c_double(0.0)
        self._check(self.lib.ewb_self_energy(self.h, _ptr(q), q.shape[0],
                                             ctypes.byref(u)))
        return u.value

    def evaluate(self, pos, q, force, rho_out=None):
        en = np.zeros(3)
        tm = np.zeros(4)
        self._check(self.lib.ewb_evaluate(self.h, _ptr(pos), _ptr(q),
                                          q.shape[0], _ptr(force),
                                          _ptr(rho_out), _ptr(en), _ptr(tm)))
        return en, tm

    # device-pointer stages (integers are raw device addresses) -------------
    def dev_load(self, d_pos, d_q, n):
        self._check(self.lib.ewb_dev_load(self.h, d_pos, d_q, int(n)))

    def dev_slot_doubles(self):
        return int(self.lib.ewb_dev_slot_doubles(self.h))

    def dev_rho_partial(self, i0, i1, d_slots):
        self._check(self.lib.ewb_dev_rho_partial(self.h, int(i0), int(i1),
                                                 d_slots))

    def dev_kspace_finalize(self, d_slots, d_rho_out=None):
        u = ctypes.c_double(0.0)
        self._check(self.lib.ewb_dev_kspace_finalize(
            self.h, d_slots, d_rho_out, ctypes.byref(u)))
        return u.value

    def dev_recip_forces(self, i0, i1, d_force):
        self._check(self.lib.ewb_dev_recip_forces(self.h, int(i0), int(i1),
                                                  d_force))

    def dev_real_space(self, part, nparts, d_force):
        u = ctypes.c_double(0.0)
        self._check(self.lib.ewb_dev_real_space(self.h, int(part),
                                                int(nparts), d_force,
                                                ctypes.byref(u)))
        return u.value

    def dev_self_energy(self):
        u = ctypes.c_double(0.0)
        self._check(self.lib.ewb_dev_self_energy(self.h, ctypes.byref(u)))
        return u.value

    # domain decomposition (distributed.SlabEwald)
    def set_geometry_n(self, n_global):
        self._check(self.lib.ewb_set_geometry_n(self.h, int(n_global)))

    def rs_geometry(self):
        info = np.zeros(4, dtype=np.int64)
        self._check(self.lib.ewb_rs_geometry(self.h, _ptr(info)))
        return dict(zip(("cpd", "rad", "n_rows", "fold"), info.tolist()))

    def dev_row_order(self, d_pos, n, d_order, d_row_start):
        self._check(self.lib.ewb_dev_row_order(self.h, d_pos, int(n), d_order, d_row_start))

    def dev_rows(self, d_pos, n, d_rows):
        self._check(self.lib.ewb_dev_rows(self.h, d_pos, int(n), d_rows))

    def dev_real_space_rows_async(self, row_lo, row_hi, d_force):
        self._check(self.lib.ewb_dev_real_space_rows(self.h, int(row_lo), int(row_hi),
                                                     d_force, None))

    def dev_self_energy_range_async(self, i0, i1):
        self._check(self.lib.ewb_dev_self_energy_range(self.h, int(i0), int(i1), None))

    # asynchronous variants: energies stay in the device slots
    def dev_real_space_async(self, part, nparts, d_force):
        self._check(self.lib.ewb_dev_real_space(self.h, int(part), int(nparts),
                                                d_force, None))

    def dev_kspace_finalize_peer(self, d_slot_ptrs, d_rho_out=None):
        """Sum the ranks' partial slots from their (peer) device pointers and
        finalise, in one kernel."""
        arr = (ctypes.c_void_p * len(d_slot_ptrs))(*[int(p) for p in d_slot_ptrs])
        self._check(self.lib.ewb_dev_kspace_finalize_peer(self.h, arr, len(d_slot_ptrs),
                                                          d_rho_out))

    def ipc_slots(self):
        """(device pointer, 64-byte IPC handle) of the handle's dedicated
        S(k) partial buffer."""
        ptr = _P()
        hd = (ctypes.c_ubyte * 64)()
        self._check(self.lib.ewb_ipc_slots(self.h, ctypes.byref(ptr), hd))
        return int(ptr.value), bytes(hd)

    def ipc_open(self, handle64):
        ptr = _P()
        hd = (ctypes.c_ubyte * 64).from_buffer_copy(handle64)
        self._check(self.lib.ewb_ipc_open(self.h, hd, ctypes.byref(ptr)))
        return int(ptr.value)

    def ipc_close(self, ptr):
        self._check(self.lib.ewb_ipc_close(self.h, _P(ptr)))

    def enable_peer_access(self, peer_device):
        self._check(self.lib.ewb_enable_peer_access(self.h, int(peer_device)))

    def dev_kspace_finalize_async(self, d_slots, d_rho_out=None):
        self._check(self.lib.ewb_dev_kspace_finalize(self.h, d_slots, d_rho_out,
                                                     None))

    def dev_self_energy_async(self):
        self._check(self.lib.ewb_dev_self_energy(self.h, None))

    def dev_energies(self, d_out3):
        self._check(self.lib.ewb_dev_energies(self.h, d_out3))

    def dev_status(self, d_out):
        self._check(self.lib.ewb_dev_status(self.h, d_out))

    def dev_check(self):
        self._check(self.lib.ewb_dev_check(self.h))

    def dev_evaluate(self, d_pos, d_q, n, d_force, d_rho_out=None,
                     timings=True):
        en = np.zeros(3)
        tm = np.zeros(4)
        self._check(self.lib.ewb_dev_evaluate(
            self.h, d_pos, d_q, int(n), d_force, d_rho_out, _ptr(en),
            _ptr(tm) if timings else None))
        return en, tm
