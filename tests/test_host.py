"""Host-side logic (CPU only): the C-ABI library loads and exports every
symbol of include/ewald_b200.h; the reference-facing set-up functions
(choose_parameters, enumerate_kvectors, ReciprocalSpace) reproduce the
reference; device entry points fail loudly without a GPU."""

import math
import os
import re

import numpy as np
import pytest

from conftest import ROOT, golden


def header_symbols():
    src = open(os.path.join(ROOT, "include", "ewald_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ewb_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_header_symbol():
    import ctypes
    from paper_1708_01135_b200 import _lib
    lib = ctypes.CDLL(_lib.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} missing from {_lib.LIB_PATH}"
    assert set(syms) == set(_lib.SIGNATURES), "ctypes table out of sync"
    assert lib.ewb_version() >= 100


def test_library_is_sm100a():
    import subprocess
    from paper_1708_01135_b200 import _lib
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf",
                          _lib.LIB_PATH], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


def test_no_device_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is present")
    import paper_1708_01135_b200 as ew
    from paper_1708_01135_b200 import _lib
    with pytest.raises(_lib.DeviceError):
        _lib.Handle(0)
    box = ew.SimulationBox(10.0)
    ps = ew.create_particle_set(2, box)
    ps.charge[:] = (1.0, -1.0)
    ps.position[1, 0] = 2.0
    with pytest.raises(RuntimeError):
        ew.total_coulomb(ps, ew.choose_parameters(2, box, 1e-4))


def test_product_never_imports_oracle():
    pkg = os.path.join(ROOT, "paper_1708_01135_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".c", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "oracle" not in re.sub(r"#.*|\"\"\".*?\"\"\"", "", txt, flags=re.S) \
                    or f == "__init__.py", f"{f} references the oracle"


def test_choose_parameters_mirror():
    import paper_1708_01135_b200 as ew
    box = ew.SimulationBox(30.0)
    p = ew.choose_parameters(1728, box, 1e-6)
    assert 0.5 * 0.062 < p.alpha < 2.0 * 0.062
    assert p.r_cutoff <= 15.0
    p = ew.choose_parameters(32768, ew.SimulationBox(80.0), 1e-6, r_cutoff=19.0)
    assert p.r_cutoff == 19.0
    assert p.alpha == pytest.approx(0.0383, abs=2e-4)
    p = ew.choose_parameters(64, ew.SimulationBox(10.0), 1e-6)
    assert p.r_cutoff == 5.0
    with pytest.raises(ew.BoxTooSmallError):
        ew.choose_parameters(2, ew.SimulationBox(0.1), 1e-6)
    with pytest.raises(ValueError):
        ew.choose_parameters(2, box, 1e-6, alpha=0.1, r_cutoff=5.0)


def test_enumerate_kvectors_matches_reference_tables():
    import paper_1708_01135_b200 as ew
    box = ew.SimulationBox(2.0 * math.pi)
    rs = ew.enumerate_kvectors(box, ew.EwaldParams(1e12, 1.0, 1.5, 1e-6))
    assert rs.count == 18
    unit = np.isclose(np.linalg.norm(rs.kvec, axis=1), 1.0)
    np.testing.assert_allclose(rs.coeff[unit], 1.0 / (2.0 * math.pi**2), rtol=1e-12)
    for name in ("rand32_s21", "rand64_s5", "rand200_s7", "rocksalt8"):
        g = golden(name)
        b = ew.SimulationBox(float(g["L"]))
        p = ew.EwaldParams(float(g["alpha"]), float(g["r_cutoff"]),
                           float(g["k_cutoff"]), float(g["tolerance"]))
        rs = ew.enumerate_kvectors(b, p)
        np.testing.assert_array_equal(rs.m_int, g["m_int"])
        np.testing.assert_allclose(rs.coeff, g["coeff"], rtol=1e-15)


def test_cube_table_counts():
    from paper_1708_01135_b200 import workloads as wl
    for n, k in ((8, 2456), (18, 25326), (35, 178955), (21, 39753), (55, 683815)):
        assert wl.cube_half_m(n).shape[0] == k == ((2 * n + 1) ** 3 - 1) // 2


def test_neutral_gas_charges_exact():
    from paper_1708_01135_b200 import workloads as wl
    for seed in range(4):
        q = wl.neutral_gaussian_charges(131072, seed)
        assert float(np.sum(q)) == 0.0
        assert float(np.sum(q[::-1])) == 0.0


def test_hardcore_gas_min_separation():
    from paper_1708_01135_b200 import workloads as wl
    pos = wl.hardcore_gas_positions(2000, 15.0, 0.8, seed=1)
    d = pos[:, None, :] - pos[None, :, :]
    d -= 15.0 * np.floor(d / 15.0 + 0.5)
    r2 = np.einsum("ijk,ijk->ij", d, d)
    np.fill_diagonal(r2, np.inf)
    assert r2.min() >= 0.64
    assert pos.min() >= 0.0 and pos.max() < 15.0


def test_pinned_zeros_falls_back_to_numpy_without_a_device():
    from paper_1708_01135_b200 import _lib
    a = _lib.pinned_zeros(1000)
    assert a.shape == (1000,) and a.dtype == np.float64 and not a.any()
    a[:] = 1.5
    assert float(a.sum()) == 1500.0
    assert _lib.pinned_zeros(0).shape == (0,)


REF_SRC = "/root/reference/pkg/src"


def _reference_core():
    """ewaldmd.core of the reference (this container only; the GPU box has
    no /root/reference)."""
    import importlib
    import sys
    if not os.path.isdir(os.path.join(REF_SRC, "ewaldmd")):
        pytest.skip("reference package not present")
    if REF_SRC not in sys.path:
        sys.path.append(REF_SRC)
    try:
        return importlib.import_module("ewaldmd.core")
    except Exception as e:  # numba or another dependency missing
        pytest.skip(f"reference not importable: {e}")


def test_registered_reference_errors_are_raised():
    """After set_error_types(ewaldmd.core) every error the facade raises is an
    instance of the reference's class of the same name (so verify.py:141-153's
    ``except NeutralityError`` catches it) and of this package's own."""
    import paper_1708_01135_b200 as ew
    from paper_1708_01135_b200 import _lib
    from paper_1708_01135_b200.core import set_error_types
    ref = _reference_core()
    set_error_types(ref)
    try:
        # neutrality: host check with the reference's expression, on the
        # reference's own ParticleSet
        ps = ref.create_particle_set(2, ref.SimulationBox(10.0))
        ps.charge[:] = 1.0
        with pytest.raises(ref.NeutralityError) as ei:
            ew.core.require_neutral(ps)
        assert isinstance(ei.value, ew.NeutralityError)
        # device statuses (ewald.py:212-213 coincident; celllist.py:84-88)
        for st, name in ((_lib.EWB_ECOINCIDENT, "CoincidentParticlesError"),
                         (_lib.EWB_ECUTOFF, "CutoffTooLargeError"),
                         (_lib.EWB_EKSPACE, "KSpaceEmptyError"),
                         (_lib.EWB_EBOX, "BoxTooSmallError"),
                         (_lib.EWB_ESIZE, "OracleSizeError")):
            with pytest.raises(getattr(ref, name)) as ei:
                _lib.raise_for(st, "x")
            assert isinstance(ei.value, getattr(ew, name))
            assert isinstance(ei.value, ref.EwaldmdError)
        # host-side parameter errors
        with pytest.raises(ref.KSpaceEmptyError):
            ew.enumerate_kvectors(ew.SimulationBox(10.0), ew.EwaldParams(0.5, 4.0, 0.1, 1e-6))
    finally:
        set_error_types(None)
    with pytest.raises(ew.CoincidentParticlesError) as ei:
        _lib.raise_for(_lib.EWB_ECOINCIDENT, "x")
    assert not isinstance(ei.value, ref.EwaldmdError)


def test_workers_resolution(monkeypatch):
    """workers = GPU count; capped at the visible GPUs unless
    ranks may share a device."""
    import torch
    from paper_1708_01135_b200 import distributed as d
    monkeypatch.setattr(torch.cuda, "is_available", lambda: True)
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 2)
    monkeypatch.delenv("EWALDB200_WORKERS", raising=False)
    monkeypatch.delenv("EWALDB200_SHARE_DEVICES", raising=False)
    assert d._resolve_devices(None) == [0]
    assert d._resolve_devices(0) == [0, 1]
    assert d._resolve_devices(8) == [0, 1]
    monkeypatch.setenv("EWALDB200_SHARE_DEVICES", "1")
    assert d._resolve_devices(3) == [0, 1, 0]
    monkeypatch.setenv("EWALDB200_WORKERS", "2")
    assert d._resolve_devices(None) == [0, 1]
    with pytest.raises(ValueError):
        d._resolve_devices(-1)


def test_reference_arm_json_contract():
    """bench.py --impl reference (the oracle port on host cores) prints ONE
    JSON line with the driver's keys, the same config dict and warm-up as
    our arm, and exits 0; on c1 it runs in seconds without a GPU."""
    import json
    import subprocess
    import sys
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference",
                          "--config", "c1", "--steps", "2", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.strip().startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step",
              "higher_is_better", "scaling", "vs_baseline", "dtype", "data", "config",
              "impl", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["steps"] == 2 and d["warmup"] == 3
    assert d["value"] > 0 and d["e2e"]["value"] == d["value"]
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "port" and d["cpu_baseline"]["cores"] >= 1
    assert d["config"]["parallelism"] == "single GPU" and d["config"]["n_particles"] == 1000


def test_host_pins_policy(monkeypatch):
    """_lib.HostPins: an owning, contiguous, large array is registered on its
    second sighting and unregistered when it dies; views, small arrays and
    non-owning arrays are never registered (the C calls are faked)."""
    import gc
    from paper_1708_01135_b200 import _lib
    calls = []

    class FakeLib:
        def ewb_host_register(self, p, n):
            calls.append(("reg", p.value, n))
            return 0

        def ewb_host_unregister(self, p):
            calls.append(("unreg", p.value))
            return 0
    monkeypatch.setattr(_lib, "load_library", lambda: FakeLib())
    pins = _lib.HostPins()
    a = np.zeros((1 << 16, 3))
    pins.touch(a)
    assert calls == []                      # first sighting: remembered only
    pins.touch(a)
    assert calls == [("reg", a.ctypes.data, a.nbytes)]
    pins.touch(a)
    assert len(calls) == 1                  # already pinned
    pins.touch(a[::2])                      # a view
    pins.touch(a[:10])
    pins.touch(np.zeros(16))                # small
    pins.touch(np.zeros(16))
    assert len(calls) == 1
    ptr = a.ctypes.data
    del a
    gc.collect()
    assert calls[-1] == ("unreg", ptr)
    assert not pins._pinned


def test_set_error_types_reset_and_partial_namespace():
    """A namespace may define only some of the classes; None restores the
    package's own classes."""
    import types
    import paper_1708_01135_b200 as ew
    from paper_1708_01135_b200 import _lib
    Mine = type("CoincidentParticlesError", (Exception,), {})
    ew.set_error_types(types.SimpleNamespace(CoincidentParticlesError=Mine))
    try:
        with pytest.raises(Mine):
            _lib.raise_for(_lib.EWB_ECOINCIDENT, "x")
        with pytest.raises(ew.KSpaceEmptyError) as ei:
            _lib.raise_for(_lib.EWB_EKSPACE, "x")
        assert type(ei.value) is ew.KSpaceEmptyError
    finally:
        ew.set_error_types(None)
    with pytest.raises(ew.CoincidentParticlesError) as ei:
        _lib.raise_for(_lib.EWB_ECOINCIDENT, "x")
    assert type(ei.value) is ew.CoincidentParticlesError
