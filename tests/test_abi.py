"""CPU checks of the C ABI: librgb.so loads, exports every symbol include/rgb.h
declares, and rejects invalid arguments before touching a device."""

import ctypes
import os
import re

import pytest

from paper_2106_11594_b200 import _build, _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    _build.build()
    return _lib.load()


def declared_symbols():
    text = open(os.path.join(ROOT, "include", "rgb.h")).read()
    return sorted(set(re.findall(r"^\s*(?:int64_t|int|void|const char \*)\s*(rgb_\w+)\s*\(", text, re.M)))


def test_header_declares_the_exports():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol(lib):
    for name in declared_symbols():
        assert hasattr(lib, name), name
    assert lib.rgb_abi_version() == _lib.RGB_ABI_VERSION


def test_struct_layouts_match_header():
    # rgb_config: int64 + 6 x int32 + 2 x double = 8 + 24 + 16
    assert ctypes.sizeof(_lib.Config) == 48
    assert ctypes.sizeof(_lib.State) == 7 * 8
    assert ctypes.sizeof(_lib.Logs) == 4 * 8


@pytest.mark.parametrize("field,value,needle", [
    ("m", 0, "num_regressors"),
    ("k", 0, "right-hand"),
    ("r_cap", 0, "r_cap"),
    ("variant", 7, "variant"),
    ("dtype", 9, "dtype"),
    ("eps_mode", 2, "eps"),
])
def test_invalid_config_is_rejected_without_a_device(lib, field, value, needle):
    cfg = _lib.Config(1, 4, 1, 4, _lib.F64, _lib.GENERAL, _lib.EPS_AUTO, 0.0, 1.0)
    setattr(cfg, field, value)
    st = _lib.State(*([ctypes.c_void_p(8)] * 7))
    rc = lib.rgb_ingest(ctypes.byref(cfg), ctypes.byref(st), ctypes.c_void_p(8), 0,
                        ctypes.c_void_p(8), 0, 1, None, None)
    assert rc == _lib.E_INVALID
    assert needle in lib.rgb_last_error().decode()
    with pytest.raises(ValueError):
        _lib.check(rc, "rgb_ingest")


def test_negative_fixed_eps_and_null_state(lib):
    cfg = _lib.Config(1, 4, 1, 4, _lib.F64, _lib.GENERAL, _lib.EPS_FIXED, -1.0, 1.0)
    st = _lib.State(*([ctypes.c_void_p(8)] * 7))
    assert lib.rgb_state_reset(ctypes.byref(cfg), ctypes.byref(st), None) == _lib.E_INVALID
    cfg.eps_value = 1e-8
    st.basis = None
    assert lib.rgb_state_reset(ctypes.byref(cfg), ctypes.byref(st), None) == _lib.E_INVALID
    assert "null" in lib.rgb_last_error().decode()


def test_memcpy_helper_validates_without_a_device(lib):
    assert lib.rgb_memcpy_async(None, None, 0, None) == _lib.OK
    assert lib.rgb_memcpy_async(ctypes.c_void_p(8), None, 16, None) == _lib.E_INVALID
    assert lib.rgb_memcpy_async(ctypes.c_void_p(8), ctypes.c_void_p(16), -1, None) == _lib.E_INVALID
    assert "rgb_memcpy_async" in lib.rgb_last_error().decode()


def test_product_has_no_oracle_dependency():
    pkg = os.path.join(ROOT, "paper_2106_11594_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                text = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in text and "from oracle" not in text, f
                assert "liborc" not in text, f


def test_compat_api_surface_matches_reference_names():
    import paper_2106_11594_b200 as p

    for name in ("RecursiveSolver", "EpsPolicy", "UpdateReport", "ProjectionResult", "VARIANTS",
                 "solve_batch", "PseudoinverseTracker", "CovarianceTracker", "pinv_from_scratch",
                 "FLOAT64", "RATIONAL", "CapabilityError", "ScalarKind"):
        assert hasattr(p, name), name
    assert p.VARIANTS == ("general", "orthogonal", "orthonormal")
    eps_m = p.FLOAT64.machine_epsilon
    assert p.EpsPolicy.auto().threshold(10, 3, eps_m) == (100 * 3 + 30 + 10) * eps_m
    with pytest.raises(ValueError):
        p.EpsPolicy.fixed(-1.0)


def test_constructor_validation_without_device():
    import paper_2106_11594_b200 as p

    with pytest.raises(ValueError):
        p.RecursiveSolver(0)
    with pytest.raises(ValueError):
        p.RecursiveSolver(2, variant="qr")
    with pytest.raises(ValueError):
        p.RecursiveSolver(2, eps=p.EpsPolicy.exact_zero())
    with pytest.raises(TypeError):
        p.RecursiveSolver(2, scalar="f64")
    with pytest.raises(p.CapabilityError):
        p.RecursiveSolver(2, variant="orthonormal", scalar=p.RATIONAL)


def test_plain_c_consumer_builds():
    """examples/rgb_demo.c uses only include/rgb.h and the CUDA runtime (no torch)."""
    from paper_2106_11594_b200 import _build

    assert os.path.exists(_build.build_demo(force=True))
