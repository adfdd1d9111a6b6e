"""The C-ABI library loads and exports every symbol include/*.h declares;
host-side helpers of the kernels (no GPU needed)."""
import re
from pathlib import Path

import numpy as np
import pytest

from paper_2510_04825_b200 import _capi

ROOT = Path(__file__).resolve().parents[1]


def _declared():
    names = set()
    for h in (ROOT / "include").glob("*.h"):
        txt = re.sub(r"/\*.*?\*/", "", h.read_text(), flags=re.S)
        for m in re.finditer(r"^\s*[A-Za-z_][\w\s\*]*?\b(sas_\w+)\s*\(", txt, flags=re.M):
            names.add(m.group(1))
    return names


def test_library_exports_every_declared_symbol():
    lib = _capi.load()
    declared = _declared()
    assert {"sas_plan_create", "sas_solve", "sas_solve_host", "sas_lift", "sas_residual"} <= declared
    for name in declared:
        assert hasattr(lib, name), name
    assert set(_capi.EXPORTS) | set(_capi.DEBUG_EXPORTS) >= declared


def test_version_and_error_plumbing():
    lib = _capi.load()
    assert b"sm_100a" in lib.sas_version()
    # argument errors are reported without touching a GPU
    import ctypes as C
    h = C.c_void_p()
    rc = lib.sas_plan_create(None, None, 0, 0, None, None, 0, None, None, 0, 0, C.byref(h))
    assert rc == _capi.SAS_ERR_ARG
    assert "null" in _capi.last_error()


def test_host_exp_matches_libm():
    lib = _capi.load()
    rng = np.random.default_rng(0)
    xs = np.concatenate([-rng.uniform(0, 40, 4000), -rng.uniform(0, 708, 2000), -rng.uniform(0, 1, 2000),
                         [0.0, -0.0, -1e-300, -708.3]])
    got = np.array([lib.sas_debug_exp64_host(float(x)) for x in xs])
    ref = np.exp(xs)
    # K3 only evaluates x <= 0 (the Gaussian kernel's argument); the argument
    # is rounded once in table units (|x| eps relative, as the
    # reference's own rounding of x = -D*inv), the rest is <= 2 ulp
    rel = np.abs(got - ref) / ref
    assert np.all(rel <= 4.5e-16 + 2.5e-16 * np.abs(xs)), (rel / (4.5e-16 + 2.5e-16 * np.abs(xs))).max()
    assert lib.sas_debug_exp64_host(-800.0) == 0.0
    assert lib.sas_debug_exp64_host(0.0) == 1.0
