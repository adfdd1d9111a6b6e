"""Offline snapshot solves on the GPU against the
reference's own full_solve (systems.py:187-222: SuperLU with up to two
refinement steps and the residual guard ||r|| <= 1e-10 (||A|| ||x|| + ||b||)).

The stencil systems of configs 3 and 5, wrapped in the reference's
ParametricSystem (matrix_fn = the harness row oracle, as
tests/golden/make_golden.py does), are solved at small grids by
  reference:  subapsnap.systems.full_solve                 (CPU, SuperLU)
  here:       offline._stencil_cg -> sas_cg_stencil          (GPU, fused CG kernels)
Both satisfy the guard, so the solutions differ by at most
cond(A) x (their two relative residuals); the test computes cond(A) exactly
(dense, small n) and requires that bound with a factor 4 of slack, plus the
guard on the GPU solution.  Skipped without the baseline/_ref install."""
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import online_ref
from paper_2510_04825_b200 import problems
from paper_2510_04825_b200.offline import _stencil_cg

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _ref():
    p = ROOT / "baseline" / "_ref"
    if not (p / "subapsnap" / "__init__.py").exists():
        pytest.skip("baseline/_ref (reference install) absent")
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))
    import subapsnap.systems
    return subapsnap


@pytest.mark.parametrize("cfg,kw", [(3, dict(grid=40)), (5, dict(grid=12)), (3, dict(grid=70))])
def test_gpu_cg_snapshot_matches_reference_full_solve(cfg, kw):
    ref = _ref()
    prob = problems.build(cfg, **kw)
    sysm = prob.system
    op = sysm.operator
    b = np.asarray(sysm.b)
    rs = ref.systems
    rsys = rs.ParametricSystem(sysm.n, rs.Domain(axes=tuple(rs.Axis(a.lo, a.hi, a.imag) for a in sysm.domain.axes)),
                               lambda p, idx: b[idx], row_fn=lambda p, idx: online_ref.stencil_rows(op, p, idx),
                               matrix_fn=lambda p: online_ref.stencil_rows(op, p, np.arange(op.n)), name=sysm.name)
    dev = torch.device("cuda:0")
    for p in prob.snapshot_points[:3]:
        x_ref = rs.full_solve(rsys, p)
        x_gpu = _stencil_cg(sysm, p, dev)
        a = rsys.matrix(p)
        ad = a.toarray()
        cond = np.linalg.cond(ad)
        fl = lambda x: np.linalg.norm(ad, "fro") * np.linalg.norm(x) + np.linalg.norm(b)  # noqa: E731
        r_gpu = np.linalg.norm(a @ x_gpu - b)
        r_ref = np.linalg.norm(a @ x_ref - b)
        assert r_gpu <= 1e-10 * fl(x_gpu)                       # the reference's guard on our solution
        bound = 4 * cond * (r_gpu + r_ref) / np.linalg.norm(b)
        rel = np.linalg.norm(x_gpu - x_ref) / np.linalg.norm(x_ref)
        assert rel <= max(bound, 1e-13), (cfg, p, rel, bound)


@pytest.mark.parametrize("grid", [60, 150])
def test_gpu_bicgstab_snapshot_matches_direct_solve(grid):
    """config 4's snapshot solver (k_bicg.cuh, sas_bicgstab_csr) against the
    reference's direct sparse solve with its residual guard (systems.py:187-222),
    complex non-symmetric A(p) = A0 + p I at small grids."""
    from paper_2510_04825_b200.offline import _affine_bicgstab, _sparse_solve
    prob = problems.convdiff_tf(grid=grid)
    s = prob.system
    for p in (1e-2j, 1.0j, 1e2j):
        x = _affine_bicgstab(s, p, "cuda:0")
        y = _sparse_solve(s.matrix(p), s.full_rhs(p), p)
        assert np.linalg.norm(x - y) <= 1e-10 * np.linalg.norm(y)
        x2 = _affine_bicgstab(s, p, "cuda:0")      # fixed-order reductions: same bits
        assert np.array_equal(x, x2)


def test_gpu_bicgstab_real_system():
    """The real-dtype instantiation on a real non-symmetric system."""
    import ctypes as C
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    from paper_2510_04825_b200 import _capi
    a = (problems.convdiff_matrix(50) + 3.0 * sp.identity(2500)).tocsr()
    a.sort_indices()
    rng = np.random.default_rng(2)
    b = rng.standard_normal(2500)
    up = lambda v: torch.from_numpy(np.ascontiguousarray(v)).cuda()
    rp, ci, va, d, bt = up(a.indptr.astype(np.int32)), up(a.indices.astype(np.int32)), up(a.data), up(a.diagonal()), up(b)
    x = torch.empty_like(bt)
    its, rn, xn = C.c_int32(0), C.c_double(0.0), C.c_double(0.0)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    _capi.check(_capi.load().sas_bicgstab_csr(2500, _capi.ptr(rp), _capi.ptr(ci), _capi.ptr(va), _capi.ptr(d),
                                              _capi.ptr(bt), _capi.ptr(x), _capi.SAS_F64, 1e-12, float(spla.norm(a)),
                                              5000, 10, 0, st, C.byref(its), C.byref(rn), C.byref(xn)), "bicgstab")
    y = spla.spsolve(a.tocsc(), b)
    xh = x.cpu().numpy()
    assert 0 < its.value < 5000
    assert np.linalg.norm(xh - y) <= 1e-9 * np.linalg.norm(y)
    assert abs(rn.value - np.linalg.norm(b - a @ xh)) <= 1e-12 * np.linalg.norm(b) + 1e-3 * rn.value
    assert abs(xn.value - np.linalg.norm(xh)) <= 1e-12 * np.linalg.norm(xh)


def test_gpu_bicgstab_residual_guard_raises():
    """A snapshot solve that has not converged raises the reference's NumericalError
    (full_solve's residual guard, systems.py:205-221) instead of returning x."""
    from paper_2510_04825_b200.errors import NumericalError
    from paper_2510_04825_b200.offline import _affine_bicgstab
    prob = problems.convdiff_tf(grid=60)
    with pytest.raises(NumericalError):
        _affine_bicgstab(prob.system, 1e-2j, "cuda:0", maxiter=3)
