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
