"""Pins of the harness row oracles against the reference's own code (CPU).

The BASELINE stencil configs (3, 5) have no generator in the reference
(SURVEY.md §0.4); their row oracle oracle/online_ref.stencil_rows (and the
device assembler K2 behind it) restates the reference's edge-midpoint
finite-difference matrix _conductivity_matrix (systems.py:306-334): node
(i, j) -> i*g + j, edges (+x, -x, +y, -y), c_e = sigma(mid_e) / h^2,
diagonal = sum_e c_e, off-diagonal -c_e for interior neighbours.  The
reference builds it on [-1, 1]^2 (h_ref = 2/(g+1)), the harness on [0, 1]^2
(h = 1/(g+1)), so with sigma_ref(x, y) = a((x+1)/2, (y+1)/2) the two matrices
differ by the factor h_ref^2 / h^2 = 4 exactly (up to the rounding of the
mid-point coordinates)."""
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import online_ref
from paper_2510_04825_b200 import problems

ROOT = Path(__file__).resolve().parents[1]


def _ref_systems():
    for p in (ROOT / "baseline" / "_ref", Path("/root/reference/pkg/src")):
        if (p / "subapsnap" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            import subapsnap.systems
            return subapsnap.systems
    pytest.skip("reference not importable here")


@pytest.mark.parametrize("grid", [7, 16])
def test_stencil_rows_equal_reference_conductivity_matrix(grid):
    rs = _ref_systems()
    prob = problems.diffusion2d(grid=grid)
    op = prob.system.operator
    rng = np.random.default_rng(3)
    for _ in range(3):
        p = tuple(rng.uniform(-0.5, 0.5, 4))

        def sigma(x, y):
            u, v = (x + 1.0) / 2.0, (y + 1.0) / 2.0
            phi = [np.sin((k * np.pi) * u) * np.sin((k * np.pi) * v) for k in range(1, 5)]
            arg = phi[0] * p[0]
            for k in range(1, 4):
                arg = arg + phi[k] * p[k]
            return float(np.exp(arg))

        want = rs._conductivity_matrix(grid, sigma).toarray()
        got = online_ref.stencil_rows(op, p, np.arange(op.n)).toarray() / 4.0
        assert np.array_equal(got != 0, want != 0)           # same sparsity: boundary edges drop out
        np.testing.assert_allclose(got, want, rtol=1e-13, atol=0)


def test_stencil_rows_constant_coefficient_is_reference_laplacian():
    """p = 0: a = 1, the reference's heat2d base matrix (systems.py:337-351) up to the factor 4."""
    rs = _ref_systems()
    g = 9
    op = problems.diffusion2d(grid=g).system.operator
    want = rs._conductivity_matrix(g, lambda x, y: 1.0).toarray()
    got = online_ref.stencil_rows(op, (0.0, 0.0, 0.0, 0.0), np.arange(op.n)).toarray() / 4.0
    np.testing.assert_allclose(got, want, rtol=1e-15, atol=0)
