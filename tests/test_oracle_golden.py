"""Pin the CPU oracle (oracle/online_ref.py) against the golden vectors the
unmodified reference produced (tests/golden/make_golden.py)."""
import numpy as np
import pytest

from _golden import GOLDEN_NAMES, full_matrix, load, oracle_solve
from oracle import online_ref


@pytest.mark.parametrize("name", GOLDEN_NAMES)
def test_oracle_matches_reference(name):
    case = load(name)
    d = case.data
    n_check = min(len(case.params), 24)
    for k in range(n_check):
        p = case.params[k]
        coef, sres, out = oracle_solve(case, p)
        ref = d["coef"][k]
        # same numpy/LAPACK calls as the reference: agreement at the rounding level
        # (the krr rows come from the reference's numba rbf_rows, whose exp can
        # differ from numpy's by an ulp, so residuals at the rounding floor are
        # compared absolutely)
        tol = max(1e-13, 2.0 * float(d["floor"][k]))
        assert np.linalg.norm(coef - ref) <= tol * np.linalg.norm(ref), (name, k)
        t = case.system.rhs(p, case.selector.indices)
        wt = np.linalg.norm(t * case.selector.weights if case.selector.weights is not None else t)
        assert abs(sres - d["sres"][k]) <= 1e-12 * abs(d["sres"][k]) + 1e3 * np.finfo(float).eps * wt, (name, k)
        if out is not None:
            assert abs(out - d["outv"][k]) <= 1e-13 * abs(d["outv"][k]) + 1e-300


@pytest.mark.parametrize("name", ["cfg1", "cfg3", "cfg4", "tridiag_leverage"])
def test_oracle_relres_matches_reference(name):
    case = load(name)
    d = case.data
    for k in range(0, len(case.params), max(1, len(case.params) // 6)):
        p = case.params[k]
        coef = d["coef"][k]
        x = case.basis.basis @ coef
        rr = online_ref.relative_residual(full_matrix(case, p), x, case.system.full_rhs(p))
        assert rr == pytest.approx(d["relres"][k], rel=1e-6, abs=1e-15)


def test_ls_matches_lstsq():
    # linalg.solve_ls vs np.linalg.lstsq (test_linalg.py:45-62)
    rng = np.random.default_rng(3)
    for _ in range(20):
        a = rng.standard_normal((50, 7))
        b = rng.standard_normal(50)
        w = rng.uniform(0.5, 2.0, 50)
        x = online_ref.solve_ls(a, b, weights=w)
        ref = np.linalg.lstsq(a * w[:, None], b * w, rcond=None)[0]
        assert np.allclose(x, ref, atol=1e-10)


def test_ls_rank_deficient():
    a = np.zeros((10, 3))
    a[:, 0] = 1.0
    a[:, 1] = 2.0
    a[:, 2] = np.arange(10)
    with pytest.raises(online_ref.OracleRankDeficiency):
        online_ref.solve_ls(a, np.ones(10))
