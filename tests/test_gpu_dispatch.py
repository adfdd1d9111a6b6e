"""Every least-squares kernel shape the dispatcher can pick (one warp per p,
multi-warp register kernels, the column-owner and blocked Householder kernels
for large real shapes, the CTA fallback), real and complex, up to the
limits (s <= 512 real / 256 complex, r <= 63), on random weighted affine
problems with repeated rows, against the CPU oracle."""
import numpy as np
import pytest
import scipy.sparse as sp

from oracle import online_ref
from paper_2510_04825_b200 import online
from paper_2510_04825_b200.offline import RowSelector, SnapshotBasis
from paper_2510_04825_b200.systems import ParametricSystem, const_term, interval, linear_term

pytestmark = pytest.mark.gpu

SHAPES = [  # (s, r, complex): every branch of launch_lsq, up to the plan limits
    (7, 6, False), (20, 8, False), (24, 11, False), (80, 20, False), (80, 23, False), (128, 11, False),
    (512, 11, False), (512, 23, False), (100, 31, False), (200, 30, False), (512, 31, False),
    (160, 40, False), (168, 47, False), (200, 50, False), (256, 55, False), (256, 63, False),
    (45, 40, False), (150, 41, False), (130, 44, False), (224, 49, False), (190, 52, False),
    (20, 8, True), (120, 8, True), (256, 11, True), (100, 31, True), (256, 40, True), (128, 63, True),
]


def _problem(s, r, complex_, seed):
    rng = np.random.default_rng(seed)
    n = max(3 * s, 4 * r)
    a0 = sp.random(n, n, density=4.0 / n, random_state=seed, format="csr") + sp.identity(n, format="csr") * 4.0
    a1 = sp.diags(rng.uniform(0.5, 1.5, n), format="csr")
    b = rng.standard_normal(n)
    if complex_:
        b = b + 1j * rng.standard_normal(n)
    q, _ = np.linalg.qr(rng.standard_normal((n, r)) + (1j * rng.standard_normal((n, r)) if complex_ else 0.0))
    system = ParametricSystem(n, interval(0.0, 1.0, imag=complex_), b,
                              affine_terms=(const_term(a0), linear_term(a1)), name="random")
    # with replacement (duplicate rows) as leverage sampling does, when s >> r
    idx = rng.choice(n, size=s, replace=s >= 3 * r)
    sel = RowSelector(indices=idx, n=n, weights=rng.uniform(0.5, 2.0, s))
    basis = SnapshotBasis(points=(), raw=q, basis=q, singular_values=np.ones(r))
    params = [1j * v for v in rng.uniform(0, 1, 6)] if complex_ else list(rng.uniform(0, 1, 6))
    return system, basis, sel, params


@pytest.mark.parametrize("s,r,complex_", SHAPES)
def test_lsq_shape_against_oracle(s, r, complex_):
    system, basis, sel, params = _problem(s, r, complex_, seed=s * 100 + r)
    plan = online.precompute_online(system, basis, sel)
    res = online.solve_params(plan, params)
    assert np.all(res.status == 0)
    blocks = online_ref.affine_blocks([t.matrix for t in system.affine_terms], basis.basis, sel.indices)
    for k, p in enumerate(params):
        m = online_ref.affine_combine([1.0, p], blocks)
        t = system.rhs(p, sel.indices)
        c, sres, _ = online_ref.solve_one(m, t, sel.weights)
        floor = online_ref.ls_floor(m, t, sel.weights, draws=2)
        d = np.linalg.norm(res.coefficients[k] - c) / np.linalg.norm(c)
        assert d <= max(1e-10, 10 * floor), (s, r, complex_, k, d, floor)
        assert res.sampled_residual[k] == pytest.approx(sres, rel=1e-8, abs=1e-12 * np.linalg.norm(t))


def test_limits_rejected():
    system, basis, sel, params = _problem(8, 8, False, 0)
    big = RowSelector(indices=np.arange(513, dtype=np.int64) % system.n, n=system.n)
    with pytest.raises(ValueError):
        online.precompute_online(system, basis, big)
    csys, cbasis, _, _ = _problem(130, 63, True, 1)
    with pytest.raises(ValueError):   # complex 256 x 64 exceeds the shared-memory budget
        online.precompute_online(csys, cbasis, RowSelector(indices=np.arange(256) % csys.n, n=csys.n))
    wide_q = np.linalg.qr(np.random.default_rng(0).standard_normal((system.n, 64)))[0] if system.n >= 64 else None
    if wide_q is not None:
        wide = SnapshotBasis(points=(), raw=wide_q, basis=wide_q, singular_values=np.ones(64))
        sel64 = RowSelector(indices=np.arange(70) % system.n, n=system.n)
        with pytest.raises(ValueError):
            online.precompute_online(system, wide, sel64)


@pytest.mark.parametrize("s,r", [(160, 40), (200, 50), (256, 55)])
def test_large_shapes_rank_deficient_and_nonfinite(s, r):
    # the column-owner (160x40, 200x50, 256x55) kernel reports the reference's
    # errors: a repeated basis column is rank-deficient (status 1, the repeated
    # column named, RankDeficiencyError from solve_batch), a NaN in a sampled
    # row is non-finite (status 2, ValueError)
    from paper_2510_04825_b200.errors import RankDeficiencyError
    system, basis, sel, params = _problem(s, r, False, seed=7)
    q = basis.basis.copy()
    q[:, r - 2] = q[:, 3]
    dup = SnapshotBasis(points=(), raw=q, basis=q, singular_values=np.ones(r))
    plan = online.precompute_online(system, dup, sel)
    res = online.solve_params(plan, params)
    assert np.all(res.status == 1) and np.all(res.bad_column == r - 2), (res.status, res.bad_column)
    assert np.all(np.isnan(res.coefficients))
    with pytest.raises(RankDeficiencyError):
        online.solve_batch(plan, params[:2])
    q = basis.basis.copy()
    q[sel.indices[s // 2], r // 2] = np.nan
    bad = SnapshotBasis(points=(), raw=q, basis=q, singular_values=np.ones(r))
    plan = online.precompute_online(system, bad, sel)
    res = online.solve_params(plan, params)
    assert np.all(res.status == 2)
    with pytest.raises(ValueError, match="non-finite"):
        online.solve_batch(plan, params[:2])
