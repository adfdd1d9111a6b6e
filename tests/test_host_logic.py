"""Host-side logic that needs no GPU: parameter marshalling, problem
definitions, the offline restatement (X, S) against the reference's own
outputs, plan artifacts, drop-in API surface."""
import dataclasses
import os
from pathlib import Path

import numpy as np
import pytest
import scipy.sparse as sp

from _golden import CFG_SIZES, load
from oracle import online_ref
from paper_2510_04825_b200 import offline, online, problems
from paper_2510_04825_b200.online import params_to_array

REF = Path(os.environ.get("SUBAPSNAP_REF", "/root/reference/pkg/src"))
needs_ref = pytest.mark.skipif(not (REF / "subapsnap").exists(), reason="reference not mounted")


def test_params_to_array_layouts():
    a = params_to_array([0.1, 0.2], 1, False)
    assert a.shape == (2, 1) and a.dtype == np.float64
    b = params_to_array([1j * 3.0, 2.0 + 1j], 1, True)
    assert b.shape == (2, 1, 2) and b[0, 0, 1] == 3.0 and b[1, 0, 0] == 2.0
    c = params_to_array([(0.1, 0.2, 0.3, 0.4)], 4, False)
    assert c.shape == (1, 4)
    with pytest.raises(ValueError):
        params_to_array([1j], 1, False)
    with pytest.raises(ValueError):
        params_to_array([(0.1, 0.2)], 4, False)
    assert params_to_array([], 3, False).shape == (0, 3)


@needs_ref
def test_snapshot_points_match_reference_layouts():
    import sys
    sys.path.insert(0, str(REF))
    from subapsnap import snapshot as rs
    from subapsnap import systems as rsys
    p1 = problems.reaction1d(n=50)
    ref = rs.default_snapshot_points(rsys.interval(0.0, 1.0), 10, "chebyshev")
    assert np.array_equal(np.array(p1.snapshot_points), np.array(ref))
    p2 = problems.gauss_krr(n=50)
    ref = rs.default_snapshot_points(rsys.interval(0.5, 2.0), 20, "log-spaced")
    assert np.array_equal(np.array(p2.snapshot_points), np.array(ref))
    p4 = problems.convdiff_tf(grid=5)
    ref = rs.default_snapshot_points(rsys.interval(1e-2, 1e2, imag=True), 30, "log-spaced")
    assert np.array_equal(np.array(p4.snapshot_points), np.array(ref))


def test_stencil_matrix_matches_oracle_rows():
    for prob, p in ((problems.diffusion2d(grid=9), (0.1, -0.2, 0.3, 0.05)),
                    (problems.diffusion3d(grid=5), (0.1, -0.2, 0.3, 0.05, 0.0, -0.1))):
        op = prob.system.operator
        a = prob.system.matrix(p)
        b = online_ref.stencil_rows(op, p, np.arange(op.n))
        assert abs(a - b).max() <= 1e-12 * abs(b).max()
        # symmetric positive definite (edge form of -div(a grad u))
        assert abs(a - a.T).max() <= 1e-12 * abs(a).max()
        # row sums of interior rows vanish only if all neighbours are interior
        nbr, _ = op.edges(np.arange(op.n))
        interior = np.all(nbr >= 0, axis=1)
        rs = np.asarray(a.sum(axis=1)).ravel()
        assert np.all(np.abs(rs[interior]) <= 1e-9 * abs(a).max())


def test_convdiff_matrix_definition():
    g = 4
    m = problems.convdiff_matrix(g)
    h = 1.0 / (g + 1)
    # interior node (1,1): diag -4/h^2 - 100/h; backward neighbours 1/h^2 + 50/h; forward 1/h^2
    k = 1 * g + 1
    row = m.getrow(k).toarray().ravel()
    assert row[k] == pytest.approx(-4 / h**2 - 100 / h)
    assert row[k - g] == pytest.approx(1 / h**2 + 50 / h)
    assert row[k - 1] == pytest.approx(1 / h**2 + 50 / h)
    assert row[k + g] == pytest.approx(1 / h**2)
    assert row[k + 1] == pytest.approx(1 / h**2)


@pytest.mark.parametrize("name", ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5"])
def test_offline_selector_restatement_matches_reference(name):
    """offline.select_rows (leverage) reproduces the reference's S and weights
    from the same X (subsample.py:95-156 via cli.build_offline)."""
    case = load(name)
    cfg = int(name[3:])
    prob = problems.build(cfg, **CFG_SIZES[cfg])
    anchor = offline.choose_anchor(prob.snapshot_points)
    X = case.basis.basis
    if cfg == 2:
        op = prob.system.operator
        b_anchor = online_ref.gauss_rows(op.points, np.arange(op.n), float(anchor), op.ridge) @ X
    elif cfg in (3, 5):
        b_anchor = online_ref.stencil_rows(prob.system.operator, anchor, np.arange(prob.system.n)) @ X
    else:
        # the reference coerces affine coefficients to complex (systems.py:92, 98)
        out = None
        for t in prob.system.affine_terms:
            f = complex(t.scale) if t.kind == "const" else complex(t.scale) * anchor
            blk = t.matrix * f
            out = blk if out is None else out + blk
        b_anchor = np.asarray(sp.csr_matrix(out) @ X)
    sel = offline.select_rows(b_anchor, prob.system.full_rhs(anchor), strategy="leverage",
                              oversample=prob.samples / (X.shape[1] + 1), seed=prob.selector_seed)
    assert sel.size == prob.samples
    assert np.array_equal(sel.indices, case.data["S"])
    assert np.allclose(sel.weights, case.data["w"], rtol=1e-12)


def test_orthonormalize_modes():
    rng = np.random.default_rng(0)
    raw = rng.standard_normal((200, 6)) @ np.diag([1, 1e-2, 1e-5, 1e-9, 1e-14, 1e-15])
    q, sig = offline.orthonormalize(raw, ("pod", 1e-13))
    assert q.shape[1] == 4
    assert np.allclose(q.T @ q, np.eye(4), atol=1e-12)
    with pytest.raises(Exception):
        offline.orthonormalize(raw, "qr")
    q2, _ = offline.orthonormalize(raw[:, :3], "qr")
    assert np.allclose(q2.T @ q2, np.eye(3), atol=1e-12)


def test_plan_artifact_layout(tmp_path):
    """save_plan writes the reference's npz keys (online.py:168-178)."""
    case = load("cfg4")
    blocks = online_ref.affine_blocks([t.matrix for t in case.system.affine_terms], case.basis.basis,
                                      case.selector.indices)
    plan = online.OnlinePlan(system=case.system, basis=case.basis, selector=case.selector, blocks=blocks,
                             sampled_basis=case.basis.basis[case.selector.indices],
                             output_projection=case.system.output_functional @ case.basis.basis)
    path = tmp_path / "plan.npz"
    online.save_plan(path, plan)
    data = np.load(path)
    assert set(data.files) == {"sampled_basis", "affine", "block_0", "block_1", "output_projection"}
    assert bool(data["affine"])
    assert np.array_equal(data["block_1"], blocks[1])


def test_snapshot_and_selector_artifacts_roundtrip(tmp_path):
    case = load("cfg1")
    b = offline.SnapshotBasis(points=(0.1, 0.5), raw=case.basis.basis, basis=case.basis.basis,
                              singular_values=np.ones(2))
    offline.save_snapshot(tmp_path / "s.npz", b)
    back = offline.load_snapshot(tmp_path / "s.npz")
    assert back.points == (0.1, 0.5) and np.array_equal(back.basis, b.basis)
    offline.save_selector(tmp_path / "sel.json", case.selector)
    sel = offline.load_selector(tmp_path / "sel.json")
    assert np.array_equal(sel.indices, case.selector.indices)
    assert np.array_equal(sel.weights, case.selector.weights)


@needs_ref
def test_dropin_surface_matches_reference():
    """Same public names and dataclass fields as subapsnap.online."""
    import sys
    sys.path.insert(0, str(REF))
    from subapsnap import online as ro
    for name in ("precompute_online", "solve_online", "solve_batch", "estimate_residual", "save_plan",
                 "load_plan", "OnlinePlan", "OnlineSolution", "BatchRow"):
        assert hasattr(online, name), name
    ref_fields = [f.name for f in dataclasses.fields(ro.OnlinePlan)]
    ours = [f.name for f in dataclasses.fields(online.OnlinePlan)]
    assert ours[:len(ref_fields)] == ref_fields
    assert [f.name for f in dataclasses.fields(online.BatchRow)] == [f.name for f in dataclasses.fields(ro.BatchRow)]
    ref_sol = [f.name for f in dataclasses.fields(ro.OnlineSolution)]
    assert [f.name for f in dataclasses.fields(online.OnlineSolution)][:len(ref_sol)] == ref_sol
    import inspect
    for fn in ("precompute_online", "solve_online", "solve_batch", "estimate_residual"):
        ra = list(inspect.signature(getattr(ro, fn)).parameters)
        oa = list(inspect.signature(getattr(online, fn)).parameters)
        assert oa[:len(ra)] == ra, fn


def test_estimate_residual_formula():
    case = load("tridiag_leverage")
    plan = online.OnlinePlan(system=case.system, basis=case.basis, selector=case.selector, blocks=None,
                             sampled_basis=None, output_projection=None)
    sol = online.OnlineSolution(parameter=-9.5, coefficients=np.zeros(case.basis.rank), sampled_residual=2.0)
    est, lo, hi, eps = online.estimate_residual(plan, sol)
    r, s = case.basis.rank, case.selector.size
    assert eps == pytest.approx(min(r * np.log(r) / s, 0.99))
    assert lo == pytest.approx(2.0 / (1 + eps)) and hi == pytest.approx(2.0 / (1 - eps))
    unweighted = dataclasses.replace(case.selector, weights=None)
    plan2 = dataclasses.replace(plan, selector=unweighted)
    with pytest.raises(ValueError):
        online.estimate_residual(plan2, sol)


def test_precompute_spot_check_raises_on_inconsistent_blocks():
    """The reference's plan check (online.py:86-96): affine blocks that disagree with the
    system's row oracle at basis.points[0] by more than 1e-10 raise RankDeficiencyError
    (before any device plan is built); consistent ones pass the same check."""
    from paper_2510_04825_b200.errors import RankDeficiencyError
    case = load("tridiag_lupp")
    system, basis, sel = case.system, case.basis, case.selector
    idx = np.asarray(sel.indices, dtype=np.int64)
    uniq, inverse = np.unique(idx, return_inverse=True)
    blocks = tuple(online._rows_times_basis(t.matrix[uniq], basis.basis)[inverse] for t in system.affine_terms)
    online._spot_check(system, basis, idx, uniq, inverse, blocks)          # consistent: no error

    class Skewed:
        """Same affine terms, but a row oracle that is off by 1e-6 relative."""
        def __init__(self, inner):
            self._inner = inner
        def __getattr__(self, name):
            return getattr(self._inner, name)
        def rows(self, p, rows):
            m = sp.csr_matrix(self._inner.matrix(p))[np.asarray(rows)]
            return m * (1.0 + 1e-6)

    with pytest.raises(RankDeficiencyError, match="disagree with row oracle"):
        online.precompute_online(Skewed(system), basis, sel)
