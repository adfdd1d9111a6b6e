"""The drop-in fed with the reference's OWN objects, side by side with the
reference's own online phase.

For the reference's test systems (systems.build_problem: tridiag with its
p-dependent right-hand side, heat2d, convdiff with its output functional,
delay with its opaque -exp(tau p) coefficient, krr with p = (lambda, sigma)
and the numba rbf_rows oracle) the reference builds the snapshot basis
(snapshot.build_snapshot) and the selector (subsample.select_rows) exactly as
cli.build_offline does; then

  reference:  subapsnap.online.precompute_online + solve_batch   (CPU)
  drop-in:    paper_2510_04825_b200.online.precompute_online + solve_batch
              on the SAME SnapshotBasis / RowSelector / ParametricSystem objects (GPU)

must agree per parameter: coefficients within max(1e-10, 10 floor_p), the
sampled residual, the residual interval and the output value.  The reference
comes from baseline/_ref (a pip install of /root/reference that travels with
the repository); the test is skipped when that install is absent."""
import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import online_ref
from paper_2510_04825_b200 import online as gpu_online

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu
EPS = np.finfo(float).eps


def _ref():
    p = ROOT / "baseline" / "_ref"
    if not (p / "subapsnap" / "__init__.py").exists():
        pytest.skip("baseline/_ref (reference install) absent")
    if str(p) not in sys.path:
        sys.path.insert(0, str(p))
    import subapsnap.online
    import subapsnap.snapshot
    import subapsnap.subsample
    import subapsnap.systems
    return subapsnap


SPECS = {
    "tridiag": ({"n": 400}, 8, "equispaced", "qr", 4.0, lambda rng: list(rng.uniform(-10.0, -9.0, 40))),
    "heat2d": ({"grid": 30}, 8, "equispaced", "qr", 4.0, lambda rng: list(rng.uniform(0.0, 5.0, 40))),
    "convdiff": ({"grid": 20}, 10, "log-spaced", ("pod", 1e-12), 4.0,
                 lambda rng: list(1j * 10 ** rng.uniform(0.0, 6.0, 40))),
    "delay": ({"n": 300}, 8, "log-spaced", ("pod", 1e-12), 4.0,
              lambda rng: list(1j * 10 ** rng.uniform(0.0, 4.0, 40))),
    "krr": ({"n_train": 400, "n_test": 10}, None, None, "qr", 4.0,
            lambda rng: [(float(10 ** rng.uniform(-3, 1)), float(rng.uniform(1.0, 9.0))) for _ in range(40)]),
}


def _offline(ref, kind):
    params, r, layout, mode, ovs, make = SPECS[kind]
    rsys = ref.systems.build_problem(ref.systems.ProblemSpec(kind, params))
    if kind == "krr":
        pts = [(1e-3, 1.0), (1e-2, 2.0), (1e-1, 3.0), (1.0, 6.0), (10.0, 9.0)]
    else:
        pts = ref.snapshot.default_snapshot_points(rsys.domain, r, layout)
    try:
        basis = ref.snapshot.build_snapshot(rsys, pts, mode=mode)
    except ref.errors.RankDeficiencyError:
        basis = ref.snapshot.build_snapshot(rsys, pts, mode=("pod", 1e-13))
    anchor = ref.subsample.choose_anchor(pts)
    b_anchor = np.asarray(rsys.matrix(anchor) @ basis.basis)
    cfg = ref.subsample.SelectorConfig(strategy="leverage", oversample=ovs, seed=0)
    sel = ref.subsample.select_rows(b_anchor, rsys.full_rhs(anchor), cfg, anchors=(anchor,))
    return rsys, basis, sel, make(np.random.default_rng(11))


@pytest.mark.parametrize("kind", sorted(SPECS))
def test_reference_objects_through_dropin(kind):
    ref = _ref()
    import subapsnap.errors  # noqa: F401
    rsys, basis, sel, params = _offline(ref, kind)
    rplan = ref.online.precompute_online(rsys, basis, sel)
    want = ref.online.solve_batch(rplan, params, want_interval=True)
    plan = gpu_online.precompute_online(rsys, basis, sel)
    got = gpu_online.solve_batch(plan, params, want_interval=True)
    assert len(got) == len(want)
    worst = 0.0
    for k, (g, w) in enumerate(zip(got, want)):
        assert g.parameter == w.parameter
        c_ref = w.solution.coefficients
        # per-p floor: the spread of the reference's own least squares under 1-ulp perturbations of M
        if rplan.affine:
            m = sum(t.coeff(params[k]) * blk for t, blk in zip(rsys.affine_terms, rplan.blocks))
        else:
            m = ref.online._sampled_rows(rsys, basis, sel.indices, params[k])
        t = rsys.rhs(params[k], sel.indices)
        floor = online_ref.ls_floor(m, t, sel.weights, draws=2)
        dc = g.solution.coefficients - c_ref
        d = np.linalg.norm(dc) / np.linalg.norm(c_ref)
        worst = max(worst, d)
        assert d <= max(1e-10, 10 * floor), (kind, k, d, floor)
        # the sampled residual ||W (M c - t)|| moves by at most ||W M dc|| plus rounding
        wv = sel.weights if sel.weights is not None else np.ones(sel.size)
        tol_r = (np.linalg.norm(wv * (m @ dc))
                 + 1e3 * EPS * (np.linalg.norm(wv[:, None] * m) * np.linalg.norm(c_ref) + np.linalg.norm(wv * t)))
        assert abs(g.sampled_residual - w.sampled_residual) <= tol_r, (kind, k, g.sampled_residual,
                                                                       w.sampled_residual, tol_r)
        assert (g.residual_interval is None) == (w.residual_interval is None)
        if w.residual_interval is not None:   # est / (1 +- eps): the same factors on both sides
            assert np.allclose(np.array(g.residual_interval) / g.sampled_residual,
                               np.array(w.residual_interval) / w.sampled_residual, rtol=1e-14)
        if w.output_value is None:
            assert g.output_value is None
        else:
            assert abs(g.output_value - w.output_value) <= max(1e-10, 10 * floor) * abs(w.output_value) + 1e-300
        assert np.asarray(g.solution.coefficients).dtype == np.asarray(c_ref).dtype
    print(f"\n{kind}: n={rsys.n} r'={basis.rank} s={sel.size}: max coefficient rel diff {worst:.2e}")
    # the drop-in's lift is the reference's lift (x = Q_X c) on the GPU
    x = got[0].solution.lift()
    assert np.allclose(x, want[0].solution.lift(), rtol=1e-9, atol=1e-12 * np.abs(want[0].solution.lift()).max())
