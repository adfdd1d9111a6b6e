"""Generate the golden vectors by running the UNMODIFIED reference package.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

For every BASELINE config (at a reduced size the reference finishes in
seconds) and for the reference's own test systems, this runs the reference's
offline phase (snapshot.build_snapshot, subsample.select_rows as
cli.build_offline does) and its online phase (online.precompute_online,
online.solve_batch), then records X, S, weights, parameters and the
reference's outputs: coefficients, sampled residuals, output values and the
verification relative residual ||A(p) x - b|| / ||b|| (cli.py:344-351).  It also
records a per-parameter parity floor (oracle.online_ref.ls_floor).

The BASELINE problems do not exist in the reference, so their row oracles are
the harness functions in oracle/online_ref.py wrapped in the reference's own
ParametricSystem (row_fn / matrix_fn / affine_terms), exactly as the reference
tests inject systems (test_acceptance.py:239-250).
"""
from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np
import scipy.sparse as sp

REPO = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(REPO))
REF = os.environ.get("SUBAPSNAP_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)

import subapsnap  # noqa: E402  (the reference)
from subapsnap import online as ref_online  # noqa: E402
from subapsnap import snapshot as ref_snapshot  # noqa: E402
from subapsnap import subsample as ref_subsample  # noqa: E402
from subapsnap import systems as ref_systems  # noqa: E402
from subapsnap.errors import RankDeficiencyError  # noqa: E402

from oracle import online_ref  # noqa: E402
from paper_2510_04825_b200 import problems  # noqa: E402
from paper_2510_04825_b200.systems import GaussianKernelOperator, StencilOperator  # noqa: E402

OUT = Path(__file__).resolve().parent

SIZES = {1: dict(n=2000), 2: dict(n=1000), 3: dict(grid=40), 4: dict(grid=40), 5: dict(grid=12)}
COUNTS = {1: 200, 2: 64, 3: 64, 4: 200, 5: 32}


def ref_system(prob):
    """Wrap a problems.Problem into a reference ParametricSystem."""
    sysm = prob.system
    b = np.asarray(sysm.b)

    def rhs_fn(p, idx):
        return b[idx]

    dom = ref_systems.Domain(axes=tuple(ref_systems.Axis(a.lo, a.hi, a.imag) for a in sysm.domain.axes))
    if sysm.affine_terms is not None:
        terms = []
        for t in sysm.affine_terms:
            if t.kind == "const":
                terms.append(ref_systems.const_term(t.matrix, t.scale))
            elif t.kind == "linear":
                terms.append(ref_systems.linear_term(t.matrix, t.scale))
            else:
                raise ValueError(t.kind)
        return ref_systems.ParametricSystem(sysm.n, dom, rhs_fn, affine_terms=terms,
                                            output_functional=sysm.output_functional, name=sysm.name)
    op = sysm.operator
    if isinstance(op, GaussianKernelOperator):
        def row_fn(p, idx):
            return online_ref.gauss_rows(op.points, idx, float(p), op.ridge)

        def matrix_fn(p):
            return online_ref.gauss_rows(op.points, np.arange(op.n), float(p), op.ridge)
    else:
        def row_fn(p, idx):
            return online_ref.stencil_rows(op, p, idx)

        def matrix_fn(p):
            return online_ref.stencil_rows(op, p, np.arange(op.n))
    return ref_systems.ParametricSystem(sysm.n, dom, rhs_fn, row_fn=row_fn, matrix_fn=matrix_fn,
                                        name=sysm.name)


def run_reference(rsys, points, mode, samples, seed, params, strategy="leverage", oversample=None,
                  selector=None):
    t0 = time.perf_counter()
    try:
        basis = ref_snapshot.build_snapshot(rsys, points, mode=mode)
        used_mode = mode
    except RankDeficiencyError:
        used_mode = ("pod", 1e-13)
        basis = ref_snapshot.build_snapshot(rsys, points, mode=used_mode)
    anchor = ref_subsample.choose_anchor(points)
    b_anchor = np.asarray(rsys.matrix(anchor) @ basis.basis)
    rhs_anchor = rsys.full_rhs(anchor)
    if selector is None:
        width = basis.rank + 1
        ovs = samples / width if oversample is None else oversample
        cfg = ref_subsample.SelectorConfig(strategy=strategy, oversample=ovs, seed=seed)
        selector = ref_subsample.select_rows(b_anchor, rhs_anchor, cfg, anchors=(anchor,))
    t_off = time.perf_counter() - t0
    plan = ref_online.precompute_online(rsys, basis, selector)
    t0 = time.perf_counter()
    rows = ref_online.solve_batch(plan, params, want_interval=selector.weights is not None)
    t_on = time.perf_counter() - t0
    coef = np.array([row.solution.coefficients for row in rows])
    sres = np.array([row.sampled_residual for row in rows])
    outv = np.array([row.output_value if row.output_value is not None else np.nan for row in rows], dtype=complex)
    relres = []
    floors = []
    for row, p in zip(rows, params):
        x = row.solution.lift()
        b = rsys.full_rhs(p)
        relres.append(np.linalg.norm(rsys.matrix(p) @ x - b) / max(np.linalg.norm(b), 1e-300))
        # parity floor from the reference's own M at this p
        if plan.affine:
            m = sum(t.coeff(p) * blk for t, blk in zip(rsys.affine_terms, plan.blocks))
            floors.append(online_ref.ls_floor(m, rsys.rhs(p, selector.indices), selector.weights))
        else:
            m = ref_online._sampled_rows(rsys, basis, selector.indices, p)
            uniq, inverse = np.unique(selector.indices, return_inverse=True)
            floors.append(online_ref.ls_floor(m, rsys.rhs(p, selector.indices), selector.weights,
                                              rows=rsys.rows_dense(p, uniq), basis=basis.basis, inverse=inverse))
    return dict(
        X=np.asarray(basis.basis), S=np.asarray(selector.indices, dtype=np.int64),
        w=np.asarray(selector.weights) if selector.weights is not None else np.zeros(0),
        coef=coef, sres=sres, outv=outv, relres=np.array(relres), floor=np.array(floors),
        singular_values=np.asarray(basis.singular_values), mode=np.array(repr(used_mode)),
        anchor=np.array(complex(np.atleast_1d(np.asarray(anchor, dtype=complex))[0])) if np.isscalar(anchor)
        else np.asarray(anchor, dtype=complex),
        t_offline=np.array(t_off), t_online=np.array(t_on),
    )


def params_array(params):
    arr = np.array([np.atleast_1d(np.asarray(p, dtype=complex)) for p in params])
    return arr


def main(which=None):
    cfgs = [c for c in (which or [1, 2, 3, 4, 5]) if isinstance(c, int)]
    for cfg in cfgs:
        prob = problems.build(cfg, **SIZES[cfg])
        params = prob.test_params(COUNTS[cfg])
        rsys = ref_system(prob)
        t0 = time.perf_counter()
        res = run_reference(rsys, prob.snapshot_points, prob.snapshot_mode, prob.samples, prob.selector_seed,
                            params)
        res["params"] = params_array(params)
        res["size"] = np.array(repr(SIZES[cfg]))
        path = OUT / f"cfg{cfg}.npz"
        np.savez_compressed(path, **res)
        print(f"cfg{cfg}: n={prob.system.n} r'={res['X'].shape[1]} s={res['S'].size} mode={res['mode']} "
              f"P={len(params)} max floor={res['floor'].max():.2e} relres~{np.median(res['relres']):.2e} "
              f"({time.perf_counter() - t0:.1f}s) -> {path.name} {path.stat().st_size // 1024} KiB")

    if which is None or "tridiag" in (which or []):
        # the reference's own test systems (test_online.py:10-15, 147-156)
        rsys = ref_systems.build_problem(ref_systems.ProblemSpec("tridiag", {"n": 120}))
        pts = ref_snapshot.default_snapshot_points(rsys.domain, 6)
        params = list(np.random.default_rng(0).uniform(-10.0, -9.0, 20))
        for strat, ovs in (("lupp", None), ("leverage", 6.0)):
            res = run_reference(rsys, pts, "qr", None, 0, params, strategy=strat, oversample=ovs or 4.0)
            res["params"] = params_array(params)
            np.savez_compressed(OUT / f"tridiag_{strat}.npz", **res)
            print(f"tridiag {strat}: r'={res['X'].shape[1]} s={res['S'].size}")
        # the reference's own KRR system: p = (lambda, sigma), 1-D points,
        # _kernels.rbf_rows row oracle (test_online.py:159-172)
        rsys = ref_systems.build_problem(ref_systems.ProblemSpec("krr", {"n_train": 120, "n_test": 10}))
        pairs = [(1e-3, 1.0), (1e-1, 3.0), (1.0, 6.0), (10.0, 9.0)]
        rng = np.random.default_rng(5)
        params = pairs + [(float(10 ** rng.uniform(-3, 1)), float(rng.uniform(1.0, 9.0))) for _ in range(20)]
        res = run_reference(rsys, pairs, "qr", None, 0, params, oversample=4.0)
        res["params"] = params_array(params)
        res["t_train"] = rsys.extras["t_train"]
        res["y_train"] = rsys.extras["y_train"]
        np.savez_compressed(OUT / "krr.npz", **res)
        print(f"krr: r'={res['X'].shape[1]} s={res['S'].size} mode={res['mode']}")
        # delay system: coefficient -exp(tau p) (an "other" term in the reference)
        rsys = ref_systems.build_problem(ref_systems.ProblemSpec("delay", {"n": 200}))
        pts = ref_snapshot.default_snapshot_points(rsys.domain, 8, "log-spaced")
        params = list(1j * np.logspace(0.0, 4.0, 40))
        res = run_reference(rsys, pts, ("pod", 1e-12), None, 0, params, oversample=4.0)
        res["params"] = params_array(params)
        np.savez_compressed(OUT / "delay.npz", **res)
        print(f"delay: r'={res['X'].shape[1]} s={res['S'].size}")


if __name__ == "__main__":
    args = sys.argv[1:]
    main([int(a) if a.isdigit() else a for a in args] or None)
