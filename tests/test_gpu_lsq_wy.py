"""The compact-WY blocked Householder kernel (k_lsq_wy + k_wy_stencil_rows):
the default K4 for real stencil plans with 33 <= r+1 <= 56, s <= 224 (configs
3 and 5).  Ragged shapes (rows not a multiple of 8, every column-tile count,
the right-hand side alone in its column tile or sharing the last panel),
weighted / unweighted / repeated rows, rank-deficient and non-finite systems,
chunked sweeps -- against the CPU oracle (reference linalg.py:89-113 via
online.py:105-134), and against the column-owner kernel in a child process
(SAS_LSQ_WY=off)."""
import os
import subprocess
import sys
from pathlib import Path

import numpy as np
import pytest
import torch

from oracle import online_ref
from paper_2510_04825_b200 import online, problems
from paper_2510_04825_b200.offline import RowSelector, SnapshotBasis

ROOT = Path(__file__).resolve().parents[1]
pytestmark = pytest.mark.gpu


def _case(kind, grid, s, r, seed, weighted=True, repeat=True):
    prob = problems.diffusion2d(grid=grid) if kind == "2d" else problems.diffusion3d(grid=grid)
    n = prob.system.n
    g = np.random.default_rng(seed)
    X, _ = np.linalg.qr(g.standard_normal((n, r)))
    idx = g.choice(n, size=s, replace=False)
    if repeat and s >= r + 8:
        idx[-3:] = idx[:3]          # leverage sampling draws with replacement
    w = g.uniform(0.5, 2.0, size=s) if weighted else None
    basis = SnapshotBasis(points=tuple(prob.snapshot_points), raw=X, basis=X, singular_values=np.ones(r))
    sel = RowSelector(indices=idx.astype(np.int64), n=n, weights=w, strategy="leverage" if weighted else "random")
    return prob, basis, sel


def _oracle_coef(prob, basis, sel, p):
    op = prob.system.operator
    fn = lambda q, rows: online_ref.stencil_rows(op, q, rows)
    m = online_ref.sampled_rows(fn, basis.basis, sel.indices, p)
    t = prob.system.rhs(p, sel.indices)
    c, res = online_ref.solve_one(m, t, sel.weights)[:2]
    uniq, inv = np.unique(sel.indices, return_inverse=True)
    floor = online_ref.ls_floor(m, t, sel.weights, draws=2, rows=fn(p, uniq), basis=basis.basis, inverse=inv)
    return c, res, floor


SHAPES = [("2d", 24, 40, 32), ("2d", 24, 57, 33), ("2d", 24, 100, 39), ("2d", 32, 160, 40), ("2d", 32, 161, 47),
          ("3d", 10, 200, 50), ("3d", 10, 224, 55), ("3d", 10, 56, 55), ("3d", 10, 129, 48), ("3d", 10, 203, 41)]


@pytest.mark.parametrize("kind,grid,s,r", SHAPES)
@pytest.mark.parametrize("weighted", [True, False])
def test_wy_shapes_against_oracle(kind, grid, s, r, weighted):
    prob, basis, sel = _case(kind, grid, s, r, seed=s * 100 + r, weighted=weighted)
    plan = online.precompute_online(prob.system, basis, sel)
    params = prob.test_params(70)
    res = online.solve_params(plan, params)
    assert np.all(res.status == 0)
    for k in (0, 1, 33, 69):
        c, sres, floor = _oracle_coef(prob, basis, sel, params[k])
        d = np.linalg.norm(res.coefficients[k] - c) / np.linalg.norm(c)
        assert d <= max(1e-10, 10 * floor), (kind, s, r, k, d, floor)
        assert res.sampled_residual[k] == pytest.approx(sres, rel=1e-9, abs=1e-13)


def test_wy_chunked_sweep_is_bitwise_batch_independent():
    prob, basis, sel = _case("3d", 10, 200, 50, seed=5)
    plan = online.precompute_online(prob.system, basis, sel)
    params = prob.test_params(1500)
    res = online.solve_params(plan, params)
    part = online.solve_params(plan, params[700:901])
    assert np.array_equal(part.coefficients, res.coefficients[700:901])
    assert np.array_equal(part.sampled_residual, res.sampled_residual[700:901])
    env = dict(os.environ, SAS_LSQ_WY_CHUNK="333")
    code = ("import numpy as np, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "from test_gpu_lsq_wy import _case; from paper_2510_04825_b200 import online\n"
            "prob, basis, sel = _case('3d', 10, 200, 50, seed=5)\n"
            "plan = online.precompute_online(prob.system, basis, sel)\n"
            "res = online.solve_params(plan, prob.test_params(1500))\n"
            "np.save(sys.argv[1], res.coefficients)\n") % (str(ROOT), str(ROOT / "tests"))
    out = ROOT / "gpurun_out" / "_wy_chunk.npy"
    out.parent.mkdir(exist_ok=True)
    r = subprocess.run([sys.executable, "-c", code, str(out)], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert np.array_equal(np.load(out), res.coefficients)
    out.unlink()


def test_wy_fused_assembly_equals_two_kernel_path():
    """The two-kernel path (k_wy_stencil_rows + k_lsq_wy per chunk, the default) and the
    fused path (SAS_LSQ_WY_FUSED=1: the next block assembled by the idle warps into the
    CTA's L2 slots) build bitwise the same blocks and run the same factorisation."""
    prob, basis, sel = _case("3d", 10, 200, 50, seed=5)
    plan = online.precompute_online(prob.system, basis, sel)
    res = online.solve_params(plan, prob.test_params(1500))
    env = dict(os.environ, SAS_LSQ_WY_FUSED="1")
    code = ("import numpy as np, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "from test_gpu_lsq_wy import _case; from paper_2510_04825_b200 import online\n"
            "prob, basis, sel = _case('3d', 10, 200, 50, seed=5)\n"
            "plan = online.precompute_online(prob.system, basis, sel)\n"
            "res = online.solve_params(plan, prob.test_params(1500))\n"
            "np.save(sys.argv[1], np.concatenate([res.coefficients, res.sampled_residual[:, None]], axis=1))\n"
            ) % (str(ROOT), str(ROOT / "tests"))
    out = ROOT / "gpurun_out" / "_wy_two.npy"
    out.parent.mkdir(exist_ok=True)
    r = subprocess.run([sys.executable, "-c", code, str(out)], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    other = np.load(out)
    out.unlink()
    assert np.array_equal(other[:, :-1], res.coefficients)
    assert np.array_equal(other[:, -1], res.sampled_residual)


def test_wy_matches_column_owner_kernel():
    """Same reflectors, different blocking: the two kernels agree to rounding."""
    prob, basis, sel = _case("2d", 32, 160, 40, seed=11)
    plan = online.precompute_online(prob.system, basis, sel)
    params = prob.test_params(300)
    res = online.solve_params(plan, params)
    env = dict(os.environ, SAS_LSQ_WY="off")
    code = ("import numpy as np, sys; sys.path.insert(0, %r); sys.path.insert(0, %r)\n"
            "from test_gpu_lsq_wy import _case; from paper_2510_04825_b200 import online\n"
            "prob, basis, sel = _case('2d', 32, 160, 40, seed=11)\n"
            "plan = online.precompute_online(prob.system, basis, sel)\n"
            "res = online.solve_params(plan, prob.test_params(300))\n"
            "np.save(sys.argv[1], res.coefficients)\n") % (str(ROOT), str(ROOT / "tests"))
    out = ROOT / "gpurun_out" / "_wy_cw.npy"
    out.parent.mkdir(exist_ok=True)
    r = subprocess.run([sys.executable, "-c", code, str(out)], cwd=ROOT, env=env, capture_output=True, text=True,
                       timeout=900)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    other = np.load(out)
    out.unlink()
    d = np.linalg.norm(other - res.coefficients, axis=1) / np.linalg.norm(res.coefficients, axis=1)
    assert d.max() < 1e-11, d.max()


def test_wy_rank_deficient_and_nonfinite():
    prob, basis, sel = _case("3d", 10, 200, 50, seed=3)
    X = basis.basis.copy()
    X[:, 17] = X[:, 4]                      # two equal basis columns: M(p) is rank deficient for every p
    bad = SnapshotBasis(points=basis.points, raw=X, basis=X, singular_values=np.ones(50))
    plan = online.precompute_online(prob.system, bad, sel)
    params = prob.test_params(40)
    res = online.solve_params(plan, params)
    assert np.all(res.status == 1)
    assert np.all(res.bad_column == 17)
    assert np.all(np.isnan(res.coefficients))
    # the reference's error for the same system (linalg.py:107-112 via the oracle)
    op = prob.system.operator
    m = online_ref.sampled_rows(lambda q, rows: online_ref.stencil_rows(op, q, rows), X, sel.indices, params[0])
    with pytest.raises(Exception):
        online_ref.solve_one(m, prob.system.rhs(params[0], sel.indices), sel.weights)
    # one non-finite parameter value poisons only its own system
    plan2 = online.precompute_online(prob.system, basis, sel)
    p2 = np.array(params, dtype=float)
    p2[7, 2] = np.inf
    p2 = list(p2)
    res2 = online.solve_params(plan2, p2)
    assert res2.status[7] == 2 and np.all(np.isnan(res2.coefficients[7]))
    ok = np.delete(np.arange(40), 7)
    assert np.all(res2.status[ok] == 0)
    good = online.solve_params(plan2, params)
    assert np.array_equal(res2.coefficients[ok], good.coefficients[ok])
