"""Parity at the BASELINE sizes (a few parameters each, against the CPU
oracle on the same X, S): config 1 (n=1e4, real offline), config 2 (n=20,000,
GPU Cholesky snapshots), configs 3 and 4 (n=1e6) with a seeded orthonormal
basis -- the online phase's arithmetic does not depend on how X was made.
Plus size-independent properties of the full sweeps: every status OK,
results independent of the batch they are solved in."""
import numpy as np
import pytest
import torch

from oracle import online_ref
from paper_2510_04825_b200 import online, problems
from paper_2510_04825_b200.offline import (SnapshotBasis, anchor_product, choose_anchor, offline,
                                           select_rows)
from paper_2510_04825_b200.systems import GaussianKernelOperator

pytestmark = pytest.mark.gpu


def _synthetic(prob, r, complex_=False, seed=7):
    g = torch.Generator(device="cpu").manual_seed(seed)
    a = torch.randn(prob.system.n, r, generator=g, dtype=torch.float64)
    if complex_:
        a = torch.complex(a, torch.randn(prob.system.n, r, generator=g, dtype=torch.float64))
    q, _ = torch.linalg.qr(a.cuda())
    X = q.cpu().numpy()
    basis = SnapshotBasis(points=tuple(prob.snapshot_points), raw=X, basis=X, singular_values=np.ones(r))
    anchor = choose_anchor(prob.snapshot_points)
    sel = select_rows(anchor_product(prob.system, anchor, X), prob.system.full_rhs(anchor), strategy="leverage",
                      oversample=prob.samples / (r + 1), seed=prob.selector_seed)
    return basis, sel


def _oracle(prob, basis, sel, p):
    sysm, X, idx = prob.system, basis.basis, sel.indices
    if sysm.affine_terms is not None:
        blocks = online_ref.affine_blocks([t.matrix for t in sysm.affine_terms], X, idx)
        coeffs = [complex(t.scale) if t.kind == "const" else complex(t.scale) * p for t in sysm.affine_terms]
        m = online_ref.affine_combine(coeffs, blocks)
        t = sysm.rhs(p, idx)
        return online_ref.solve_one(m, t, sel.weights)[0], online_ref.ls_floor(m, t, sel.weights, draws=2)
    op = sysm.operator
    fn = ((lambda q, rows: online_ref.gauss_rows(op.points, rows, float(q), op.ridge))
          if isinstance(op, GaussianKernelOperator) else (lambda q, rows: online_ref.stencil_rows(op, q, rows)))
    m = online_ref.sampled_rows(fn, X, idx, p)
    t = sysm.rhs(p, idx)
    uniq, inv = np.unique(idx, return_inverse=True)
    return (online_ref.solve_one(m, t, sel.weights)[0],
            online_ref.ls_floor(m, t, sel.weights, draws=2, rows=fn(p, uniq), basis=X, inverse=inv))


@pytest.fixture(scope="module", params=[1, 2, 3, 4])
def full(request):
    cfg = request.param
    prob = problems.build(cfg)
    if cfg in (1, 2):
        basis, sel = offline(prob, device=torch.device("cuda:0"))
    else:
        basis, sel = _synthetic(prob, {3: 40, 4: 8}[cfg], complex_=(cfg == 4))
    plan = online.precompute_online(prob.system, basis, sel)
    params = prob.test_params(min(prob.default_count, 8192))
    res = online.solve_params(plan, params)
    return cfg, prob, basis, sel, plan, params, res


def test_fullsize_status_and_parity(full):
    cfg, prob, basis, sel, plan, params, res = full
    assert np.all(res.status == 0)
    for k in np.linspace(0, len(params) - 1, 3).astype(int):
        c, floor = _oracle(prob, basis, sel, params[k])
        d = np.linalg.norm(res.coefficients[k] - c) / np.linalg.norm(c)
        assert d <= max(1e-10, 10 * floor), (cfg, k, d, floor)


def test_fullsize_batch_independence(full):
    cfg, prob, basis, sel, plan, params, res = full
    part = online.solve_params(plan, params[100:357])
    assert np.array_equal(part.coefficients, res.coefficients[100:357])


def test_diffusion3d_pipeline_with_cg_snapshots():
    """Config 5's operator end to end at a reduced grid (48^3): GPU CG snapshot
    solves with the reference's residual guard, leverage selection, online
    solve, full-residual checker (K5 DMMA lift + K6) against the oracle."""
    prob = problems.diffusion3d(grid=48)
    basis, sel = offline(prob, device=torch.device("cuda:0"), prefer_cg=True)
    plan = online.precompute_online(prob.system, basis, sel)
    params = prob.test_params(64)
    res = online.solve_params(plan, params)
    assert np.all(res.status == 0)
    for k in (0, 31, 63):
        c, floor = _oracle(prob, basis, sel, params[k])
        d = np.linalg.norm(res.coefficients[k] - c) / np.linalg.norm(c)
        assert d <= max(1e-10, 10 * floor)
    rr = online.relative_residual(plan, params[:8], res.coefficients[:8])
    for k in range(0, 8, 3):
        a = prob.system.matrix(params[k])
        x = basis.basis @ res.coefficients[k]
        ref = online_ref.relative_residual(a, x, prob.system.full_rhs(params[k]))
        assert rr[k] == pytest.approx(ref, rel=1e-3)
    assert np.median(rr) < 1e-2  # the snapshot basis actually approximates the solutions
