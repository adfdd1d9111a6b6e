"""The five BASELINE.json workloads as parametric systems (shared inputs).

None of them exists as a generator in the reference, so they
are defined here once, with every detail BASELINE.json leaves open pinned
(SURVEY.md §8(d)).  The same definitions feed the GPU plan, the CPU oracle
(oracle/) and the golden-vector script (tests/golden/make_golden.py, which
wraps them in reference ParametricSystem objects).

 cfg  name              A(p)                                   online path
 1    reaction1d        T + p diag(c)            (affine, K=2)  K1 + K4
 2    gauss_krr         K_p + 1e-3 I, d=8        (kernel rows)  K3 + K4
 3    diffusion2d       5-point -div(a grad u), a=exp(sum_4 p_k phi_k)  K2 + K4
 4    convdiff_tf       p I - M, p = i w         (affine, c128) K1 + K4
 5    diffusion3d       7-point, a=exp(sum_6 p_k phi_k)         K2 + K4

Every generator takes a size argument so tests can use reduced grids.
"""
from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Optional

import numpy as np
import scipy.sparse as sp

from .systems import (Axis, Domain, GaussianKernelOperator, ParametricSystem, StencilOperator,
                      box, const_term, interval, linear_term)


@dataclass
class Problem:
    """A BASELINE workload: the system, its offline recipe and its test sweep."""

    key: str
    system: ParametricSystem
    snapshot_points: list
    snapshot_mode: object          # "qr" or ("pod", tol)
    samples: int                   # s
    selector_seed: int
    make_params: Callable          # (count, seed) -> list of parameters
    default_count: int
    param_seed: int
    extras: dict = field(default_factory=dict)

    def test_params(self, count: Optional[int] = None):
        return self.make_params(self.default_count if count is None else count, self.param_seed)


# --------------------------------------------------------------------------
# config 1: 1-D parametric reaction-diffusion (CPU plumbing)
# --------------------------------------------------------------------------
def reaction1d(n: int = 10_000, seed: int = 0) -> Problem:
    rng = np.random.default_rng(seed)
    c = rng.uniform(0.5, 1.5, n)
    b = rng.standard_normal(n)
    t = sp.diags([-np.ones(n - 1), 2.0 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr") * float((n + 1) ** 2)
    terms = (const_term(t), linear_term(sp.diags(c, format="csr")))
    system = ParametricSystem(n, interval(0.0, 1.0), b, affine_terms=terms, name="reaction1d",
                              extras={"c": c})
    r = 10
    nodes = np.cos(np.pi * (2 * np.arange(r) + 1) / (2 * r))[::-1]   # snapshot.py:69-71
    pts = list(0.5 + 0.5 * nodes)

    def make_params(count, pseed):
        return list(np.random.default_rng(pseed).uniform(0.0, 1.0, count))

    return Problem("reaction1d", system, pts, ("pod", 1e-13), samples=20, selector_seed=0,
                   make_params=make_params, default_count=1000, param_seed=101)


# --------------------------------------------------------------------------
# config 2: Gaussian-kernel ridge regression over the bandwidth
# --------------------------------------------------------------------------
def gauss_krr(n: int = 20_000, d: int = 8, seed: int = 0, ridge: float = 1e-3) -> Problem:
    rng = np.random.default_rng(seed)
    xs = rng.standard_normal((n, d))
    b = np.sin(xs.sum(axis=1)) + 0.1 * rng.standard_normal(n)
    op = GaussianKernelOperator(points=np.ascontiguousarray(xs), ridge=ridge)
    system = ParametricSystem(n, interval(0.5, 2.0), b, operator=op, name="gauss_krr")
    r = 20
    pts = list(np.logspace(np.log10(0.5), np.log10(2.0), r))       # snapshot.py:61-64

    def make_params(count, pseed):
        u = np.random.default_rng(pseed).uniform(np.log(0.5), np.log(2.0), count)
        return list(np.exp(u))

    return Problem("gauss_krr", system, pts, "qr", samples=80, selector_seed=0,
                   make_params=make_params, default_count=4096, param_seed=102)


# --------------------------------------------------------------------------
# configs 3 and 5: diffusion with exp-affine coefficient (stencil rows)
# --------------------------------------------------------------------------
def _phi2d(mids: np.ndarray) -> np.ndarray:
    """phi_k(x) = sin(k pi x1) sin(k pi x2), k = 1..4."""
    x1, x2 = mids[:, 0], mids[:, 1]
    return np.stack([np.sin((k * np.pi) * x1) * np.sin((k * np.pi) * x2) for k in range(1, 5)], axis=1)


PHI3D_MODES = ((1, 1, 1), (2, 1, 1), (1, 2, 1), (1, 1, 2), (2, 2, 1), (1, 2, 2))


def _phi3d(mids: np.ndarray) -> np.ndarray:
    """phi_k(x) = sin(a pi x1) sin(b pi x2) sin(c pi x3), (a,b,c) in PHI3D_MODES."""
    x1, x2, x3 = mids[:, 0], mids[:, 1], mids[:, 2]
    return np.stack([np.sin((a * np.pi) * x1) * np.sin((b * np.pi) * x2) * np.sin((c * np.pi) * x3)
                     for a, b, c in PHI3D_MODES], axis=1)


def _halton(d: int, count: int, lo: float, hi: float):
    from scipy.stats import qmc
    pts = qmc.Halton(d=d, scramble=False).random(count + 1)[1:]    # drop the origin
    return [tuple(float(v) for v in row) for row in lo + (hi - lo) * pts]


def diffusion2d(grid: int = 1000) -> Problem:
    op = StencilOperator(grid=grid, dims=2, basis_fns=_phi2d, n_params=4)
    system = ParametricSystem(op.n, box(*([(-0.5, 0.5)] * 4)), np.ones(op.n), operator=op,
                              name="diffusion2d")

    def make_params(count, pseed):
        return [tuple(row) for row in np.random.default_rng(pseed).uniform(-0.5, 0.5, (count, 4))]

    return Problem("diffusion2d", system, _halton(4, 40, -0.5, 0.5), "qr", samples=160,
                   selector_seed=0, make_params=make_params, default_count=65_536, param_seed=103)


def diffusion3d(grid: int = 216) -> Problem:
    op = StencilOperator(grid=grid, dims=3, basis_fns=_phi3d, n_params=6)
    system = ParametricSystem(op.n, box(*([(-0.3, 0.3)] * 6)), np.ones(op.n), operator=op,
                              name="diffusion3d")

    def make_params(count, pseed):
        return [tuple(row) for row in np.random.default_rng(pseed).uniform(-0.3, 0.3, (count, 6))]

    return Problem("diffusion3d", system, _halton(6, 50, -0.3, 0.3), "qr", samples=200,
                   selector_seed=0, make_params=make_params, default_count=1_000_000, param_seed=105,
                   extras={"residual_subset": 1024})


# --------------------------------------------------------------------------
# config 4: transfer-function sweep of an upwind convection-diffusion operator
# --------------------------------------------------------------------------
def convdiff_matrix(grid: int, velocity=(50.0, 50.0)) -> sp.csr_matrix:
    """M = Lap_h - v1 Dx^- - v2 Dy^-: 5-point Laplacian and first-order backward
    (upwind for v > 0) differences, node index i*g + j with i along x1."""
    g = grid
    h = 1.0 / (g + 1)
    e = np.ones(g)
    lap1 = sp.diags([e[:-1], -2.0 * e, e[:-1]], [-1, 0, 1], format="csr") / (h * h)
    back1 = sp.diags([e, -e[:-1]], [0, -1], format="csr") / h
    eye = sp.identity(g, format="csr")
    lap = sp.kron(lap1, eye, format="csr") + sp.kron(eye, lap1, format="csr")
    dx = sp.kron(back1, eye, format="csr")
    dy = sp.kron(eye, back1, format="csr")
    return sp.csr_matrix(lap - velocity[0] * dx - velocity[1] * dy)


def convdiff_tf(grid: int = 1000, seed: int = 1) -> Problem:
    n = grid * grid
    m = convdiff_matrix(grid)
    rng = np.random.default_rng(seed)
    b = rng.standard_normal(n) / np.sqrt(n)
    c = rng.standard_normal(n) / np.sqrt(n)
    terms = (linear_term(sp.identity(n, format="csr")), const_term(m, -1.0))
    system = ParametricSystem(n, interval(1e-2, 1e2, imag=True), b, affine_terms=terms,
                              output_functional=c, name="convdiff_tf")
    pts = list(1j * np.logspace(-2.0, 2.0, 30))

    def make_params(count, pseed):
        return list(1j * np.logspace(-2.0, 2.0, count))

    return Problem("convdiff_tf", system, pts, ("pod", 1e-13), samples=120, selector_seed=0,
                   make_params=make_params, default_count=100_000, param_seed=104)


BUILDERS = {
    1: reaction1d,
    2: gauss_krr,
    3: diffusion2d,
    4: convdiff_tf,
    5: diffusion3d,
}


def build(cfg: int, **kw) -> Problem:
    return BUILDERS[cfg](**kw)
