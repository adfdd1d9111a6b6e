"""Shared loaders for the golden vectors in tests/golden (made by make_golden.py
from the unmodified reference)."""
from __future__ import annotations

import ast
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import scipy.sparse as sp

from oracle import online_ref
from paper_2510_04825_b200 import problems
from paper_2510_04825_b200.offline import RowSelector, SnapshotBasis
from paper_2510_04825_b200.systems import (GaussianKernelOperator, ParametricSystem, StencilOperator,
                                           const_term, exp_term, interval, linear_term)

GOLDEN = Path(__file__).resolve().parent / "golden"
CFG_SIZES = {1: dict(n=2000), 2: dict(n=1000), 3: dict(grid=40), 4: dict(grid=40), 5: dict(grid=12)}


@dataclass
class Case:
    name: str
    system: ParametricSystem
    basis: SnapshotBasis
    selector: RowSelector
    params: list
    data: dict


def _params_list(arr, dim, imag):
    out = []
    for row in arr:
        if dim == 1:
            v = complex(row[0])
            out.append(v if imag else v.real)
        else:
            out.append(tuple(float(complex(v).real) for v in row))
    return out


def tridiag_system(n=120, seed=0):
    """The reference's tridiag test problem (systems.py:289-303) as a drop-in
    system: A(p) = A0 - p I, b(p) = exp(b0 sin(p/10) p) (p-dependent rhs)."""
    a0 = sp.diags([-np.ones(n - 1), 2.0 * np.ones(n), -np.ones(n - 1)], [-1, 0, 1], format="csr")
    b0 = np.random.default_rng(seed).standard_normal(n)

    def rhs_fn(p, idx):
        return np.exp(b0[idx] * np.sin(p / 10.0) * p)

    terms = (const_term(a0), linear_term(sp.identity(n, format="csr"), -1.0))
    return ParametricSystem(n, interval(-10.0, -9.0), rhs_fn, affine_terms=terms, name="tridiag")


def delay_system(n=200, tau=0.1, kappa=2.1, seed=0):
    """The reference's delay problem (systems.py:389-420); -exp(tau p) is an exp term."""
    t = sp.diags([np.ones(n - 1), np.ones(n - 1)], [-1, 1], format="lil")
    t[0, 0] = 1.0
    t[n - 1, n - 1] = 1.0
    a1 = sp.csr_matrix((t.tocsr() - kappa * sp.identity(n)) / tau)
    a0 = sp.csr_matrix(3.0 * a1)
    rng = np.random.default_rng(seed)
    b = rng.standard_normal(n)
    c = rng.standard_normal(n)
    terms = (linear_term(sp.identity(n, format="csr")), const_term(a0, -1.0), exp_term(a1, tau, -1.0))
    return ParametricSystem(n, interval(1.0, 1e4, imag=True), b, affine_terms=terms, output_functional=c,
                            name="delay")


def krr_system(t_train, y_train):
    """The reference's KRR system (systems.py:423-463) as a drop-in system:
    p = (lambda, sigma), K_sigma + lambda I on 1-D points."""
    from paper_2510_04825_b200.systems import Axis, Domain
    op = GaussianKernelOperator(points=np.ascontiguousarray(np.asarray(t_train)[:, None]), ridge_from_param=True)
    return ParametricSystem(len(t_train), Domain(axes=(Axis(1e-5, 1e2), Axis(0.1, 10.0))), np.asarray(y_train),
                            operator=op, name="krr")


def load(name: str) -> Case:
    d = dict(np.load(GOLDEN / f"{name}.npz"))
    if name.startswith("cfg"):
        cfg = int(name[3:])
        system = problems.build(cfg, **CFG_SIZES[cfg]).system
    elif name.startswith("tridiag"):
        system = tridiag_system()
    elif name == "delay":
        system = delay_system()
    elif name == "krr":
        system = krr_system(d["t_train"], d["y_train"])
    else:
        raise KeyError(name)
    imag = any(a.imag for a in system.domain.axes)
    params = _params_list(d["params"], system.domain.dim, imag)
    X = d["X"]
    basis = SnapshotBasis(points=(), raw=X, basis=X, singular_values=d["singular_values"])
    w = d["w"] if d["w"].size else None
    sel = RowSelector(indices=d["S"], n=system.n, weights=w)
    return Case(name, system, basis, sel, params, d)


def oracle_M(case: Case, p):
    """M(p) and t via the oracle, with the reference's coefficient semantics
    (const/linear coefficients coerced to Python complex, systems.py:91-100)."""
    sysm, X, idx = case.system, case.basis.basis, case.selector.indices
    if sysm.affine_terms is not None:
        blocks = online_ref.affine_blocks([t.matrix for t in sysm.affine_terms], X, idx)
        coeffs = []
        for t in sysm.affine_terms:
            if t.kind == "const":
                coeffs.append(complex(t.scale))
            elif t.kind == "linear":
                coeffs.append(complex(t.scale) * p)
            else:
                coeffs.append(t.coeff(p))
        m = online_ref.affine_combine(coeffs, blocks)
    else:
        op = sysm.operator
        if isinstance(op, GaussianKernelOperator):
            if op.ridge_from_param:
                fn = lambda q, rows: online_ref.gauss_rows(op.points, rows, float(q[1]), float(q[0]))
            else:
                fn = lambda q, rows: online_ref.gauss_rows(op.points, rows, float(q), op.ridge)
            m = online_ref.sampled_rows(fn, X, idx, p)
        else:
            fn = lambda q, rows: online_ref.stencil_rows(op, q, rows).toarray()
            m = online_ref.sampled_rows(fn, X, idx, p)
    return m, sysm.rhs(p, idx)


def oracle_solve(case: Case, p):
    m, t = oracle_M(case, p)
    proj = None
    if case.system.output_functional is not None:
        proj = case.system.output_functional.conj() @ case.basis.basis
    return online_ref.solve_one(m, t, case.selector.weights, proj)


def full_matrix(case: Case, p):
    sysm = case.system
    if sysm.affine_terms is not None:
        out = None
        for t in sysm.affine_terms:
            if t.kind == "const":
                f = complex(t.scale)
            elif t.kind == "linear":
                f = complex(t.scale) * p
            else:
                f = t.coeff(p)
            blk = t.matrix * f
            out = blk if out is None else out + blk
        return sp.csr_matrix(out)
    op = sysm.operator
    if isinstance(op, GaussianKernelOperator):
        if op.ridge_from_param:
            return online_ref.gauss_rows(op.points, np.arange(op.n), float(p[1]), float(p[0]))
        return online_ref.gauss_rows(op.points, np.arange(op.n), float(p), op.ridge)
    return online_ref.stencil_rows(op, p, np.arange(op.n))


GOLDEN_NAMES = ["cfg1", "cfg2", "cfg3", "cfg4", "cfg5", "tridiag_lupp", "tridiag_leverage", "delay", "krr"]
