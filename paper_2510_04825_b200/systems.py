"""Parametric systems A(p) x(p) = b(p) as GPU operator descriptors.

The reference describes A(p) through opaque Python callables (row_fn,
rhs_fn, AffineTerm.coeff; /root/reference/pkg/src/subapsnap/systems.py:76-126)
that a GPU cannot execute.  This module keeps the reference's vocabulary
(ParametricSystem, AffineTerm, const_term, linear_term, Domain/Axis/interval)
and adds the two non-affine row operators the BASELINE configs need, each of
which can emit its C-ABI descriptor (include/sas.h `sas_desc`) for a given row
selection S:

* affine   A(p) = sum_k f_k(p) A_k with f_k in {const, linear, c*exp(a*p)}
           (systems.py:91-100, 549-570) or an opaque callable evaluated per p
           into a coefficient table;
* StencilOperator  edge-midpoint finite differences of -div(a(x;p) grad u) on a
           regular 2-D/3-D grid with a(x;p) = exp(sum_k p_k phi_k(x)), in the
           edge form of the reference's _conductivity_matrix (systems.py:306-334);
* GaussianKernelOperator  K_p + ridge I with K_p(i,j) = exp(-|x_i-x_j|^2/(2p^2))
           (the d-dimensional generalisation of _kernels.rbf_rows, _kernels.py:38-50).
"""
from __future__ import annotations

import cmath
from dataclasses import dataclass, field
from typing import Callable, Optional, Sequence

import numpy as np
import scipy.sparse as sp

from .errors import ConfigError


# --------------------------------------------------------------------------
# parameter domains (systems.py:30-69)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class Axis:
    lo: float
    hi: float
    imag: bool = False

    def __post_init__(self):
        if not self.hi >= self.lo:
            raise ConfigError(f"axis endpoints out of order: [{self.lo}, {self.hi}]")


@dataclass(frozen=True)
class Domain:
    axes: tuple

    @property
    def dim(self) -> int:
        return len(self.axes)


def interval(lo: float, hi: float, imag: bool = False) -> Domain:
    return Domain(axes=(Axis(lo, hi, imag),))


def box(*bounds) -> Domain:
    return Domain(axes=tuple(Axis(lo, hi) for lo, hi in bounds))


def param_vector(p) -> np.ndarray:
    if np.isscalar(p):
        return np.array([p], dtype=complex)
    return np.asarray(p, dtype=complex).ravel()


# --------------------------------------------------------------------------
# affine terms (systems.py:76-100)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class AffineTerm:
    """One term f_k(p) A_k.  kind: "const" (f = scale), "linear" (f = scale*p),
    "exp" (f = scale*exp(rate*p)), or "other" (opaque `coeff`, evaluated on the
    host per parameter and shipped as a coefficient table)."""

    coeff: Callable
    matrix: sp.csr_matrix
    kind: str = "other"
    scale: complex = 1.0
    rate: complex = 0.0


def const_term(a, scale=1.0) -> AffineTerm:
    s = scale
    return AffineTerm(coeff=lambda p, s=s: s, matrix=sp.csr_matrix(a), kind="const", scale=s)


def linear_term(a, scale=1.0) -> AffineTerm:
    s = scale
    return AffineTerm(coeff=lambda p, s=s: s * p, matrix=sp.csr_matrix(a), kind="linear", scale=s)


def exp_term(a, rate, scale=1.0) -> AffineTerm:
    """f(p) = scale * exp(rate * p)  (the "c*exp(a*p)" grammar, systems.py:549-570)."""
    s, r = scale, rate
    return AffineTerm(coeff=lambda p, s=s, r=r: s * cmath.exp(r * p), matrix=sp.csr_matrix(a),
                      kind="exp", scale=s, rate=r)


# --------------------------------------------------------------------------
# non-affine row operators
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class StencilOperator:
    """-div(a(x;p) grad u) with zero Dirichlet data on the interior nodes of
    the unit cube [0,1]^d, g nodes per axis, h = 1/(g+1), node coordinates
    x = (i+1) h, node index i0*g^(d-1) + ... + i_{d-1} (row-major).  Row of node
    i:  A_ii = sum_e c_e,  A_{i,nbr(e)} = -c_e for interior neighbours,
    c_e = exp(sum_k p_k phi_k(mid_e)) / h^2 with mid_e the edge midpoint.
    Edge order: +axis0, -axis0, +axis1, -axis1, ...

    `basis_fns(coords) -> (m, d_p)` evaluates phi_k at midpoints given as an
    (m, d) array.
    """

    grid: int
    dims: int
    basis_fns: Callable
    n_params: int

    @property
    def n(self) -> int:
        return self.grid ** self.dims

    @property
    def h(self) -> float:
        return 1.0 / (self.grid + 1)

    @property
    def n_edges(self) -> int:
        return 2 * self.dims

    def offsets(self) -> np.ndarray:
        out = []
        for ax in range(self.dims):
            for sgn in (1, -1):
                o = [0] * self.dims
                o[ax] = sgn
                out.append(o)
        return np.array(out, dtype=np.int64)

    def node_coords(self, nodes) -> np.ndarray:
        """Integer grid coordinates (m, d) of node indices."""
        nodes = np.asarray(nodes, dtype=np.int64)
        g = self.grid
        out = np.empty((nodes.size, self.dims), dtype=np.int64)
        rem = nodes.copy()
        for ax in range(self.dims - 1, -1, -1):
            out[:, ax] = rem % g
            rem //= g
        return out

    def edges(self, nodes):
        """(nbr (m,E) int64 with -1 on the boundary, phi (m,E,d_p) float64)."""
        nodes = np.asarray(nodes, dtype=np.int64)
        ij = self.node_coords(nodes)
        g, h = self.grid, self.h
        offs = self.offsets()
        m, E = nodes.size, self.n_edges
        nbr = np.empty((m, E), dtype=np.int64)
        mids = np.empty((m, E, self.dims))
        x = (ij + 1) * h  # node coordinates
        for e, o in enumerate(offs):
            nij = ij + o
            inside = np.all((nij >= 0) & (nij < g), axis=1)
            lin = np.zeros(m, dtype=np.int64)
            for ax in range(self.dims):
                lin = lin * g + nij[:, ax]
            nbr[:, e] = np.where(inside, lin, -1)
            # midpoint x + o*h/2, evaluated as in systems.py:323 (x + di*h/2.0)
            mids[:, e, :] = x + (o * h) / 2.0
        phi = self.basis_fns(mids.reshape(-1, self.dims)).reshape(m, E, self.n_params)
        return nbr, np.ascontiguousarray(phi)


@dataclass(frozen=True)
class GaussianKernelOperator:
    """Rows of K_p + ridge I, K_p(i,j) = exp(-(D_ij * inv)), D_ij = sum_k
    (x_ik - x_jk)^2 summed sequentially over k, inv = 1/(2 sigma^2).  The
    parameter is the bandwidth sigma (fixed `ridge`), or with
    `ridge_from_param` the pair p = (lambda, sigma) of the reference's KRR
    system (systems.py:423-463, rows by _kernels.rbf_rows for 1-D points)."""

    points: np.ndarray
    ridge: float = 0.0
    ridge_from_param: bool = False

    @property
    def n(self) -> int:
        return self.points.shape[0]


# --------------------------------------------------------------------------
class ParametricSystem:
    """A(p) x = b(p).  `rhs` is either a constant vector b (length n) or a
    callable rhs_fn(p, idx) (evaluated on the host per parameter).  Exactly one
    of `affine_terms` or `operator` describes A(p)."""

    def __init__(self, n, domain, rhs, affine_terms=None, operator=None, output_functional=None,
                 name="", extras=None):
        if affine_terms is None and operator is None:
            raise ValueError("need affine terms or a row operator")
        self.n = int(n)
        self.domain = domain
        self.affine_terms = tuple(affine_terms) if affine_terms else None
        self.operator = operator
        if callable(rhs):
            self._rhs_fn = rhs
            self.b = None
        else:
            self.b = np.asarray(rhs)
            self._rhs_fn = None
            if self.b.shape != (self.n,):
                raise ValueError("rhs vector must have length n")
        self.output_functional = None if output_functional is None else np.asarray(output_functional)
        self.name = name
        self.extras = dict(extras or {})

    @property
    def dim(self) -> int:
        return self.domain.dim

    @property
    def rhs_constant(self) -> bool:
        return self.b is not None

    def rhs(self, p, indices) -> np.ndarray:
        indices = np.asarray(indices, dtype=np.int64)
        if indices.size and (indices.min() < 0 or indices.max() >= self.n):
            raise IndexError(f"rhs index out of range for n={self.n}")
        if self.b is not None:
            return self.b[indices]
        return np.asarray(self._rhs_fn(p, indices))

    def full_rhs(self, p) -> np.ndarray:
        return self.rhs(p, np.arange(self.n))

    def matrix(self, p) -> sp.csr_matrix:
        """Assembled A(p) (host; for verification and small problems only)."""
        if self.affine_terms is not None:
            out = None
            for term in self.affine_terms:
                blk = term.matrix * term.coeff(p)
                out = blk if out is None else out + blk
            return sp.csr_matrix(out)
        op = self.operator
        if isinstance(op, StencilOperator):
            nodes = np.arange(op.n)
            nbr, phi = op.edges(nodes)
            pv = np.asarray(p, dtype=float).ravel()
            arg = phi[..., 0] * pv[0]
            for k in range(1, pv.size):
                arg = arg + phi[..., k] * pv[k]
            c = np.exp(arg) / (op.h * op.h)
            diag = c[:, 0].copy()
            for e in range(1, c.shape[1]):
                diag = diag + c[:, e]
            rows = [nodes]
            cols = [nodes]
            vals = [diag]
            for e in range(c.shape[1]):
                ok = nbr[:, e] >= 0
                rows.append(nodes[ok])
                cols.append(nbr[ok, e])
                vals.append(-c[ok, e])
            return sp.csr_matrix((np.concatenate(vals), (np.concatenate(rows), np.concatenate(cols))),
                                 shape=(op.n, op.n))
        raise ValueError("matrix() is not available for this operator on the host")
