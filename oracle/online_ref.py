"""numpy restatement of the reference online path (TEST INFRASTRUCTURE ONLY).

Each function cites the reference lines it follows.  Arithmetic order is kept
where it is observable (affine combine, weighting, explicit residual).
"""
from __future__ import annotations

import math

import numpy as np
import scipy.linalg as sla
import scipy.sparse as sp

DEFAULT_RTOL = 1e-12  # linalg.py:15


class OracleRankDeficiency(Exception):
    pass


def solve_ls(m, rhs, weights=None, rtol=DEFAULT_RTOL):
    """linalg.py:89-113: weighted Householder LS with the 1e-12 rank test."""
    m = np.asarray(m)
    if m.ndim == 1:
        m = m[:, None]
    if not np.all(np.isfinite(m)):                       # linalg.py:36-37
        raise ValueError("matrix has non-finite entries")
    rhs = np.asarray(rhs)
    if rhs.shape[0] != m.shape[0]:
        raise ValueError("rhs length does not match row count")
    if m.shape[0] < m.shape[1]:
        raise ValueError("solve_ls requires rows >= cols")
    if weights is not None:                              # linalg.py:102-105
        weights = np.asarray(weights)
        m = m * weights[:, None]
        rhs = rhs * weights
    q, rmat = np.linalg.qr(m)                            # linalg.py:106
    diag = np.abs(np.diag(rmat))
    if diag.size and diag.min() < rtol * max(diag.max(), np.finfo(float).tiny):
        raise OracleRankDeficiency(int(np.argmin(diag)))  # linalg.py:107-112
    return sla.solve_triangular(rmat, q.conj().T @ rhs)  # linalg.py:113


def affine_combine(coeffs, blocks):
    """online.py:108-112: m = f0*B0; m = m + fk*Bk."""
    m = coeffs[0] * blocks[0]
    for f, blk in zip(coeffs[1:], blocks[1:]):
        m = m + f * blk
    return m


def affine_blocks(matrices, basis, indices):
    """online.py:78-85: blocks on unique rows, expanded by the inverse map."""
    uniq, inverse = np.unique(indices, return_inverse=True)
    return tuple(np.asarray(a[uniq] @ basis)[inverse] for a in matrices)


def gauss_rows(points, rows, sigma, ridge):
    """Rows of K_sigma + ridge I for d-dimensional points (the harness row
    oracle of config 2; _kernels.py:38-50 generalised from 1-D):
    D = sum_k (x_ik - x_jk)^2 sequentially, K = exp(-(D * inv)), inv = 1/(2 s s),
    ridge added to the diagonal entry."""
    rows = np.asarray(rows, dtype=np.int64)
    pts = np.asarray(points)
    d = np.zeros((rows.size, pts.shape[0]))
    for k in range(pts.shape[1]):
        df = pts[rows, k][:, None] - pts[None, :, k]
        d = d + df * df
    inv = 1.0 / (2.0 * sigma * sigma)
    out = np.exp(-(d * inv))
    for k, i in enumerate(rows):
        out[k, i] += ridge
    return out


def stencil_rows(op, p, rows):
    """Rows of the edge-midpoint FD operator (systems.py:306-334 in edge form):
    c_e = exp(sum_k p_k phi_k(mid_e)) / h^2 (sequential sum), diag = sum_e c_e,
    off-diagonal -c_e for interior neighbours.  Returns CSR (len(rows) x n)."""
    rows = np.asarray(rows, dtype=np.int64)
    nbr, phi = op.edges(rows)
    pv = np.asarray(p, dtype=float).ravel()
    arg = phi[..., 0] * pv[0]
    for k in range(1, pv.size):
        arg = arg + phi[..., k] * pv[k]
    c = np.exp(arg) / (op.h * op.h)
    diag = c[:, 0].copy()
    for e in range(1, c.shape[1]):
        diag = diag + c[:, e]
    m = rows.size
    ri = [np.arange(m)]
    ci = [rows]
    vv = [diag]
    for e in range(c.shape[1]):
        ok = nbr[:, e] >= 0
        ri.append(np.arange(m)[ok])
        ci.append(nbr[ok, e])
        vv.append(-c[ok, e])
    return sp.csr_matrix((np.concatenate(vv), (np.concatenate(ri), np.concatenate(ci))), shape=(m, op.n))


def sampled_rows(row_fn, basis, indices, p):
    """online.py:57-65: rows on unique indices, @ basis, expanded by inverse."""
    uniq, inverse = np.unique(indices, return_inverse=True)
    block = row_fn(p, uniq) @ basis
    return np.asarray(block)[inverse]


def solve_one(m, tb, weights, proj=None):
    """online.py:117-127: LS, explicit sampled residual, output value."""
    coeff = solve_ls(m, tb, weights=weights)
    resid = m @ coeff - tb
    if weights is not None:
        resid = resid * weights
    sres = float(np.linalg.norm(resid))
    out = None if proj is None else complex(proj @ coeff)
    return coeff, sres, out


def interval(r, s, est):
    """online.py:151-153."""
    eps = min(max(r * math.log(r) / s if r > 1 else 0.0, 0.0), 0.99)
    return est / (1.0 + eps), est / (1.0 - eps), eps


def relative_residual(a_matrix, x, b):
    """cli.py:285, 344-351."""
    return float(np.linalg.norm(a_matrix @ x - b) / max(np.linalg.norm(b), 1e-300))


def ls_floor(m, tb, weights, draws=4, seed=0, rows=None, basis=None, inverse=None):
    """Parity floor of the LS solution at one parameter: relative spread of the
    solution under 1-ulp relative perturbations of the data, i.e. how far two
    valid fp64 evaluations can disagree.  For row-oracle
    systems pass the operator rows (dense, unique rows), the basis and the
    inverse map: the perturbation is then applied to the row entries before the
    contraction with X, which is where the cancellation of stencil rows
    (diagonal ~ sum of off-diagonals) amplifies rounding."""
    rng = np.random.default_rng(seed)
    base = solve_ls(m, tb, weights=weights)
    nb = max(np.linalg.norm(base), 1e-300)
    worst = 0.0
    eps = np.finfo(float).eps
    for _ in range(draws):
        dt = 1.0 + eps * rng.choice([-1.0, 1.0], size=tb.shape)
        if rows is not None and hasattr(rows, "tocsr"):  # sparse rows: perturb the stored entries
            rr = rows.tocsr(copy=True)
            rr.data = rr.data * (1.0 + eps * rng.choice([-1.0, 1.0], size=rr.data.shape))
            mp = np.asarray(rr @ basis)[inverse]
        elif rows is not None:
            rr = np.asarray(rows)
            dr = 1.0 + eps * rng.choice([-1.0, 1.0], size=rr.shape)
            mp = np.asarray((rr * dr) @ basis)[inverse]
        else:
            mp = m * (1.0 + eps * rng.choice([-1.0, 1.0], size=m.shape))
        c = solve_ls(mp, tb * dt, weights=weights)
        worst = max(worst, np.linalg.norm(c - base) / nb)
    return worst
