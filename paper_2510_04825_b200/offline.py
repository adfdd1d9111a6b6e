"""Offline-phase inputs of the online path: snapshot basis X and row selector S.

The offline phase is not on the hot path (BASELINE.json north_star: "the
offline snapshot solves and subsample selection stay in the reference and are
timed separately").  On the GPU box the reference is not available, and its
SuperLU snapshot solves are impractical at the BASELINE sizes,
so this module restates the reference's offline recipe with the same
semantics and data types to produce X and S there:

  SnapshotBasis, build_snapshot(mode qr | pod(tol) | none)   snapshot.py:14-34, 79-134
  RowSelector, select_rows(strategy leverage | random)        subsample.py:22-67, 95-156
  choose_anchor                                               subsample.py:198-209
  save/load_snapshot, save/load_selector (reference formats)  snapshot.py:137-158, subsample.py:212-235

Snapshot solves use a harness solver per operator kind (documented in
DESIGN.md): sparse direct (scipy) for affine/stencil systems small enough for
it, dense Cholesky for the Gaussian kernel (torch on the GPU when available),
preconditioned CG on the GPU for large SPD stencils.  Each solve carries the
reference's residual guard (systems.py:187-222).
"""
from __future__ import annotations

import json
import math
from dataclasses import dataclass
from typing import Optional

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from .errors import ConfigError, NumericalError, RankDeficiencyError
from .systems import GaussianKernelOperator, StencilOperator

FULL_SOLVE_RTOL = 1e-10


@dataclass(frozen=True)
class SnapshotBasis:
    points: tuple
    raw: np.ndarray
    basis: np.ndarray
    singular_values: np.ndarray

    @property
    def n(self) -> int:
        return self.basis.shape[0]

    @property
    def rank(self) -> int:
        return self.basis.shape[1]


@dataclass(frozen=True)
class RowSelector:
    indices: np.ndarray
    n: int
    weights: Optional[np.ndarray] = None
    strategy: str = ""
    anchors: tuple = ()

    def __post_init__(self):
        object.__setattr__(self, "indices", np.asarray(self.indices, dtype=np.int64))
        if self.weights is not None:
            object.__setattr__(self, "weights", np.asarray(self.weights, dtype=float))
            if self.weights.shape != self.indices.shape:
                raise ValueError("weights/indices length mismatch")
            if np.any(self.weights <= 0):
                raise ValueError("weights must be positive")
        if self.indices.size and (self.indices.min() < 0 or self.indices.max() >= self.n):
            raise ValueError("selector index out of range")

    @property
    def size(self) -> int:
        return int(self.indices.size)

    def apply(self, m) -> np.ndarray:
        m = np.asarray(m)
        out = m[self.indices]
        if self.weights is not None:
            out = out * (self.weights[:, None] if out.ndim == 2 else self.weights)
        return out


# --------------------------------------------------------------------------
# snapshot solves
# --------------------------------------------------------------------------
def _guard(a_apply, a_norm, x, b, p):
    res = np.linalg.norm(a_apply(x) - b)
    floor = max(a_norm * np.linalg.norm(x) + np.linalg.norm(b), 1e-300)
    if not np.all(np.isfinite(x)) or res > FULL_SOLVE_RTOL * floor:
        raise NumericalError(f"full_solve residual {res:.3e} exceeds {FULL_SOLVE_RTOL:.0e} * "
                             f"(||A|| ||x|| + ||b||) at p={p}")


def _sparse_solve(a: sp.csr_matrix, b: np.ndarray, p):
    """spsolve with up to two refinement steps and the residual guard (systems.py:187-222)."""
    lu = spla.splu(a.tocsc())
    x = lu.solve(b.astype(np.result_type(a.dtype, b.dtype)))
    a_norm = spla.norm(a)
    floor = lambda x: max(a_norm * np.linalg.norm(x) + np.linalg.norm(b), 1e-300)
    res = np.linalg.norm(a @ x - b)
    for _ in range(2):
        if np.all(np.isfinite(x)) and res <= FULL_SOLVE_RTOL * floor(x):
            break
        x = x + lu.solve(b - a @ x)
        res = np.linalg.norm(a @ x - b)
    _guard(lambda v: a @ v, a_norm, x, b, p)
    return x


def _gauss_solve_all(op: GaussianKernelOperator, b: np.ndarray, points, device=None):
    """Dense Cholesky solves of (K_p + ridge I) x = b for every snapshot p."""
    xs = op.points
    n = xs.shape[0]
    cols = []
    if device is not None:
        import torch
        X = torch.from_numpy(xs).to(device)
        # D_ij = sum_k (x_ik - x_jk)^2, sequential in k (same order as the row oracle)
        D = torch.zeros((n, n), dtype=torch.float64, device=device)
        for k in range(xs.shape[1]):
            df = X[:, k][:, None] - X[:, k][None, :]
            D += df * df
        bt = torch.from_numpy(b).to(device)
        for p in points:
            inv = 1.0 / (2.0 * p * p)
            K = torch.exp(-(D * inv))
            K.diagonal().add_(op.ridge)
            L = torch.linalg.cholesky(K)
            x = torch.cholesky_solve(bt[:, None], L)[:, 0]
            res = torch.linalg.norm(K @ x - bt).item()
            fl = torch.linalg.norm(K).item() * torch.linalg.norm(x).item() + torch.linalg.norm(bt).item()
            if not math.isfinite(res) or res > FULL_SOLVE_RTOL * fl:
                raise NumericalError(f"snapshot solve failed at p={p}: residual {res:.3e}")
            cols.append(x.cpu().numpy())
            del K, L
        return cols
    import scipy.linalg as sla
    D = np.zeros((n, n))
    for k in range(xs.shape[1]):
        df = xs[:, k][:, None] - xs[:, k][None, :]
        D += df * df
    for p in points:
        inv = 1.0 / (2.0 * p * p)
        K = np.exp(-(D * inv))
        K[np.arange(n), np.arange(n)] += op.ridge
        x = sla.cho_solve(sla.cho_factor(K), b)
        _guard(lambda v: K @ v, np.linalg.norm(K), x, b, p)
        cols.append(x)
    return cols


def _stencil_tensors(system, device):
    """All nodes' neighbours (-1 on Dirichlet edges) and edge-midpoint basis
    values on the device (once per system)."""
    import torch
    op: StencilOperator = system.operator
    nbr, phi = op.edges(np.arange(op.n))
    return {"nbr": torch.from_numpy(nbr).to(device), "phi": torch.from_numpy(phi).to(device),
            "b": torch.from_numpy(np.asarray(system.b, dtype=float)).to(device)}


def _stencil_cg(system, p, device, tol=1e-11, maxiter=50_000, tensors=None):
    """Jacobi-preconditioned CG on the GPU for the SPD stencil operator, by
    libsas's fused CG kernels (k_cg.cuh, sas_cg_stencil: q = A p with the
    search-direction update fused in, then x/r/z updates with the dot
    products; no host round trip between iterations).  Stops at
    ||r|| <= tol ||b|| or, if that is below what fp64 CG can attain for this
    conditioning, once ||r|| <= 1e-12 (||A|| ||x|| + ||b||); the reference's
    full_solve guard ||r|| <= 1e-10 (||A|| ||x|| + ||b||) is then checked on
    the true residual (systems.py:205-221)."""
    import ctypes as C

    import torch

    from . import _capi
    op: StencilOperator = system.operator
    tz = tensors if tensors is not None else _stencil_tensors(system, device)
    pv = np.asarray(p, dtype=float).ravel()
    phi, nbr, b = tz["phi"], tz["nbr"], tz["b"]
    arg = phi[..., 0] * float(pv[0])
    for k in range(1, pv.size):
        arg = arg + phi[..., k] * float(pv[k])
    c = torch.exp(arg) / (op.h * op.h)
    del arg
    dg = c.sum(dim=1).contiguous()
    ct = torch.where(nbr >= 0, c, torch.zeros_like(c)).contiguous()
    del c
    bn = float(torch.linalg.norm(b))
    a_norm = float(torch.sqrt((dg * dg).sum() + (ct * ct).sum()))
    x = torch.empty_like(b)
    its, rn, xn = C.c_int32(0), C.c_double(0.0), C.c_double(0.0)
    lib = _capi.load()
    dev_index = b.device.index or 0
    st = torch.cuda.current_stream(b.device)
    _capi.check(lib.sas_cg_stencil(op.n, op.n_edges, _capi.ptr(dg), _capi.ptr(ct), _capi.ptr(nbr), _capi.ptr(b),
                                   _capi.ptr(x), tol, a_norm, maxiter, 50, dev_index, C.c_void_p(st.cuda_stream),
                                   C.byref(its), C.byref(rn), C.byref(xn)), "sas_cg_stencil")
    if not math.isfinite(rn.value) or rn.value > FULL_SOLVE_RTOL * (a_norm * xn.value + bn):
        raise NumericalError(f"CG snapshot solve failed at p={p}: residual {rn.value:.3e} after {its.value} "
                             f"iterations")
    return x.cpu().numpy()


def _affine_bicgstab(system, p, device, tol=1e-11, maxiter=40_000):
    """Jacobi-preconditioned BiCGSTAB on the GPU for a large affine (possibly
    complex, non-symmetric) A(p) = sum_k f_k(p) A_k (config 4's transfer-function
    sweep), in place of the reference's SuperLU solve (systems.py:187-222), by
    libsas's fused BiCGSTAB kernels (k_bicg.cuh, sas_bicgstab_csr: direction
    update, CSR SpMV with its dot products, vector updates; device-side
    fixed-order reductions, no host round trip between iterations).
    Stops at ||r|| <= tol ||b|| or, if fp64 cannot attain that, once the
    reference's full_solve guard ||r|| <= 1e-10 (||A|| ||x|| + ||b||) holds
    with a 100x margin; the guard is checked on the true residual."""
    import ctypes as C

    import torch

    from . import _capi
    a = system.matrix(p).tocsr()
    a.sort_indices()
    b_np = np.asarray(system.full_rhs(p))
    cplx_ = np.iscomplexobj(a.data) or np.iscomplexobj(b_np)
    npdt = np.complex128 if cplx_ else np.float64
    if a.nnz >= 2 ** 31:
        raise ConfigError("BiCGSTAB snapshot solve: nnz above 2^31")
    dev = torch.device(device)
    up = lambda arr: torch.from_numpy(np.ascontiguousarray(arr)).to(dev)
    rp, ci, va = up(a.indptr.astype(np.int32)), up(a.indices.astype(np.int32)), up(a.data.astype(npdt))
    d, b = up(a.diagonal().astype(npdt)), up(b_np.astype(npdt))
    x = torch.empty_like(b)
    a_norm = float(spla.norm(a))
    bn = float(np.linalg.norm(b_np))
    its, rn, xn = C.c_int32(0), C.c_double(0.0), C.c_double(0.0)
    lib = _capi.load()
    st = torch.cuda.current_stream(dev)
    _capi.check(lib.sas_bicgstab_csr(a.shape[0], _capi.ptr(rp), _capi.ptr(ci), _capi.ptr(va), _capi.ptr(d),
                                     _capi.ptr(b), _capi.ptr(x), _capi.SAS_C128 if cplx_ else _capi.SAS_F64, tol,
                                     a_norm, maxiter, 25, int(dev.index or 0), C.c_void_p(st.cuda_stream),
                                     C.byref(its), C.byref(rn), C.byref(xn)), "sas_bicgstab_csr")
    if not math.isfinite(rn.value) or rn.value > FULL_SOLVE_RTOL * max(a_norm * xn.value + bn, 1e-300):
        raise NumericalError(f"full_solve residual {rn.value:.3e} exceeds {FULL_SOLVE_RTOL:.0e} * "
                             f"(||A|| ||x|| + ||b||) at p={p} (BiCGSTAB, {its.value} iterations)")
    return x.cpu().numpy()


def snapshot_solves(system, points, device=None, prefer_cg: bool = False):
    """Columns x(p_i) = A(p_i)^{-1} b(p_i) with the harness solver for the system."""
    op = getattr(system, "operator", None)
    if isinstance(op, GaussianKernelOperator):
        return _gauss_solve_all(op, np.asarray(system.b, dtype=float), points, device)
    cols = []
    use_cg = isinstance(op, StencilOperator) and (prefer_cg or op.n > 200_000) and device is not None
    use_bicg = system.affine_terms is not None and system.n > 200_000 and device is not None
    tensors = _stencil_tensors(system, device) if use_cg else None
    for p in points:
        if use_cg:
            cols.append(_stencil_cg(system, p, device, tensors=tensors))
        elif use_bicg:
            cols.append(_affine_bicgstab(system, p, device))
        else:
            cols.append(_sparse_solve(system.matrix(p), system.full_rhs(p), p))
    return cols


def _parse_mode(mode):
    if isinstance(mode, tuple):
        name, tol = mode
        return name, float(tol)
    if isinstance(mode, str) and mode.startswith("pod(") and mode.endswith(")"):
        return "pod", float(mode[4:-1])
    if mode == "pod":
        return "pod", 1e-10
    return mode, 0.0


def orthonormalize(raw: np.ndarray, mode="qr"):
    """snapshot.py:107-123: thin SVD for sigma, then qr / pod(tol) / none."""
    _, sigma, _ = np.linalg.svd(raw, full_matrices=False)
    name, tol = _parse_mode(mode)
    if name == "qr":
        q, rmat = np.linalg.qr(raw)
        diag = np.abs(np.diag(rmat))
        if diag.size and diag.min() < 1e-12 * max(diag.max(), np.finfo(float).tiny):
            raise RankDeficiencyError(f"numerically rank-deficient: min |R_ii| = {diag.min():.3e}, "
                                      f"max |R_ii| = {diag.max():.3e}")
        basis = q
    elif name == "pod":
        w, s, _ = np.linalg.svd(raw, full_matrices=False)
        keep = s > tol * s[0] if s[0] > 0 else np.ones_like(s, dtype=bool)
        basis = w[:, :max(int(np.count_nonzero(keep)), 1)]
    elif name == "none":
        basis = raw
    else:
        raise ConfigError(f"unknown snapshot mode {mode!r}")
    return basis, sigma


def build_snapshot(system, points, mode="qr", device=None, prefer_cg: bool = False) -> SnapshotBasis:
    points = list(points)
    if not points:
        raise ConfigError("no snapshot points given")
    cols = snapshot_solves(system, points, device=device, prefer_cg=prefer_cg)
    raw = np.column_stack(cols)
    basis, sigma = orthonormalize(raw, mode)
    return SnapshotBasis(points=tuple(points), raw=raw, basis=basis, singular_values=sigma)


# --------------------------------------------------------------------------
# row selection (subsample.py:95-156, 198-209)
# --------------------------------------------------------------------------
def choose_anchor(points):
    pts = list(points)

    def key(p):
        vec = np.atleast_1d(np.asarray(p, dtype=complex))
        if vec.size > 1 or vec.imag.any():
            return float(np.linalg.norm(vec))
        return float(vec.real[0])

    order = sorted(range(len(pts)), key=lambda k: key(pts[k]))
    return pts[order[(len(pts) - 1) // 2]]


def _range_basis(target, rtol=1e-12):
    m = np.asarray(target)
    norms = np.linalg.norm(m, axis=0)
    norms = np.where(norms == 0, 1.0, norms)
    w, s, _ = np.linalg.svd(m / norms, full_matrices=False)
    if s[0] == 0:
        raise RankDeficiencyError("zero matrix has no range basis")
    keep = max(int(np.count_nonzero(s > rtol * s[0])), 1)
    return w[:, :keep]


def leverage_scores(q) -> np.ndarray:
    q = np.asarray(q)
    r = q.shape[1]
    gram = q.conj().T @ q
    if np.linalg.norm(gram - np.eye(r)) > 1e-8:
        raise ValueError("leverage_scores needs orthonormal columns")
    return np.einsum("ij,ij->i", q.conj(), q).real


def leverage_scores_gpu(target, device=0, rtol=1e-12, max_passes=4):
    """Leverage scores of the numerical range of a tall `target` on the GPU with
    libsas kernels (subsample.py:84-94 + 144-159 without the n x w host SVD):

      R = TSQR(target)                      sas_tsqr_r (column norms = ||R[:, j]||)
      R diag(1/norms) = U S V^H             w x w host SVD; keep s_j > rtol s_0
      C = diag(1/norms) V_k S_k^-1          so that W = target C = U_k in exact arithmetic
      repeat: (W, scores) = range_rows(target, C); R2 = TSQR(W);
              done if ||R2^H R2 - I|| <= 1e-10, else C <- C R2^-1

    W from the first pass is orthonormal only to eps s_0 / s_k; one more pass
    brings it to rounding.  The final ||W^H W - I|| takes the place of the
    reference's 1e-8 orthonormality check.  The scores are those of the SAME
    subspace the reference's thin SVD spans; they agree with it to the
    conditioning of that subspace (about eps s_0 / s_k), not bit for bit.
    Returns (scores as a CUDA tensor, kept rank)."""
    import ctypes as C_
    import torch
    from . import _capi
    dev = torch.device(f"cuda:{device}" if isinstance(device, int) else device)
    A = target if isinstance(target, torch.Tensor) else torch.from_numpy(np.ascontiguousarray(target))
    A = A.to(dev).contiguous()
    m, w = A.shape
    if w > 64:
        raise ConfigError("leverage_scores_gpu: width above 64")
    lib = _capi.load()
    dt = _capi.SAS_C128 if A.is_complex() else _capi.SAS_F64
    npdt = np.complex128 if A.is_complex() else np.float64
    st = C_.c_void_p(torch.cuda.current_stream(dev).cuda_stream)
    di = int(dev.index or 0)

    def tsqr(M):
        R = torch.empty((M.shape[1], M.shape[1]), dtype=M.dtype, device=dev)
        _capi.check(lib.sas_tsqr_r(_capi.ptr(M), M.shape[0], M.shape[1], dt, _capi.ptr(R), di, st), "sas_tsqr_r")
        return np.triu(R.cpu().numpy())

    R = tsqr(A)
    norms = np.linalg.norm(R, axis=0)
    norms = np.where(norms == 0, 1.0, norms)
    _, sv, vh = np.linalg.svd(R / norms)
    if sv[0] == 0:
        raise RankDeficiencyError("zero matrix has no range basis")
    keep = max(int(np.count_nonzero(sv > rtol * sv[0])), 1)
    Cm = (vh[:keep].conj().T / sv[:keep]) / norms[:, None]
    scores = torch.empty(m, dtype=torch.float64, device=dev)
    W = torch.empty((m, keep), dtype=A.dtype, device=dev)
    err = np.inf
    for _ in range(max_passes):
        Ch = np.ascontiguousarray(Cm, dtype=npdt)
        _capi.check(lib.sas_range_rows(_capi.ptr(A), m, w, Ch.ctypes.data_as(C_.c_void_p), keep, dt, _capi.ptr(W),
                                       _capi.ptr(scores), di, st), "sas_range_rows")
        R2 = tsqr(W)
        err = float(np.linalg.norm(R2.conj().T @ R2 - np.eye(keep)))
        if err <= 1e-10:
            break
        Cm = np.linalg.solve(R2.T, Cm.T).T    # C R2^-1
    if not err <= 1e-8:
        raise ValueError("leverage_scores needs orthonormal columns")
    return scores, keep


def select_rows(b, rhs=None, strategy="leverage", oversample=4.0, augment_rhs=True, seed=0,
                rng=None, anchors=(), device=None) -> RowSelector:
    """device=None: the host restatement (bit-identical to the reference's S and
    weights).  device=<cuda>: the leverage scores come from the GPU kernels
    (leverage_scores_gpu); the draw itself (numpy's rng.choice on the n
    probabilities) stays the reference's."""
    b_t = b if device is not None and not isinstance(b, np.ndarray) else None
    if b_t is None:
        b = np.asarray(b)
    n, _ = b.shape
    if rng is None:
        rng = np.random.default_rng(seed)
    if device is not None and strategy == "leverage":
        import torch
        bt = b_t if b_t is not None else torch.from_numpy(np.ascontiguousarray(b))
        bt = bt.to(device)
        if augment_rhs and rhs is not None:
            rt = torch.as_tensor(np.asarray(rhs)).to(device)
            dtp = torch.promote_types(bt.dtype, rt.dtype)
            bt = torch.cat([bt.to(dtp), rt.to(dtp)[:, None]], dim=1)
        width = bt.shape[1]
        s = int(math.ceil(oversample * width))
        scores_t, _ = leverage_scores_gpu(bt, device=device)
        scores = scores_t.cpu().numpy()
        total = scores.sum()
        if total <= 0:
            raise RankDeficiencyError("all-zero leverage scores")
        pi = scores / total
        idx = rng.choice(n, size=s, replace=True, p=pi)
        weights = 1.0 / np.sqrt(s * pi[idx])
        return RowSelector(indices=idx, n=n, weights=weights, strategy=strategy, anchors=tuple(anchors))
    target = b
    if augment_rhs and rhs is not None:
        target = np.column_stack([b, np.asarray(rhs)])
    width = target.shape[1]
    s = int(math.ceil(oversample * width))
    if strategy == "random":
        s = min(s, n)
        idx = np.sort(rng.choice(n, size=s, replace=False))
        return RowSelector(indices=idx, n=n, strategy=strategy, anchors=tuple(anchors))
    if strategy == "leverage":
        q = _range_basis(target)
        scores = leverage_scores(q)
        total = scores.sum()
        if total <= 0:
            raise RankDeficiencyError("all-zero leverage scores")
        pi = scores / total
        idx = rng.choice(n, size=s, replace=True, p=pi)
        weights = 1.0 / np.sqrt(s * pi[idx])
        return RowSelector(indices=idx, n=n, weights=weights, strategy=strategy, anchors=tuple(anchors))
    raise ConfigError(f"strategy {strategy!r} is not restated here (use the reference's select_rows)")


def anchor_product(system, anchor, basis, device=None) -> np.ndarray:
    """B = A(anchor) Q_X (cli.py:247)."""
    op = getattr(system, "operator", None)
    X = np.asarray(basis)
    if isinstance(op, GaussianKernelOperator):
        xs = op.points
        n = xs.shape[0]
        inv = 1.0 / (2.0 * anchor * anchor)
        if device is not None:
            import torch
            P = torch.from_numpy(xs).to(device)
            D = torch.zeros((n, n), dtype=torch.float64, device=device)
            for k in range(xs.shape[1]):
                df = P[:, k][:, None] - P[:, k][None, :]
                D += df * df
            K = torch.exp(-(D * inv))
            K.diagonal().add_(op.ridge)
            return (K @ torch.from_numpy(X).to(device)).cpu().numpy()
        D = np.zeros((n, n))
        for k in range(xs.shape[1]):
            df = xs[:, k][:, None] - xs[:, k][None, :]
            D += df * df
        K = np.exp(-(D * inv))
        K[np.arange(n), np.arange(n)] += op.ridge
        return K @ X
    return np.asarray(system.matrix(anchor) @ X)


def offline(problem, device=None, prefer_cg=False, basis: Optional[SnapshotBasis] = None,
            gpu_select: bool = False):
    """Full offline recipe of a problems.Problem: snapshot basis, anchor,
    leverage selector with `samples` rows (cli.py:239-265).  gpu_select: the
    selector's leverage scores from the GPU kernels (select_rows(device=...))
    instead of the host thin SVD."""
    system = problem.system
    if basis is None:
        basis = build_snapshot(system, problem.snapshot_points, problem.snapshot_mode, device=device,
                               prefer_cg=prefer_cg)
    anchor = choose_anchor(basis.points)
    b_anchor = anchor_product(system, anchor, basis.basis, device=device)
    rhs_anchor = system.full_rhs(anchor)
    width = basis.rank + 1
    sel = select_rows(b_anchor, rhs_anchor, strategy="leverage", oversample=problem.samples / width,
                      seed=problem.selector_seed, anchors=(anchor,),
                      device=(device if gpu_select and device is not None else None))
    if sel.size != problem.samples:
        raise ConfigError(f"selector size {sel.size} != requested samples {problem.samples}")
    return basis, sel


# --------------------------------------------------------------------------
# artifacts in the reference's formats
# --------------------------------------------------------------------------
def save_snapshot(path, basis: SnapshotBasis) -> None:
    pts = np.array([np.atleast_1d(np.asarray(p, dtype=complex)) for p in basis.points])
    np.savez_compressed(path, points=pts, raw=basis.raw, basis=basis.basis,
                        singular_values=basis.singular_values)


def load_snapshot(path) -> SnapshotBasis:
    data = np.load(path)
    points = []
    for row in data["points"]:
        row = np.atleast_1d(row)
        if row.size == 1:
            val = complex(row[0])
            points.append(val.real if val.imag == 0 else val)
        else:
            points.append(tuple(complex(v).real if complex(v).imag == 0 else complex(v) for v in row))
    return SnapshotBasis(points=tuple(points), raw=data["raw"], basis=data["basis"],
                         singular_values=data["singular_values"])


def save_selector(path, selector: RowSelector) -> None:
    payload = {"n": selector.n, "indices": [int(i) for i in selector.indices],
               "weights": None if selector.weights is None else [float(w) for w in selector.weights],
               "strategy": selector.strategy, "anchors": [repr(a) for a in selector.anchors]}
    with open(path, "w") as fh:
        json.dump(payload, fh, indent=1)


def load_selector(path) -> RowSelector:
    with open(path) as fh:
        payload = json.load(fh)
    return RowSelector(indices=np.array(payload["indices"], dtype=np.int64), n=int(payload["n"]),
                       weights=None if payload["weights"] is None else np.array(payload["weights"], dtype=float),
                       strategy=payload["strategy"], anchors=tuple(payload["anchors"]))
