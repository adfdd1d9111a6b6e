"""Online phase on the GPU — drop-in for subapsnap.online.

Same public names, argument order, return types and error behaviour as
/root/reference/pkg/src/subapsnap/online.py:

  precompute_online(system, basis, selector) -> OnlinePlan      (online.py:68-102)
  solve_online(plan, p, want_interval=False) -> OnlineSolution  (online.py:105-134)
  solve_batch(plan, parameters, want_interval=False, workers=1) (online.py:208-225)
  estimate_residual(plan, solution)                            (online.py:137-153)
  OnlineSolution.lift()                                        (online.py:50-54)
  save_plan / load_plan                                        (online.py:168-195)

plus the columnar batch API the GPU needs (per-p Python objects would cost
more than the solve itself):

  solve_params(plan, parameters) -> BatchResult       (host arrays in/out)
  solve_device(plan, params_tensor, ...) -> tensors   (device-resident, torch)
  lift_batch(plan, coefficients) -> x (P x n)
  relative_residual(plan, parameters, coefficients)   (cli.py:344-351 checker)

Every numerical step of the per-parameter solve runs in libsas.so; this
module only marshals arguments.
"""
from __future__ import annotations

import ctypes as C
import math
import time
import warnings
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _capi
from .errors import BackendError, RankDeficiencyError
from .systems import GaussianKernelOperator, StencilOperator

PLAN_CHECK_RTOL = 1e-10   # online.py:93 (affine blocks vs the row oracle)


# --------------------------------------------------------------------------
# GPU plan (owner of the libsas handle)
# --------------------------------------------------------------------------
_KIND_CODES = {"const": _capi.SAS_COEF_CONST, "linear": _capi.SAS_COEF_LINEAR,
               "exp": _capi.SAS_COEF_EXP}


def params_to_array(parameters, dp: int, pcomplex: bool) -> np.ndarray:
    """Parameter list (floats, complex numbers or d_p-tuples, as the reference
    accepts them, systems.py:61-65) -> the C-ABI layout: P x d_p doubles, or
    P x d_p x 2 (re, im) for complex-parameter plans."""
    vals = [np.atleast_1d(np.asarray(p, dtype=complex)).ravel() for p in parameters]
    if any(v.size != dp for v in vals):
        raise ValueError(f"parameters must have {dp} component(s)")
    arr = np.array(vals, dtype=complex).reshape(len(vals), dp)
    if pcomplex:
        return np.ascontiguousarray(np.stack([arr.real, arr.imag], axis=-1))
    if len(vals) and np.any(arr.imag != 0):
        raise ValueError("complex parameter for a real-parameter plan")
    return np.ascontiguousarray(arr.real)


def is_cuda_tensor(a) -> bool:
    return hasattr(a, "data_ptr") and getattr(a, "is_cuda", False)


def row_operator(system):
    """The GPU row operator of a non-affine system: our `operator` attribute,
    or, for the reference's own KRR system (systems.py:423-463: row_fn =
    _kernels.rbf_rows over the 1-D training points, p = (lambda, sigma)), the
    equivalent Gaussian-kernel descriptor."""
    op = getattr(system, "operator", None)
    if op is not None:
        return op
    ex = getattr(system, "extras", None) or {}
    if getattr(system, "name", "") == "krr" and "t_train" in ex and system.affine_terms is None:
        pts = np.ascontiguousarray(np.asarray(ex["t_train"], dtype=np.float64).reshape(-1, 1))
        return GaussianKernelOperator(points=pts, ridge=0.0, ridge_from_param=True)
    return None


def probe_point(system, basis=None):
    """A parameter value inside the system's domain: the basis' first snapshot
    point (the point the reference's plan spot check uses, online.py:87), else
    the domain's lower corner."""
    pts = getattr(basis, "points", None)
    if pts is not None and len(pts):
        return pts[0]
    axes = system.domain.axes
    vals = [(1j * a.lo if a.imag else a.lo) for a in axes]
    return vals[0] if len(vals) == 1 else tuple(vals)


class GpuPlan:
    """libsas plan for one (system, basis, selector) on one CUDA device."""

    def __init__(self, system, basis, selector, blocks, proj, device: int = 0,
                 force_complex: bool = False):
        self.lib = _capi.load()
        self.system = system
        self.device = int(device)
        Xb = basis.basis
        self.x_device = is_cuda_tensor(Xb)
        X = Xb if self.x_device else np.asarray(Xb)
        self.n, self.r = X.shape
        idx = np.ascontiguousarray(selector.indices, dtype=np.int64)
        self.s = idx.size
        self.dp = int(system.domain.dim) if hasattr(system, "domain") else 1
        self.pcomplex = bool(getattr(system.domain, "axes", None) and any(a.imag for a in system.domain.axes))
        terms = system.affine_terms
        complex_data = ((X.is_complex() if self.x_device else np.iscomplexobj(X)) or force_complex or self.pcomplex
                        or (blocks is not None and any(np.iscomplexobj(b) for b in blocks))
                        or (proj is not None and np.iscomplexobj(proj)))
        if terms is not None:
            for t in terms:
                for v in (getattr(t, "scale", 0.0), getattr(t, "rate", 0.0)):
                    if complex(v).imag != 0.0:
                        complex_data = True
        self.rhs_constant = getattr(system, "rhs_constant", None)
        if self.rhs_constant is None:  # duck-typed reference system: rhs_fn is opaque
            self.rhs_constant = False
        if self.rhs_constant and np.iscomplexobj(system.b):
            complex_data = True
        # opaque callables (kind "other" coefficients, rhs_fn) are evaluated on the
        # host per parameter; probe them once at a domain point so a complex value
        # on a real-parameter domain selects a complex plan (the reference computes
        # such systems in complex128, online.py:108-117)
        if not complex_data:
            p0 = probe_point(system, basis)
            if terms is not None:
                for t in terms:
                    if getattr(t, "kind", "other") not in _KIND_CODES and complex(t.coeff(p0)).imag != 0.0:
                        complex_data = True
            if not self.rhs_constant and np.iscomplexobj(np.asarray(system.rhs(p0, idx[:1]))):
                complex_data = True
        self.complex = bool(complex_data)
        self.np_dtype = np.complex128 if self.complex else np.float64
        # the reference coerces const/linear coefficients to complex (systems.py:92, 98):
        # keep its result dtype for duck-typed systems whose scales are Python complex
        self.result_dtype = self.np_dtype
        if terms is not None and any(isinstance(getattr(t, "scale", None), complex) for t in terms):
            self.result_dtype = np.complex128

        desc = _capi.SasDesc()
        desc.dtype = _capi.SAS_C128 if self.complex else _capi.SAS_F64
        desc.param_dim = self.dp
        desc.param_complex = 1 if self.pcomplex else 0
        keep = []  # keep host arrays alive during the call
        self.table_terms = []
        op = row_operator(system)
        if terms is not None:
            K = len(terms)
            kinds = np.zeros(K, dtype=np.int32)
            scales = np.zeros((K, 2))
            rates = np.zeros((K, 2))
            for k, t in enumerate(terms):
                kind = getattr(t, "kind", "other")
                if kind in _KIND_CODES:
                    kinds[k] = _KIND_CODES[kind]
                    sc = complex(getattr(t, "scale", 1.0))
                    rt = complex(getattr(t, "rate", 0.0))
                    scales[k] = (sc.real, sc.imag)
                    rates[k] = (rt.real, rt.imag)
                else:
                    kinds[k] = _capi.SAS_COEF_TABLE
                    self.table_terms.append(k)
            blk = np.ascontiguousarray(np.stack([np.asarray(b) for b in blocks]).astype(self.np_dtype))
            keep += [kinds, scales, rates, blk]
            desc.op_kind = _capi.SAS_OP_AFFINE
            desc.n_terms = K
            desc.term_kind = kinds.ctypes.data_as(C.POINTER(C.c_int32))
            desc.term_scale = scales.ctypes.data_as(C.POINTER(C.c_double))
            desc.term_rate = rates.ctypes.data_as(C.POINTER(C.c_double))
            desc.blocks = C.c_void_p(blk.ctypes.data)
            self.K = K
        elif isinstance(op, StencilOperator):
            nbr, phi = op.edges(idx)
            keep += [nbr, phi]
            desc.op_kind = _capi.SAS_OP_STENCIL
            desc.n_edges = op.n_edges
            desc.edge_nbr = nbr.ctypes.data_as(C.POINTER(C.c_int64))
            desc.edge_phi = phi.ctypes.data_as(C.POINTER(C.c_double))
            desc.edge_div = op.h * op.h
            self.K = 0
        elif isinstance(op, GaussianKernelOperator):
            pts = np.ascontiguousarray(op.points, dtype=np.float64)
            keep.append(pts)
            desc.op_kind = _capi.SAS_OP_GAUSS
            desc.points = pts.ctypes.data_as(C.POINTER(C.c_double))
            desc.point_dim = pts.shape[1]
            desc.ridge = float(op.ridge)
            self.K = 0
        else:
            raise ValueError("system has neither affine terms nor a GPU row operator")

        flags = 0
        if self.x_device:  # e.g. the NCCL-broadcast basis: no host round trip
            import torch
            Xc = X.to(device=f"cuda:{self.device}",
                      dtype=torch.complex128 if self.complex else torch.float64).contiguous()
            flags |= _capi.SAS_FLAG_INPUT_DEVICE
            torch.cuda.synchronize(self.device)
        else:
            Xc = np.ascontiguousarray(X.astype(self.np_dtype, copy=False))
        w = None if selector.weights is None else np.ascontiguousarray(selector.weights, dtype=np.float64)
        if self.rhs_constant:
            t = np.ascontiguousarray(np.asarray(system.b)[idx].astype(self.np_dtype))
        else:
            t = np.zeros(self.s, dtype=self.np_dtype)
        pj = None if proj is None else np.ascontiguousarray(np.asarray(proj).astype(self.np_dtype))
        keep += [Xc, w, t, pj, idx]
        handle = C.c_void_p()
        rc = self.lib.sas_plan_create(C.byref(desc), _capi.ptr(Xc), self.n, self.r,
                                      idx.ctypes.data_as(C.POINTER(C.c_int64)),
                                      None if w is None else w.ctypes.data_as(C.POINTER(C.c_double)),
                                      self.s, _capi.ptr(t), _capi.ptr(pj), self.device, flags, C.byref(handle))
        _capi.check(rc, "sas_plan_create")
        self.handle = handle
        self.has_proj = proj is not None
        self.indices = idx
        self._operator_set = False

    # -- argument marshalling ------------------------------------------------
    def params_array(self, parameters) -> np.ndarray:
        return params_to_array(parameters, self.dp, self.pcomplex)

    def coef_table(self, parameters) -> Optional[np.ndarray]:
        if not self.table_terms:
            return None
        tab = np.zeros((len(parameters), self.K, 2))
        for i, p in enumerate(parameters):
            for k in self.table_terms:
                v = complex(self.system.affine_terms[k].coeff(p))
                if v.imag != 0.0 and not self.complex:
                    raise ValueError(f"affine term {k} has a complex coefficient at p={p} on a real plan")
                tab[i, k] = (v.real, v.imag)
        return tab

    def rhs_table(self, parameters) -> Optional[np.ndarray]:
        if self.rhs_constant:
            return None
        rows = np.stack([np.asarray(self.system.rhs(p, self.indices)) for p in parameters])
        if not self.complex and np.iscomplexobj(rows) and np.any(rows.imag != 0):
            raise ValueError("complex right-hand side on a real plan")
        return np.ascontiguousarray(rows.astype(self.np_dtype))

    # -- calls -----------------------------------------------------------------
    def solve_host(self, parameters):
        P = len(parameters)
        pa = self.params_array(parameters)
        ct = self.coef_table(parameters)
        rt = self.rhs_table(parameters)
        coef = np.empty((P, self.r), dtype=self.np_dtype)
        sres = np.empty(P)
        outv = np.empty((P, 2))
        status = np.empty(P, dtype=np.int32)
        bad = np.empty(P, dtype=np.int32)
        rc = self.lib.sas_solve_host(self.handle, _capi.ptr(pa), P, _capi.ptr(ct), _capi.ptr(rt),
                                     _capi.ptr(coef), _capi.ptr(sres), _capi.ptr(outv), _capi.ptr(status),
                                     _capi.ptr(bad))
        _capi.check(rc, "sas_solve_host")
        return coef, sres, outv[:, 0] + 1j * outv[:, 1], status, bad

    def launches(self) -> int:
        return int(self.lib.sas_last_launch_count(self.handle))

    def set_timing(self, enable: bool):
        _capi.check(self.lib.sas_plan_set_timing(self.handle, 1 if enable else 0), "sas_plan_set_timing")

    def stage_times(self, cap: int = 4096):
        """[(stage_id, ms)] for every kernel of the last solve (needs set_timing(True))."""
        ms = (C.c_float * cap)()
        st = (C.c_int32 * cap)()
        n = self.lib.sas_stage_times(self.handle, ms, st, cap)
        return [(int(st[i]), float(ms[i])) for i in range(max(n, 0))]

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            self.lib.sas_plan_destroy(self.handle)
            self.handle = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------
# reference data types (online.py:26-54, 198-205)
# --------------------------------------------------------------------------
@dataclass(frozen=True)
class OnlinePlan:
    system: object
    basis: object
    selector: object
    blocks: Optional[tuple]          # per affine term, s x r' (unweighted)
    sampled_basis: np.ndarray        # S Q_X, s x r'
    output_projection: Optional[np.ndarray]  # c^H Q_X
    gpu: Optional[GpuPlan] = field(default=None, repr=False, compare=False)

    @property
    def affine(self) -> bool:
        return self.blocks is not None


@dataclass
class OnlineSolution:
    parameter: object
    coefficients: np.ndarray
    sampled_residual: float
    residual_interval: Optional[tuple] = None
    output_value: Optional[complex] = None
    _basis: object = field(default=None, repr=False)
    _lifted: Optional[np.ndarray] = field(default=None, repr=False)
    _plan: object = field(default=None, repr=False)

    def lift(self) -> np.ndarray:
        """x = Q_X c, computed on the GPU (libsas sas_lift), cached."""
        if self._lifted is None:
            if self._plan is None:
                raise BackendError("solution has no device plan to lift with")
            self._lifted = lift_batch(self._plan, self.coefficients[None, :])[0]
        return self._lifted


@dataclass(frozen=True)
class BatchRow:
    parameter: object
    sampled_residual: float
    residual_interval: Optional[tuple]
    output_value: Optional[complex]
    wall_time: float
    solution: OnlineSolution


@dataclass
class BatchResult:
    """Columnar results of solve_params (input order)."""

    parameters: list
    coefficients: np.ndarray      # P x r'
    sampled_residual: np.ndarray  # P
    output_value: Optional[np.ndarray]  # P complex, or None
    status: np.ndarray            # P int32 (0 ok, 1 rank-deficient, 2 non-finite)
    bad_column: np.ndarray        # P int32
    seconds: float


# --------------------------------------------------------------------------
def _rows_times_basis(m, X):
    """(sparse rows m) @ X for a host array X, or for a CUDA tensor X by
    gathering only the rows of X that m touches (same entries in the same
    stored order, so the products match m @ X_host)."""
    import scipy.sparse as sp
    m = sp.csr_matrix(m)
    if not is_cuda_tensor(X):
        return np.asarray(m @ X)
    import torch
    cols = np.unique(m.indices)
    xs = X[torch.from_numpy(cols).to(X.device)].cpu().numpy()
    sub = sp.csr_matrix((m.data, np.searchsorted(cols, m.indices), m.indptr), shape=(m.shape[0], cols.size))
    return np.asarray(sub @ xs)


def _spot_check(system, basis, idx, uniq, inverse, blocks):
    """The reference's plan check (online.py:86-96): at basis.points[0] the
    combined affine blocks must match a direct row-oracle assembly to 1e-10
    relative, else RankDeficiencyError.  The direct rows come from the
    system's own row oracle when it has one (reference ParametricSystem.rows,
    systems.py:134-149), else from the affine terms row by row."""
    p0 = probe_point(system, basis)
    if hasattr(system, "rows"):
        rows = system.rows(p0, uniq)
    else:
        rows = None
        for term in system.affine_terms:
            blk = term.matrix[uniq] * term.coeff(p0)
            rows = blk if rows is None else rows + blk
    direct = _rows_times_basis(rows, basis.basis)[inverse]
    combined = sum(term.coeff(p0) * blk for term, blk in zip(system.affine_terms, blocks))
    err = np.linalg.norm(combined - direct)
    ref = max(np.linalg.norm(direct), 1e-300)
    if err > PLAN_CHECK_RTOL * ref:
        raise RankDeficiencyError(f"affine blocks disagree with row oracle (rel err {err / ref:.2e})")


def precompute_online(system, basis, selector, device: int = 0) -> OnlinePlan:
    """Precompute the selector-row blocks of each affine term (host, as the
    reference does, online.py:77-85), run the reference's spot check
    (online.py:86-96) and build the device plan.  `basis.basis` may be a host
    array or a CUDA tensor (e.g. the NCCL-broadcast basis, parallel.py); only
    the rows the blocks touch are then read back."""
    if basis.n != system.n or selector.n != system.n:
        raise ValueError("system/basis/selector dimension mismatch")
    idx = np.asarray(selector.indices, dtype=np.int64)
    uniq, inverse = np.unique(idx, return_inverse=True)
    X = basis.basis
    if is_cuda_tensor(X):
        import torch
        sampled_basis = X[torch.from_numpy(idx).to(X.device)].cpu().numpy()
    else:
        sampled_basis = np.asarray(X)[idx]
    blocks = None
    if system.affine_terms is not None:
        blocks = tuple(_rows_times_basis(term.matrix[uniq], X)[inverse] for term in system.affine_terms)
        _spot_check(system, basis, idx, uniq, inverse, blocks)
    proj = None
    if system.output_functional is not None:
        if is_cuda_tensor(X):
            import torch
            c = torch.from_numpy(np.ascontiguousarray(np.asarray(system.output_functional).conj())).to(X.device)
            proj = (c.to(torch.promote_types(c.dtype, X.dtype)) @ X.to(torch.promote_types(c.dtype, X.dtype))).cpu().numpy()
        else:
            proj = system.output_functional.conj() @ X
    gpu = GpuPlan(system, basis, selector, blocks, proj, device=device)
    return OnlinePlan(system=system, basis=basis, selector=selector, blocks=blocks,
                      sampled_basis=sampled_basis, output_projection=proj, gpu=gpu)


def _gpu(plan: OnlinePlan) -> GpuPlan:
    if plan.gpu is None:
        raise BackendError("plan has no device plan (load_plan/precompute_online builds one)")
    return plan.gpu


def solve_params(plan: OnlinePlan, parameters) -> BatchResult:
    """Solve many parameters in one GPU call; results in input order."""
    parameters = list(parameters)
    g = _gpu(plan)
    t0 = time.perf_counter()
    coef, sres, outv, status, bad = g.solve_host(parameters)
    dt = time.perf_counter() - t0
    coef = coef.astype(g.result_dtype, copy=False)
    return BatchResult(parameters=parameters, coefficients=coef, sampled_residual=sres,
                       output_value=outv if g.has_proj else None, status=status, bad_column=bad,
                       seconds=dt)


def _raise_for_status(res: BatchResult):
    bad = np.nonzero(res.status)[0]
    if bad.size == 0:
        return
    k = int(bad[0])
    p = res.parameters[k]
    if res.status[k] == _capi.SAS_ST_RANK_DEFICIENT:
        raise RankDeficiencyError(
            f"subsampled system rank-deficient at p={p}: "
            f"rank-deficient least-squares matrix at column {int(res.bad_column[k])}")
    raise ValueError("matrix has non-finite entries")


def _interval(plan: OnlinePlan, est):
    sel = plan.selector
    r = plan.basis.rank
    eps = min(max(r * math.log(r) / sel.size if r > 1 else 0.0, 0.0), 0.99)
    return est / (1.0 + eps), est / (1.0 - eps)


def _solution(plan, res: BatchResult, k: int, want_interval: bool) -> OnlineSolution:
    out = None if res.output_value is None else complex(res.output_value[k])
    sol = OnlineSolution(parameter=res.parameters[k], coefficients=res.coefficients[k].copy(),
                         sampled_residual=float(res.sampled_residual[k]), output_value=out,
                         _basis=plan.basis, _plan=plan)
    if want_interval and plan.selector.weights is not None:
        _, lower, upper, _ = estimate_residual(plan, sol)
        sol.residual_interval = (lower, upper)
    return sol


def solve_online(plan: OnlinePlan, p, want_interval: bool = False) -> OnlineSolution:
    """Solve the weighted subsampled least-squares problem at parameter p."""
    res = solve_params(plan, [p])
    _raise_for_status(res)
    return _solution(plan, res, 0, want_interval)


def estimate_residual(plan: OnlinePlan, solution: OnlineSolution):
    """Heuristic residual interval (online.py:137-153)."""
    sel = plan.selector
    r = plan.basis.rank
    if sel.weights is None:
        raise ValueError("residual estimation requires a weighted selector")
    if sel.size <= r:
        raise ValueError("residual estimation requires oversampling (s > r)")
    eps = min(max(r * math.log(r) / sel.size if r > 1 else 0.0, 0.0), 0.99)
    est = solution.sampled_residual
    return est, est / (1.0 + eps), est / (1.0 - eps), eps


def solve_batch(plan: OnlinePlan, parameters, want_interval: bool = False, workers: int = 1) -> list:
    """Solve many parameters; rows come back in input order.  One batched GPU
    call; `workers` is accepted for API compatibility (the GPU batch replaces
    the reference's thread pool, online.py:222-224).  wall_time is the batch
    time divided evenly over its parameters."""
    parameters = list(parameters)
    if not parameters:
        return []
    res = solve_params(plan, parameters)
    _raise_for_status(res)
    per = res.seconds / len(parameters)
    rows = []
    for k, p in enumerate(parameters):
        sol = _solution(plan, res, k, want_interval)
        rows.append(BatchRow(parameter=p, sampled_residual=sol.sampled_residual,
                             residual_interval=sol.residual_interval, output_value=sol.output_value,
                             wall_time=per, solution=sol))
    return rows


def _operator_times_basis(system, X, p, dev):
    """B = A(p) X on the GPU (torch), for the full least squares of solve_apsnap."""
    import torch
    op = getattr(system, "operator", None)
    if system.affine_terms is not None:
        fs = [complex(t.coeff(p)) for t in system.affine_terms]
        cplx_ = X.is_complex() or np.iscomplexobj(p) or any(f.imag != 0.0 for f in fs)
        cdt = torch.complex128 if cplx_ else torch.float64
        B = torch.zeros(X.shape, dtype=cdt, device=dev)
        for t in system.affine_terms:
            m = t.matrix.tocsr()
            with warnings.catch_warnings():  # torch's beta/invariant notices for CSR tensors
                warnings.filterwarnings("ignore", message="Sparse", category=UserWarning)
                A = torch.sparse_csr_tensor(torch.from_numpy(m.indptr.astype(np.int64)),
                                            torch.from_numpy(m.indices.astype(np.int64)),
                                            torch.from_numpy(m.data.astype(np.complex128 if cdt == torch.complex128
                                                                           else np.float64)),
                                            size=m.shape, device=dev, check_invariants=True)
            f = fs[system.affine_terms.index(t)]
            B += (f if cdt == torch.complex128 else f.real) * (A @ X.to(cdt))
        return B
    if isinstance(op, StencilOperator):
        nbr, phi = op.edges(np.arange(op.n))
        pv = torch.tensor(np.asarray(p, dtype=float).ravel(), device=dev)
        ph = torch.from_numpy(phi).to(dev)
        arg = ph[..., 0] * pv[0]
        for k in range(1, pv.numel()):
            arg = arg + ph[..., k] * pv[k]
        c = torch.exp(arg) / (op.h * op.h)
        nb = torch.from_numpy(nbr).to(dev)
        inside = nb >= 0
        B = c.sum(dim=1, keepdim=True) * X
        for e in range(nb.shape[1]):
            idx = torch.where(inside[:, e], nb[:, e], torch.zeros_like(nb[:, e]))
            B -= (c[:, e] * inside[:, e])[:, None] * X[idx]
        return B
    if isinstance(op, GaussianKernelOperator):
        pts = torch.from_numpy(op.points).to(dev)
        lam, sg = (float(p[0]), float(p[1])) if op.ridge_from_param else (op.ridge, float(p))
        D = torch.zeros((op.n, op.n), dtype=torch.float64, device=dev)
        for k in range(pts.shape[1]):
            df = pts[:, k][:, None] - pts[:, k][None, :]
            D += df * df
        K = torch.exp(-(D * (1.0 / (2.0 * sg * sg))))
        K.diagonal().add_(lam)
        return K @ X
    raise ValueError("system has no GPU operator")


def tsqr_r(A, device: int = 0):
    """R factor (w x w, upper triangular) of a tall m x w CUDA tensor (w <= 64,
    float64 or complex128) by the TSQR kernel tree of libsas (k_tsqr_block,
    sas_tsqr_r): block Householder QRs in shared memory, then the stacked R
    blocks, level by level.  R equals numpy's qr R up to the signs of its rows."""
    import torch
    A = A.contiguous()
    m, w = A.shape
    R = torch.empty((w, w), dtype=A.dtype, device=A.device)
    lib = _capi.load()
    st = torch.cuda.current_stream(A.device)
    dt = _capi.SAS_C128 if A.is_complex() else _capi.SAS_F64
    _capi.check(lib.sas_tsqr_r(_capi.ptr(A), m, w, dt, _capi.ptr(R), int(A.device.index or 0),
                               C.c_void_p(st.cuda_stream)), "sas_tsqr_r")
    return R


def solve_apsnap(system, basis, p, device: int = 0):
    """Full least squares min ||A(p) Q_X c - b(p)|| (online.py:156-165) on the
    GPU: B = A(p) X from the GPU operator, the R factor of [B | b] by libsas's
    TSQR kernels (sas_tsqr_r), the reference's 1e-12 rank test on |R_ii|
    (linalg.py:107-112), c from the triangular system R c = (Q^H b)[:r'] (the
    last column of R), and the true residual ||B c - b|| recomputed explicitly
    as the reference does.  Returns (coefficients, residual).  Not on the
    online hot path: O(n r'^2) per parameter."""
    import scipy.linalg as sla
    import torch
    dev = torch.device(f"cuda:{device}")
    X = torch.from_numpy(np.ascontiguousarray(basis.basis)).to(dev)
    B = _operator_times_basis(system, X, p, dev)
    rhs = torch.from_numpy(np.ascontiguousarray(np.asarray(system.full_rhs(p)))).to(dev)
    if rhs.is_complex() and not B.is_complex():
        B = B.to(torch.complex128)
    rhs = rhs.to(B.dtype)
    if not bool(torch.isfinite(B).all()):
        raise ValueError("matrix has non-finite entries")   # linalg._as_matrix, linalg.py:36-37
    n, r = B.shape
    if n < r:
        raise ValueError("solve_ls requires rows >= cols")
    R = tsqr_r(torch.cat([B, rhs[:, None]], dim=1), device=device).cpu().numpy()
    diag = np.abs(np.diag(R)[:r])
    if diag.size and diag.min() < 1e-12 * max(diag.max(), np.finfo(float).tiny):
        raise RankDeficiencyError(f"rank-deficient least-squares matrix at column {int(np.argmin(diag))}")
    coeff = sla.solve_triangular(R[:r, :r], R[:r, r])
    c_t = torch.from_numpy(np.ascontiguousarray(coeff)).to(dev)
    residual = float(torch.linalg.norm(B @ c_t - rhs))
    return coeff, residual


# --------------------------------------------------------------------------
# device-resident API (torch tensors; used by bench.py and the multi-GPU driver)
# --------------------------------------------------------------------------
def device_params(plan: OnlinePlan, parameters, device=None):
    import torch
    g = _gpu(plan)
    arr = g.params_array(list(parameters))
    return torch.from_numpy(arr).to(device or f"cuda:{g.device}")


def alloc_outputs(plan: OnlinePlan, P: int, device=None):
    import torch
    g = _gpu(plan)
    dev = device or f"cuda:{g.device}"
    cdt = torch.complex128 if g.complex else torch.float64
    return {
        "coef": torch.empty((P, g.r), dtype=cdt, device=dev),
        "sres": torch.empty(P, dtype=torch.float64, device=dev),
        "outv": torch.empty((P, 2), dtype=torch.float64, device=dev),
        "status": torch.empty(P, dtype=torch.int32, device=dev),
        "bad": torch.empty(P, dtype=torch.int32, device=dev),
    }


def solve_device(plan: OnlinePlan, params_t, out: dict, stream=None, coef_table=None, rhs_table=None) -> int:
    """Enqueue the batched solve on `stream` (torch stream; default: current).
    All tensors live on the plan's device.  Returns the number of kernels
    launched."""
    import torch
    g = _gpu(plan)
    st = stream if stream is not None else torch.cuda.current_stream(g.device)
    P = params_t.shape[0]
    rc = g.lib.sas_solve(g.handle, _capi.ptr(params_t), P, _capi.ptr(coef_table), _capi.ptr(rhs_table),
                         _capi.ptr(out["coef"]), _capi.ptr(out["sres"]), _capi.ptr(out["outv"]),
                         _capi.ptr(out["status"]), _capi.ptr(out["bad"]), C.c_void_p(st.cuda_stream))
    _capi.check(rc, "sas_solve")
    return g.launches()


def lift_batch(plan: OnlinePlan, coefficients) -> np.ndarray:
    """x = Q_X c for a batch of coefficient vectors (P x r' -> P x n), on the GPU."""
    import torch
    g = _gpu(plan)
    cf = np.ascontiguousarray(np.asarray(coefficients).astype(g.np_dtype))
    P = cf.shape[0]
    dev = f"cuda:{g.device}"
    ct = torch.from_numpy(cf).to(dev)
    x = torch.empty((P, g.n), dtype=ct.dtype, device=dev)
    st = torch.cuda.current_stream(g.device)
    _capi.check(g.lib.sas_lift(g.handle, _capi.ptr(ct), P, _capi.ptr(x), C.c_void_p(st.cuda_stream)), "sas_lift")
    out = x.cpu().numpy()
    return out.astype(g.result_dtype, copy=False)


def set_full_operator(plan: OnlinePlan):
    """Upload the full operator (for relative_residual).  A p-dependent
    right-hand side is passed per call instead (relative_residual)."""
    g = _gpu(plan)
    sysm = plan.system
    if g.rhs_constant:
        b = np.asarray(sysm.full_rhs(None) if hasattr(sysm, "operator") else sysm.b)
    else:
        b = np.zeros(g.n)
    b = np.ascontiguousarray(b.astype(g.np_dtype))
    keep = [b]
    op = row_operator(sysm)
    if sysm.affine_terms is not None:
        K = len(sysm.affine_terms)
        rps, cis, vas = (C.c_void_p * K)(), (C.c_void_p * K)(), (C.c_void_p * K)()
        for k, t in enumerate(sysm.affine_terms):
            m = t.matrix.tocsr()
            rp = np.ascontiguousarray(m.indptr.astype(np.int64))
            ci = np.ascontiguousarray(m.indices.astype(np.int64))
            va = np.ascontiguousarray(m.data.astype(g.np_dtype))
            keep += [rp, ci, va]
            rps[k], cis[k], vas[k] = rp.ctypes.data, ci.ctypes.data, va.ctypes.data
        rc = g.lib.sas_plan_set_operator(g.handle, rps, cis, vas, None, None, _capi.ptr(b))
    elif isinstance(op, StencilOperator):
        nbr, phi = op.edges(np.arange(op.n))
        keep += [nbr, phi]
        rc = g.lib.sas_plan_set_operator(g.handle, None, None, None, _capi.ptr(nbr), _capi.ptr(phi), _capi.ptr(b))
    else:
        rc = g.lib.sas_plan_set_operator(g.handle, None, None, None, None, None, _capi.ptr(b))
    _capi.check(rc, "sas_plan_set_operator")
    g._operator_set = True


def relative_residual(plan: OnlinePlan, parameters, coefficients, return_floor: bool = False):
    """||A(p) Q_X c - b(p)|| / max(||b(p)||, 1e-300) per parameter (cli.py:285,
    344-351), on the GPU (sas_residual).  With return_floor, also the rounding
    floor 100 eps || |A(p)| |x| || / ||b(p)||: a relative
    residual below it is rounding noise.  Opaque affine coefficients and a
    p-dependent right-hand side are evaluated on the host per parameter."""
    import torch
    g = _gpu(plan)
    if not g._operator_set:
        set_full_operator(plan)
    parameters = list(parameters)
    dev = f"cuda:{g.device}"
    pt = torch.from_numpy(g.params_array(parameters)).to(dev)
    ct = torch.from_numpy(np.ascontiguousarray(np.asarray(coefficients).astype(g.np_dtype))).to(dev)
    tab = g.coef_table(parameters)
    tab_t = None if tab is None else torch.from_numpy(tab).to(dev)
    b_t = None
    if not g.rhs_constant:
        rows = np.stack([np.asarray(plan.system.full_rhs(p)) for p in parameters]).astype(g.np_dtype)
        b_t = torch.from_numpy(np.ascontiguousarray(rows)).to(dev)
    out = torch.empty(len(parameters), dtype=torch.float64, device=dev)
    fl = torch.empty(len(parameters), dtype=torch.float64, device=dev) if return_floor else None   # NULL: not computed
    st = torch.cuda.current_stream(g.device)
    _capi.check(g.lib.sas_residual(g.handle, _capi.ptr(pt), _capi.ptr(ct), len(parameters), _capi.ptr(tab_t),
                                   _capi.ptr(b_t), _capi.ptr(out), _capi.ptr(fl), C.c_void_p(st.cuda_stream)),
                "sas_residual")
    if return_floor:
        return out.cpu().numpy(), fl.cpu().numpy()
    return out.cpu().numpy()


# --------------------------------------------------------------------------
# plan artifacts (online.py:168-195): same npz layout as the reference
# --------------------------------------------------------------------------
def save_plan(path, plan: OnlinePlan) -> None:
    payload = {"sampled_basis": plan.sampled_basis, "affine": np.array(plan.affine)}
    if plan.blocks is not None:
        for k, blk in enumerate(plan.blocks):
            payload[f"block_{k}"] = blk
    if plan.output_projection is not None:
        payload["output_projection"] = plan.output_projection
    np.savez_compressed(path, **payload)


def load_plan(path, system, basis, selector, device: int = 0) -> OnlinePlan:
    data = np.load(path)
    blocks = None
    if bool(data["affine"]):
        blocks = []
        k = 0
        while f"block_{k}" in data:
            blocks.append(data[f"block_{k}"])
            k += 1
        blocks = tuple(blocks)
    proj = data["output_projection"] if "output_projection" in data else None
    gpu = GpuPlan(system, basis, selector, blocks, proj, device=device)
    return OnlinePlan(system=system, basis=basis, selector=selector, blocks=blocks,
                      sampled_basis=data["sampled_basis"], output_projection=proj, gpu=gpu)
