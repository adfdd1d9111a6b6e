"""Throughput and full-size parity spot checks for all five BASELINE configs on one GPU.

    python tools/bench_configs.py [--configs 1,2,3,4,5] [--steps 5] [--out gpurun_out/configs.jsonl]

For each config: build the problem at its BASELINE size, obtain X and S
(offline: host sparse solves for config 1, GPU Cholesky for config 2, GPU CG
for configs 3 and 5, GPU BiCGSTAB for config 4; --synthetic uses a seeded
orthonormal basis for every config but 2 -- the online cost does not depend
on the values of X), then time the device-resident online sweep of the
config's per-GPU parameter count and compare a few parameters against the CPU
oracle at full size.  One JSON line per config.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

import torch  # noqa: E402

from oracle import online_ref  # noqa: E402
from paper_2510_04825_b200 import _capi, online, problems  # noqa: E402
from paper_2510_04825_b200.offline import (RowSelector, SnapshotBasis, anchor_product, choose_anchor,  # noqa: E402
                                           offline, select_rows)
from paper_2510_04825_b200.systems import GaussianKernelOperator, StencilOperator  # noqa: E402

P_PER_GPU = {1: 1000, 2: 4096, 3: 65_536, 4: 100_000, 5: 125_000}


def synthetic_basis(prob, r, complex_=False, seed=7, device=None):
    g = torch.Generator(device="cpu").manual_seed(seed)
    n = prob.system.n
    a = torch.randn(n, r, generator=g, dtype=torch.float64)
    if complex_:
        a = torch.complex(a, torch.randn(n, r, generator=g, dtype=torch.float64))
    if device is not None:
        a = a.to(device)
    q, _ = torch.linalg.qr(a)
    X = q.cpu().numpy()
    basis = SnapshotBasis(points=tuple(prob.snapshot_points[:r]), raw=X, basis=X, singular_values=np.ones(r))
    anchor = choose_anchor(prob.snapshot_points)
    b_anchor = anchor_product(prob.system, anchor, X)
    sel = select_rows(b_anchor, prob.system.full_rhs(anchor), strategy="leverage",
                      oversample=prob.samples / (r + 1), seed=prob.selector_seed)
    return basis, sel


def oracle_coef(prob, basis, sel, p):
    sysm = prob.system
    X, idx = basis.basis, sel.indices
    if sysm.affine_terms is not None:
        blocks = online_ref.affine_blocks([t.matrix for t in sysm.affine_terms], X, idx)
        coeffs = [complex(t.scale) if t.kind == "const" else complex(t.scale) * p for t in sysm.affine_terms]
        m = online_ref.affine_combine(coeffs, blocks)
        t = sysm.rhs(p, idx)
        c, sres, _ = online_ref.solve_one(m, t, sel.weights)
        return c, sres, online_ref.ls_floor(m, t, sel.weights, draws=2)
    op = sysm.operator
    if isinstance(op, GaussianKernelOperator):
        fn = lambda q, rows: online_ref.gauss_rows(op.points, rows, float(q), op.ridge)
    else:
        fn = lambda q, rows: online_ref.stencil_rows(op, q, rows)
    m = online_ref.sampled_rows(fn, X, idx, p)
    t = sysm.rhs(p, idx)
    c, sres, _ = online_ref.solve_one(m, t, sel.weights)
    uniq, inverse = np.unique(idx, return_inverse=True)
    floor = online_ref.ls_floor(m, t, sel.weights, draws=2, rows=fn(p, uniq), basis=X, inverse=inverse)
    return c, sres, floor


DMMA_PEAK_TF, DFMA_PEAK_TF = 37.0, 34.1  # measured on this pool (profiles/r01_fp64_peaks.jsonl)


def algorithmic_flops(prob, r, s, complex_):
    """Per parameter value: assembly of S A(p) X, and the
    least squares (Householder QR 2sr^2 - 2/3 r^3, Q^T t 4sr - 2r^2, back
    solve r^2, explicit residual 2sr); complex counts x4."""
    sysm = prob.system
    op = getattr(sysm, "operator", None)
    ls = 2 * s * r * r - 2 * r ** 3 / 3 + 4 * s * r - 2 * r * r + r * r + 2 * s * r
    if sysm.affine_terms is not None:
        asm = 2 * len(sysm.affine_terms) * s * r
    elif isinstance(op, GaussianKernelOperator):
        asm = 2 * s * sysm.n * r
    else:
        E, dp = op.n_edges, op.n_params
        asm = 2 * E * s * dp + 2 * (E + 1) * s * r
    mul = 4 if complex_ else 1
    return mul * asm, mul * ls


def run(cfg, steps, dev, synthetic=False, P=None, check=True, resid_count=0):
    t0 = time.perf_counter()
    prob = problems.build(cfg)
    if synthetic and cfg != 2:
        r = {1: 8, 3: 40, 4: 30, 5: 50}[cfg]   # the real bases: r' = 8, 40, 30, 50
        basis, sel = synthetic_basis(prob, r, complex_=(cfg == 4), device=dev)
        src = f"synthetic orthonormal basis r={r}"
    elif cfg in (1, 2):
        basis, sel = offline(prob, device=dev)
        src = "offline (reference recipe)"
    elif cfg in (3, 5):
        basis, sel = offline(prob, device=dev, prefer_cg=True)
        src = "offline (GPU CG snapshots)"
    elif cfg == 4:
        basis, sel = offline(prob, device=dev)
        src = "offline (GPU BiCGSTAB snapshots, pod(1e-13))"

    t_off = time.perf_counter() - t0
    plan = online.precompute_online(prob.system, basis, sel, device=0)
    P = P or P_PER_GPU[cfg]
    params = prob.test_params(P)
    pt = online.device_params(plan, params, device=dev)
    out = online.alloc_outputs(plan, P, device=dev)
    online.solve_device(plan, pt, out)
    torch.cuda.synchronize()
    g = plan.gpu
    g.set_timing(True)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    stage = {}
    total = 0.0
    for _ in range(steps):
        ev0.record()
        online.solve_device(plan, pt, out)
        ev1.record()
        torch.cuda.synchronize()
        total += ev0.elapsed_time(ev1)
        for sid, ms in g.stage_times():
            stage.setdefault(sid, []).append(ms)
    g.set_timing(False)
    ms = total / steps
    st = out["status"].cpu().numpy()
    coef = out["coef"].cpu().numpy()
    # full-size parity spot check against the oracle
    worst = 0.0
    checks = []
    for k in (np.linspace(0, P - 1, 4).astype(int) if check else []):
        c, sres, floor = oracle_coef(prob, basis, sel, params[k])
        d = float(np.linalg.norm(coef[k] - c) / np.linalg.norm(c))
        checks.append({"k": int(k), "rel_diff": d, "floor": float(floor)})
        worst = max(worst, d / max(1e-10, 10 * floor))
    resid = None
    if resid_count:
        sub = params[:resid_count]
        online.set_full_operator(plan)
        online.relative_residual(plan, sub[:2], coef[:2])  # warm-up
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rr = online.relative_residual(plan, sub, coef[:resid_count])
        torch.cuda.synchronize()
        t_rr = time.perf_counter() - t1
        resid = {"count": resid_count, "seconds": round(t_rr, 4), "median_relres": float(np.median(rr))}
        if prob.system.n <= 2_000_000:
            x = basis.basis @ coef[0]
            op = getattr(prob.system, "operator", None)
            if isinstance(op, GaussianKernelOperator):
                a = online_ref.gauss_rows(op.points, np.arange(op.n), float(params[0]), op.ridge)
            else:
                a = prob.system.matrix(params[0])
            b = prob.system.full_rhs(params[0])
            ref = online_ref.relative_residual(a, x, b)
            resid["relres0_gpu"] = float(rr[0])
            resid["relres0_oracle"] = ref
    f_asm, f_ls = algorithmic_flops(prob, basis.rank, sel.size, g.complex)
    st_ms = {("K3" if k == _capi.SAS_STAGE_GAUSS_ROWS else "K4"): sum(v) / steps for k, v in stage.items()}
    roof = {"gflop_per_sweep": round((f_asm + f_ls) * P / 1e9, 3), "tflops_sweep": round((f_asm + f_ls) * P / ms / 1e9, 3)}
    if "K3" in st_ms:  # contraction on DMMA, least squares (K4) on DFMA
        roof["K3_tflops"] = round(f_asm * P / st_ms["K3"] / 1e9, 3)
        roof["K3_frac_dmma_peak"] = round(roof["K3_tflops"] / DMMA_PEAK_TF, 4)
        roof["K4_tflops"] = round(f_ls * P / st_ms["K4"] / 1e9, 3)
        roof["K4_frac_dfma_peak"] = round(roof["K4_tflops"] / DFMA_PEAK_TF, 4)
    else:  # assembly fused into K4
        roof["K4_tflops"] = round((f_asm + f_ls) * P / st_ms["K4"] / 1e9, 3)
        roof["K4_frac_dfma_peak"] = round(roof["K4_tflops"] / DFMA_PEAK_TF, 4)
    return {
        "resid": resid, "roofline": roof,
        "config": cfg, "name": prob.key, "n": prob.system.n, "r": basis.rank, "s": sel.size, "P": P,
        "dtype": "c128" if g.complex else "f64", "basis": src, "offline_s": round(t_off, 1),
        "ms_per_sweep": round(ms, 3), "p_per_s": round(P / ms * 1e3, 1),
        "stage_ms": {("K3" if k == _capi.SAS_STAGE_GAUSS_ROWS else "K4"): round(sum(v) / steps, 3)
                     for k, v in stage.items()},
        "status_ok": bool(np.all(st == 0)), "parity": checks, "parity_ok": bool(worst <= 1.0),
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default=None)
    ap.add_argument("--synthetic", action="store_true", help="seeded orthonormal basis for every config but 2")
    ap.add_argument("--P", type=int, default=None)
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--resid", type=int, default=0, help="time the full-residual checker on the first N p")
    args = ap.parse_args()
    dev = torch.device("cuda:0")
    for cfg in [int(c) for c in args.configs.split(",")]:
        res = run(cfg, args.steps, dev, synthetic=args.synthetic, P=args.P, check=not args.no_parity,
                  resid_count=args.resid)
        line = json.dumps(res)
        print(line, flush=True)
        if args.out:
            with open(args.out, "a") as fh:
                fh.write(line + "\n")


if __name__ == "__main__":
    main()
