#!/usr/bin/env python
"""bench.py — SubApSnap online solves per second on B200.

Headline workload (BASELINE.json configs[1], "config 2"): Gaussian-kernel
ridge regression over the bandwidth, n = 20,000 points in d = 8, r = 20
snapshots, s = 80 leverage-sampled rows, one step = the online solve of a
batch of 4,096 bandwidths per GPU (weak scaling).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl ours|reference]

`value`  device-resident p-values/s over all ranks (params and results in
         HBM, CUDA events on the launching stream, max over ranks, L2 flushed
         between steps).
`e2e`    the same metric through the C-ABI host entry point sas_solve_host:
         pinned host params in, host results out, every step.
`roofline` the dominant kernel (K3 Gaussian kernel-row contraction, DMMA) —
         algorithmic flops 2 s n r per parameter over its event-timed launch
         duration against the measured FP64 tensor (DMMA) peak.
`cpu_baseline` the CPU oracle port (oracle/online_ref.py: the reference's
         numpy online path) on a bounded sample, all host cores.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

P_PER_GPU = {1: 1000, 2: 4096, 3: 65_536, 4: 100_000, 5: 125_000}
FP64_DMMA_PEAK_TFLOPS = 37.0   # profiles/r01_fp64_peaks.jsonl: DMMA.8x8x4 microbenchmark, this pool
FP64_DFMA_PEAK_TFLOPS = 34.1   # same file, DFMA


# --------------------------------------------------------------------------
# CPU side: the oracle port (reference numpy online path), multi-process
# --------------------------------------------------------------------------
_W = {}


def _cpu_init(state):
    from threadpoolctl import threadpool_limits
    threadpool_limits(1)
    _W.update(state)


def _cpu_solve_chunk(ps):
    from oracle import online_ref
    st = _W
    out = []
    if st["kind"] == "gauss":
        fn = lambda q, rows: online_ref.gauss_rows(st["points"], rows, float(q), st["ridge"])
        for p in ps:
            m = online_ref.sampled_rows(fn, st["X"], st["S"], p)
            c, s, _ = online_ref.solve_one(m, st["t"], st["w"])
            out.append(c)
    return out


class CpuPort:
    """Multi-process pool running the oracle port of the reference online path."""

    def __init__(self, state, cores):
        import multiprocessing as mp
        self.cores = cores
        self.pool = mp.get_context("spawn").Pool(cores, initializer=_cpu_init, initargs=(state,))

    def run(self, params):
        chunks = [list(params[i::self.cores]) for i in range(self.cores)]
        chunks = [c for c in chunks if c]
        t0 = time.perf_counter()
        self.pool.map(_cpu_solve_chunk, chunks)
        return time.perf_counter() - t0

    def close(self):
        self.pool.close()
        self.pool.join()


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_state(plan_inputs):
    X, S, w, t, pts, ridge = plan_inputs
    return {"kind": "gauss", "X": X, "S": S, "w": w, "t": t, "points": pts, "ridge": ridge}


def cpu_rate(port: CpuPort, params, target_s: float):
    """p/s of the port on a sample sized to ~target_s seconds."""
    probe = list(params[: port.cores * 2])
    dt = port.run(probe)
    per = dt / len(probe)
    count = int(min(len(params), max(port.cores * 2, target_s / max(per, 1e-9))))
    sample = list(params[:count])
    dt = port.run(sample)
    return len(sample) / dt, count, dt


# --------------------------------------------------------------------------
# GPU helpers
# --------------------------------------------------------------------------
class ClockSampler:
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.12)
        self.proc.terminate()
        out, _ = self.proc.communicate(timeout=10)
        sm, smax, reasons = [], [], set()
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                smax.append(float(parts[1]))
            except ValueError:
                continue
            for name, val in zip(self.NAMES, parts[3:7]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def ncu_traffic(kernel: str):
    """dram bytes per launch of `kernel` from the committed ncu summary, or None."""
    path = ROOT / "profiles" / "ncu_traffic.json"
    try:
        return json.loads(path.read_text()).get(kernel, {}).get("dram_bytes_per_launch")
    except Exception:
        return None


def build_inputs(cfg: int, env, device):
    """Offline phase on rank 0 (untimed), broadcast of X/S/weights to all ranks."""
    from paper_2510_04825_b200 import problems
    from paper_2510_04825_b200.offline import RowSelector, SnapshotBasis, offline
    prob = problems.build(cfg)
    arrays = None
    t0 = time.perf_counter()
    if env.rank == 0:
        basis, sel = offline(prob, device=device)
        arrays = {"X": basis.basis, "S": sel.indices, "w": sel.weights,
                  "sv": basis.singular_values}
    if env.world > 1:
        from paper_2510_04825_b200 import parallel
        arrays = parallel.broadcast_inputs(arrays if env.rank == 0 else {}, src=0, local_rank=env.local_rank)
    t_off = time.perf_counter() - t0
    basis = SnapshotBasis(points=tuple(prob.snapshot_points), raw=arrays["X"], basis=arrays["X"],
                          singular_values=arrays["sv"])
    sel = RowSelector(indices=arrays["S"], n=prob.system.n, weights=arrays["w"])
    return prob, basis, sel, t_off


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--P", type=int, default=None, help="parameter values per GPU per step")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    args = ap.parse_args()
    if args.config != 2:
        raise SystemExit("bench.py measures the headline workload (config 2); other configs are parity cases")

    from paper_2510_04825_b200 import parallel
    env = parallel.dist_env()
    import torch
    # SAS_BENCH_SHARED_GPU=1: test hook for the N>1 code path on a single-GPU box
    # (all ranks on cuda:0, host collectives over gloo; ranks never wait on each
    # other inside a kernel).  Production runs use one GPU per rank and NCCL.
    shared = os.environ.get("SAS_BENCH_SHARED_GPU") == "1"
    gpu = 0 if shared else env.local_rank
    if env.world > 1:
        import torch.distributed as dist
        torch.cuda.set_device(gpu)
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{gpu}"))
    P = args.P or P_PER_GPU[args.config]
    K, W = args.steps, args.warmup

    if args.impl == "reference":
        return run_reference_arm(args, env, P)

    dev = torch.device(f"cuda:{gpu}")
    torch.cuda.set_device(dev)
    from paper_2510_04825_b200 import online
    prob, basis, sel, t_off = build_inputs(args.config, env, dev)
    sysm = prob.system
    op = sysm.operator
    n, r, s = sysm.n, basis.rank, sel.size
    all_params = prob.test_params(P * env.world)
    my_params = parallel.shard(all_params, env.world, env.rank)
    Pl = len(my_params)

    t0 = time.perf_counter()
    plan = online.precompute_online(sysm, basis, sel, device=gpu)
    t_plan = time.perf_counter() - t0
    g = plan.gpu
    params_t = online.device_params(plan, my_params, device=dev)
    out = online.alloc_outputs(plan, Pl, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # 256 MiB > 126 MB L2
    stream = torch.cuda.current_stream(dev)

    for _ in range(W):
        online.solve_device(plan, params_t, out, stream)
    torch.cuda.synchronize(dev)
    assert int((out["status"] != 0).sum().item()) == 0, "solver reported failures"

    # ---- timed: device-resident --------------------------------------------
    g.set_timing(True)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(K)]
    stage_ms = {}
    launches = 0
    clocks = ClockSampler(torch.cuda.current_device())
    clocks.start()
    parallel.barrier(env.local_rank)
    torch.cuda.synchronize(dev)
    for k in range(K):
        flush.fill_(k & 0xFF)
        ev[k][0].record(stream)
        launches += online.solve_device(plan, params_t, out, stream)
        ev[k][1].record(stream)
        for sid, ms in g.stage_times():
            stage_ms.setdefault(sid, []).append(ms)
    torch.cuda.synchronize(dev)
    parallel.barrier(env.local_rank)
    clk = clocks.stop()
    g.set_timing(False)
    local_ms = sum(a.elapsed_time(b) for a, b in ev)
    total_ms = parallel.max_over_ranks(local_ms, env.local_rank)
    ms_per_step = total_ms / K
    value = P * env.world * K / (total_ms / 1e3)

    # ---- timed: end to end through the C-ABI host entry point ---------------
    import ctypes as C
    from paper_2510_04825_b200 import _capi
    pa = g.params_array(my_params)
    h_params = torch.from_numpy(pa).pin_memory()
    h_coef = torch.empty((Pl, r), dtype=torch.float64).pin_memory()
    h_sres = torch.empty(Pl, dtype=torch.float64).pin_memory()
    h_outv = torch.empty((Pl, 2), dtype=torch.float64).pin_memory()
    h_status = torch.empty(Pl, dtype=torch.int32).pin_memory()

    if env.world == 1:
        def e2e_step():
            rc = g.lib.sas_solve_host(g.handle, _capi.ptr(h_params), Pl, None, None, _capi.ptr(h_coef),
                                      _capi.ptr(h_sres), _capi.ptr(h_outv), _capi.ptr(h_status), None)
            _capi.check(rc, "sas_solve_host")
        gather_rows = Pl
    else:
        # N > 1: each rank copies its shard's parameters in, solves, the result rows
        # are gathered in input order over NCCL and rank 0 reads the full sweep back
        d_params = torch.empty_like(params_t)
        n_all = Pl * env.world
        gathered = torch.empty((n_all, r), dtype=out["coef"].dtype, device=dev)
        st_all = torch.empty(n_all, dtype=torch.int32, device=dev)
        h_all = torch.empty((n_all, r), dtype=torch.float64).pin_memory()
        h_st_all = torch.empty(n_all, dtype=torch.int32).pin_memory()

        def e2e_step():
            d_params.copy_(h_params, non_blocking=True)
            online.solve_device(plan, d_params, out, stream)
            parallel.all_gather_device(gathered, out["coef"])
            parallel.all_gather_device(st_all, out["status"])
            if env.rank == 0:
                h_all.copy_(gathered, non_blocking=True)
                h_st_all.copy_(st_all, non_blocking=True)
            torch.cuda.synchronize(dev)
            h_status.copy_(h_st_all[:Pl] if env.rank == 0 else out["status"])
        gather_rows = n_all

    for _ in range(W):
        e2e_step()
    parallel.barrier(env.local_rank)
    torch.cuda.synchronize(dev)
    e2e_s = 0.0
    for k in range(K):
        flush.fill_(k & 0xFF)
        torch.cuda.synchronize(dev)
        t1 = time.perf_counter()
        e2e_step()
        e2e_s += time.perf_counter() - t1
    e2e_s = parallel.max_over_ranks(e2e_s, env.local_rank)
    e2e_val = P * env.world * K / e2e_s
    assert int(h_status.sum().item()) == 0
    h2d = pa.nbytes
    if env.world == 1:
        d2h = h_coef.numel() * 8 + h_sres.numel() * 8 + h_outv.numel() * 8 + h_status.numel() * 4
    else:  # rank 0 reads back the gathered coefficients and status of the whole sweep
        d2h = gather_rows * r * 8 + gather_rows * 4

    # ---- roofline of the dominant kernel ------------------------------------
    k3 = stage_ms.get(_capi.SAS_STAGE_GAUSS_ROWS, [])
    k4 = stage_ms.get(_capi.SAS_STAGE_LSQ, [])
    k3_avg = sum(k3) / len(k3) if k3 else float("nan")
    k4_avg = sum(k4) / len(k4) if k4 else float("nan")
    launches_per_step = launches / K
    k3_per_step = len(k3) / K
    p_per_k3 = Pl / max(k3_per_step, 1)
    flops_per_p = 2.0 * s * n * r
    achieved = flops_per_p * p_per_k3 / (k3_avg / 1e3) / 1e12
    step_dev_ms = local_ms / K
    roofline = {
        "bound": "tensor", "pipe": "FP64 DMMA.8x8x4 (shared with DFMA)",
        "kernel": "k_gauss_rows (K3; timed over its fast-exp and masked-exp launches, CUDA events on the "
                  "launching stream)", "achieved": round(achieved, 3), "peak": FP64_DMMA_PEAK_TFLOPS,
        "peak_source": "measured FP64 DMMA microbenchmark on this pool (profiles/r01_fp64_peaks.jsonl); "
                       "MEASURED_PEAKS.json has no FP64 entry",
        "unit": "TFLOP/s", "frac": round(achieved / FP64_DMMA_PEAK_TFLOPS, 4),
        "traffic": ncu_traffic("k_gauss_rows"),
        "algorithmic_flops_per_p": flops_per_p, "launch_ms": round(k3_avg, 4),
        "share_of_step": round(sum(k3) / max(local_ms, 1e-9), 4),
        "exps_per_p": s * n,
        "lsq_kernel_ms": round(k4_avg, 4), "lsq_share_of_step": round(sum(k4) / max(local_ms, 1e-9), 4),
    }

    # ---- CPU baseline (rank 0, N=1 only) ------------------------------------
    cpu = None
    if env.rank == 0 and env.world == 1 and not args.no_cpu_baseline:
        cores = host_cores()
        port = CpuPort(cpu_state((np.asarray(basis.basis), np.asarray(sel.indices), sel.weights,
                                  sysm.rhs(None, sel.indices), op.points, op.ridge)), cores)
        try:
            rate, count, dt = cpu_rate(port, my_params, args.cpu_seconds)
        finally:
            port.close()
        cpu = {"value": round(rate, 3), "unit": "p-values/s", "cores": cores, "kind": "port",
               "sample": f"first {count} of the {Pl} config-2 bandwidths, oracle/online_ref.py (reference "
                         f"numpy online path: dense kernel rows + GEMM + Householder LS), {cores} worker "
                         f"processes x 1 BLAS thread, {dt:.1f} s"}

    if env.rank == 0:
        line = {
            "metric": "SubApSnap online solves/sec (p-values/s)",
            "value": round(value, 1), "unit": "p-values/s", "n_gpus": env.world, "steps": K, "warmup": W,
            "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded, BASELINE config 2 definition)",
            "config": {"workload": f"config 2 gauss_krr: n={n} d={op.points.shape[1]} r={r} s={s} "
                                   f"P={P}/GPU bandwidths", "l2": "flushed between steps (256 MiB write)",
                       "offline_s": round(t_off, 2), "plan_s": round(t_plan, 3),
                       "parallelism": f"p-sharded x{env.world}"},
            "e2e": {"value": round(e2e_val, 1), "unit": "p-values/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "api": ("sas_solve_host (C ABI, pinned host buffers)" if env.world == 1 else
                            "pinned H2D of each shard, sas_solve, NCCL all-gather of the rows, D2H on rank 0")},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if env.world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference_arm(args, env, P):
    """--impl reference: the reference's CPU online path (oracle port), all host cores."""
    import torch
    if env.rank != 0:
        if env.world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    dev = torch.device("cuda:0") if torch.cuda.is_available() else None
    from paper_2510_04825_b200 import problems
    from paper_2510_04825_b200.offline import offline
    prob = problems.build(args.config)
    basis, sel = offline(prob, device=dev)   # inputs only (untimed), shared recipe with our arm
    sysm = prob.system
    op = sysm.operator
    params = prob.test_params(P)
    cores = host_cores()
    port = CpuPort(cpu_state((np.asarray(basis.basis), np.asarray(sel.indices), sel.weights,
                              sysm.rhs(None, sel.indices), op.points, op.ridge)), cores)
    try:
        probe = list(params[: cores * 2])
        per = port.run(probe) / len(probe)
        count = int(min(len(params), max(cores, 6.0 / max(per, 1e-9))))
        sample = list(params[:count])
        for _ in range(args.warmup):
            port.run(sample[:cores])
        total = 0.0
        for _ in range(args.steps):
            total += port.run(sample)
    finally:
        port.close()
    value = count * args.steps / total
    line = {
        "metric": "SubApSnap online solves/sec (p-values/s)", "impl": "reference",
        "value": round(value, 3), "unit": "p-values/s", "n_gpus": env.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, BASELINE config 2 definition)",
        "config": {"workload": f"config 2 gauss_krr: n={sysm.n} d={op.points.shape[1]} r={basis.rank} "
                               f"s={sel.size}; each step = {count} of the {P} bandwidths",
                   "parallelism": f"{cores} CPU worker processes"},
        "cpu_baseline": {"value": round(value, 3), "unit": "p-values/s", "cores": cores, "kind": "port",
                         "sample": f"{count} bandwidths per step: oracle/online_ref.py (the reference's numpy "
                                   f"online path restated; the reference itself is Python and cannot be "
                                   f"compiled into oracle/_ref)"},
        "e2e": {"value": round(value, 3), "unit": "p-values/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if env.world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
