#!/usr/bin/env python
"""bench.py — SubApSnap online solves per second on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--scaling strong|weak]
                    [--impl ours|reference]

Workloads: the five BASELINE.json configs (problems.build(C)); the default is
config 2 (configs[1], the headline): Gaussian-kernel ridge regression over
the bandwidth, n = 20,000 points in d = 8, r = 20 snapshots, s = 80
leverage-sampled rows, 4,096 test bandwidths.  One step = the online solve of
the config's whole parameter sweep (`--scaling strong`, the default: the
sweep is the config's fixed total, 4,096 bandwidths for config 2 or 10^6
parameter values for config 5, sharded contiguously over the N ranks), or of
the config's per-GPU count on every rank (`--scaling weak`).

`--gpus N` without a torchrun environment re-launches this script under
torch.distributed.run with N ranks (127.0.0.1); one process per GPU, NCCL.
SAS_BENCH_SHARED_GPU=1 puts every rank on cuda:0 with gloo host collectives
(the N > 1 code path on a one-GPU box; ranks never wait on each other inside
a kernel).

`value`   device-resident p-values/s over all ranks (params and results in
          HBM, CUDA events on the launching stream, max over ranks, L2 flushed
          between steps).
`e2e`     the same metric through the C-ABI host entry point sas_solve_host
          (N = 1: pinned host params in, host results out, every step) or, for
          N > 1, pinned H2D of each shard + sas_solve + NCCL all-gather + D2H on
          rank 0.
`roofline` the dominant stage (largest share of the step): K3 (Gaussian
          kernel-row contraction, FP64 DMMA) or K4 (batched least squares with
          the fused row assembly, FP64 DFMA), algorithmic flops per SURVEY.md
          §8(d) over its event-timed launch duration, against the measured FP64
          peaks (profiles/r01_fp64_peaks.jsonl).
`cpu_baseline` (rank 0, N = 1) the reference's own online.solve_batch
          (baseline/_ref install of /root/reference, timed with perf_counter as
          cli.py:338-343 does) on a bounded sample of the same sweep: workers=1
          with default BLAS threads and workers=cores with 1 BLAS thread; the
          better one is the value.  Falls back to the oracle port
          (oracle/online_ref.py) when the reference is not importable.
"""
from __future__ import annotations

import argparse
import json
import os
import socket
import statistics
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

# the config's parameter sweep (BASELINE.json configs): the strong-scaling total
P_TOTAL = {1: 1000, 2: 4096, 3: 65_536, 4: 100_000, 5: 1_000_000}
# per-GPU count for --scaling weak (config 5: 10^6 over 8 GPUs)
P_PER_GPU = {1: 1000, 2: 4096, 3: 65_536, 4: 100_000, 5: 125_000}
FP64_DMMA_PEAK_TFLOPS = 37.0   # profiles/r01_fp64_peaks.jsonl: DMMA.8x8x4 microbenchmark, this pool
FP64_DFMA_PEAK_TFLOPS = 34.1   # same file, DFMA
PEAK_SOURCE = ("measured FP64 microbenchmarks on this pool (profiles/r01_fp64_peaks.jsonl: DMMA.8x8x4 37.0, "
               "DFMA 34.1 TF/s at 1965 MHz); MEASURED_PEAKS.json has no FP64 entry")
REF_DIR = ROOT / "baseline" / "_ref"


def _hbm_peak_gbs() -> float:
    """Measured copy bandwidth of this pool (driver-written MEASURED_PEAKS.json),
    else the profiling recipe's fallback."""
    try:
        return float(json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        return 6553.0


HBM_PEAK_GBS = _hbm_peak_gbs()


# --------------------------------------------------------------------------
# algorithmic work per parameter value
# --------------------------------------------------------------------------
def lsq_flops(s: int, r: int, cplx: bool) -> float:
    """Householder QR 2sr^2 - 2/3 r^3, Q^H t 4sr - 2r^2, back-solve r^2,
    sampled residual 2sr; complex counts x4."""
    f = 2.0 * s * r * r - 2.0 / 3.0 * r ** 3 + 4.0 * s * r - 2.0 * r * r + r * r + 2.0 * s * r
    return 4.0 * f if cplx else f


def assembly_flops(plan) -> float:
    g = plan.gpu
    s, r = g.s, g.r
    if plan.blocks is not None:  # K1: M = sum_k f_k(p) B_k
        return len(plan.blocks) * (8.0 if g.complex else 2.0) * s * r
    op = plan.system.operator
    if hasattr(op, "n_edges"):   # K2: phi dot products + the (E+1)-point contraction
        E = op.n_edges
        return 2.0 * E * s * g.dp + 2.0 * (E + 1) * s * r
    return 0.0                   # Gaussian rows: K3 (separate stage)


# --------------------------------------------------------------------------
# CPU baseline: the reference's own solve_batch (or the oracle port)
# --------------------------------------------------------------------------
def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def import_reference():
    """The reference package from baseline/_ref (installed by build()), else
    from /root/reference when present (this container only).  None if absent."""
    for p in (REF_DIR, Path("/root/reference/pkg/src")):
        if (p / "subapsnap" / "__init__.py").exists():
            if str(p) not in sys.path:
                sys.path.insert(0, str(p))
            try:
                import subapsnap.online  # noqa: F401
                import subapsnap.snapshot  # noqa: F401
                import subapsnap.subsample  # noqa: F401
                import subapsnap.systems  # noqa: F401
                import subapsnap
                return subapsnap
            except Exception:
                return None
    return None


def reference_system(ref, prob):
    """problems.Problem -> the reference's ParametricSystem.  The BASELINE
    problems do not exist in the reference: affine configs
    use the reference's const_term/linear_term, the non-affine ones the harness
    row oracles of oracle/online_ref.py as row_fn, exactly as
    tests/golden/make_golden.py wraps them."""
    from oracle import online_ref
    rs = ref.systems
    sysm = prob.system
    b = np.asarray(sysm.b)

    def rhs_fn(p, idx):
        return b[idx]

    dom = rs.Domain(axes=tuple(rs.Axis(a.lo, a.hi, a.imag) for a in sysm.domain.axes))
    if sysm.affine_terms is not None:
        terms = [rs.const_term(t.matrix, t.scale) if t.kind == "const" else rs.linear_term(t.matrix, t.scale)
                 for t in sysm.affine_terms]
        return rs.ParametricSystem(sysm.n, dom, rhs_fn, affine_terms=terms,
                                   output_functional=sysm.output_functional, name=sysm.name)
    op = sysm.operator
    if hasattr(op, "n_edges"):
        def row_fn(p, idx):
            return online_ref.stencil_rows(op, p, idx)
    else:
        def row_fn(p, idx):
            return online_ref.gauss_rows(op.points, idx, float(p), op.ridge)
    return rs.ParametricSystem(sysm.n, dom, rhs_fn, row_fn=row_fn, name=sysm.name)


class CpuReference:
    """Times the reference's online.solve_batch (cli.py:338-343 convention) on
    this host.  `dense_row_bytes` bounds concurrency for the non-affine configs
    (the reference materialises s_u x n dense rows per parameter value,
    online.py:57-65)."""

    def __init__(self, prob, X, S, w, sv):
        self.ref = import_reference()
        self.prob = prob
        self.cores = host_cores()
        self.kind = "reference" if self.ref is not None else "port"
        n = prob.system.n
        s_u = np.unique(S).size
        self.dense_row_bytes = 0 if prob.system.affine_terms is not None else s_u * n * 8
        if self.ref is not None:
            rsys = reference_system(self.ref, prob)
            basis = self.ref.snapshot.SnapshotBasis(points=tuple(prob.snapshot_points), raw=X, basis=X,
                                                    singular_values=np.asarray(sv))
            sel = self.ref.subsample.RowSelector(indices=S, n=n, weights=w)
            self.plan = self.ref.online.precompute_online(rsys, basis, sel)   # untimed (cli.py:239-265)
        else:
            self.port = (X, S, w)

    def max_workers(self) -> int:
        if not self.dense_row_bytes:
            return self.cores
        try:
            import psutil
            avail = psutil.virtual_memory().available
        except Exception:
            avail = 16 << 30
        return max(0, min(self.cores, int(avail // (3 * self.dense_row_bytes))))

    def run(self, params, workers: int) -> float:
        from threadpoolctl import threadpool_limits
        params = list(params)
        if self.ref is not None:
            if workers > 1:
                with threadpool_limits(1):
                    t0 = time.perf_counter()
                    self.ref.online.solve_batch(self.plan, params, workers=workers)
                    return time.perf_counter() - t0
            t0 = time.perf_counter()
            self.ref.online.solve_batch(self.plan, params, workers=1)
            return time.perf_counter() - t0
        return self._run_port(params, workers)

    def _run_port(self, params, workers):
        from concurrent.futures import ThreadPoolExecutor

        from threadpoolctl import threadpool_limits

        from oracle import online_ref
        X, S, w = self.port
        sysm = self.prob.system
        t = sysm.rhs(None, S)
        if sysm.affine_terms is not None:
            blocks = online_ref.affine_blocks([tm.matrix for tm in sysm.affine_terms], X, S)

            def one(p):
                fs = [complex(tm.scale) if tm.kind == "const" else complex(tm.scale) * p for tm in sysm.affine_terms]
                m = online_ref.affine_combine(fs, blocks)
                return online_ref.solve_one(m, t, w)
        else:
            op = sysm.operator
            if hasattr(op, "n_edges"):
                fn = lambda q, rows: online_ref.stencil_rows(op, q, rows)  # noqa: E731
            else:
                fn = lambda q, rows: online_ref.gauss_rows(op.points, rows, float(q), op.ridge)  # noqa: E731

            def one(p):
                return online_ref.solve_one(online_ref.sampled_rows(fn, X, S, p), t, w)
        t0 = time.perf_counter()
        if workers > 1:
            with threadpool_limits(1), ThreadPoolExecutor(workers) as pool:
                list(pool.map(one, params))
        else:
            for p in params:
                one(p)
        return time.perf_counter() - t0

    def rate(self, params, workers: int, budget_s: float, max_count: int):
        """p/s on a sample sized to ~budget_s (after a 2-parameter probe)."""
        probe_n = max(1, min(max(2, workers), len(params), max_count))
        per = self.run(params[:probe_n], workers) / probe_n
        count = int(min(len(params), max_count, max(probe_n, budget_s / max(per, 1e-9))))
        dt = self.run(params[:count], workers)
        return count / dt, count, dt

    def baseline(self, params, budget_s: float):
        """Both protocols of SURVEY.md §8(d): workers=1 (default BLAS threads)
        and workers=cores (1 BLAS thread each); returns the cpu_baseline dict."""
        cap = 4 if self.dense_row_bytes > (4 << 30) else len(params)
        r1, c1, t1 = self.rate(params, 1, budget_s / 2, cap)
        wmax = self.max_workers()
        rw = cw = tw = None
        if wmax > 1:
            rw, cw, tw = self.rate(params, wmax, budget_s / 2, cap * wmax if cap < len(params) else len(params))
        best = max(r1, rw or 0.0)
        what = ("the reference's online.solve_batch (baseline/_ref install of /root/reference; harness row "
                "oracles for the non-affine BASELINE problems)" if self.kind == "reference"
                else "oracle/online_ref.py (the reference's numpy online path restated; reference not importable)")
        # workers=1 runs with the default BLAS thread count (all host cores)
        return {"value": round(best, 3), "unit": "p-values/s", "cores": self.cores,
                "kind": self.kind, "host_cores": self.cores, "cpu_model": cpu_model(),
                "workers1": {"value": round(r1, 3), "count": c1, "seconds": round(t1, 2),
                             "blas_threads": "default"},
                "workers_cores": None if rw is None else {"value": round(rw, 3), "workers": wmax, "count": cw,
                                                          "seconds": round(tw, 2), "blas_threads": 1},
                "sample": f"{what}: the first {max(c1, cw or 0)} parameter values of the sweep, perf_counter "
                          f"around solve_batch (cli.py:338-343)"}


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

    def stop(self, busy=None):
        """Stop sampling.  A timed region shorter than nvidia-smi's first
        samples (config 1: 20 steps in < 1 ms) is extended by `busy()` -- more
        steps of the same work -- until two samples have been taken under load."""
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        if busy is not None:
            t_end = time.perf_counter() + 0.6
            while time.perf_counter() < t_end:
                busy()
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
    """Offline phase on rank 0 (untimed), NCCL broadcast of X/S/weights to all
    ranks (X stays on the device)."""
    from paper_2510_04825_b200 import problems
    from paper_2510_04825_b200.offline import RowSelector, SnapshotBasis, offline
    prob = problems.build(cfg)
    arrays = None
    t0 = time.perf_counter()
    if env.rank == 0:
        basis, sel = offline(prob, device=device)
        arrays = {"X": basis.basis, "S": sel.indices, "w": sel.weights, "sv": basis.singular_values}
    if env.world > 1:
        from paper_2510_04825_b200 import parallel
        arrays = parallel.broadcast_inputs(arrays if env.rank == 0 else {}, src=0, local_rank=env.local_rank,
                                           device_keys=("X",))
    t_off = time.perf_counter() - t0
    basis = SnapshotBasis(points=tuple(prob.snapshot_points), raw=arrays["X"], basis=arrays["X"],
                          singular_values=arrays["sv"])
    sel = RowSelector(indices=arrays["S"], n=prob.system.n, weights=arrays["w"])
    return prob, basis, sel, t_off


def free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def relaunch(n: int) -> int:
    """--gpus N outside torchrun: run this script under torch.distributed.run."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(free_port()), str(Path(__file__).resolve()),
           *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=2, choices=[1, 2, 3, 4, 5])
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"])
    ap.add_argument("--P", type=int, default=None, help="override: parameter values per step (strong) or per GPU (weak)")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=16.0)
    args = ap.parse_args()

    from paper_2510_04825_b200 import parallel
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        raise SystemExit(relaunch(args.gpus))
    env = parallel.dist_env()
    if args.impl == "reference":
        return run_reference_arm(args, env)

    import torch
    shared = os.environ.get("SAS_BENCH_SHARED_GPU") == "1"
    gpu = 0 if shared else env.local_rank
    torch.cuda.set_device(gpu)
    if env.world > 1:
        import torch.distributed as dist
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device(f"cuda:{gpu}"))
    K, W = args.steps, args.warmup
    cfg = args.config
    if args.scaling == "strong":
        P_all = args.P or P_TOTAL[cfg]
    else:
        P_all = (args.P or P_PER_GPU[cfg]) * env.world

    dev = torch.device(f"cuda:{gpu}")
    from paper_2510_04825_b200 import _capi, online
    prob, basis, sel, t_off = build_inputs(cfg, env, dev)
    sysm = prob.system
    n, r, s = sysm.n, basis.rank, sel.size
    all_params = prob.test_params(P_all)
    my_params = parallel.shard(all_params, env.world, env.rank)
    Pl = len(my_params)

    t0 = time.perf_counter()
    plan = online.precompute_online(sysm, basis, sel, device=gpu)
    torch.cuda.synchronize(dev)
    t_plan = time.perf_counter() - t0
    g = plan.gpu
    params_t = online.device_params(plan, my_params, device=dev)
    out = online.alloc_outputs(plan, Pl, device=dev)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)   # 256 MiB > 126 MB L2
    # a dedicated (non-default) stream: the solve's CUDA graph is captured and
    # replayed on it directly; events, the L2 flush and copies go to it too
    stream = torch.cuda.Stream(device=dev)
    torch.cuda.set_stream(stream)

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
    g.set_timing(False)

    def busy():  # the same solve, untimed, to keep the GPU loaded while nvidia-smi samples
        for _ in range(8):
            online.solve_device(plan, params_t, out, stream)
        torch.cuda.synchronize(dev)
    local_ms = sum(a.elapsed_time(b) for a, b in ev)
    clk = clocks.stop(busy if local_ms < 1000.0 else None)
    total_ms = parallel.max_over_ranks(local_ms, env.local_rank)
    ms_per_step = total_ms / K
    value = P_all * K / (total_ms / 1e3)

    # ---- timed: end to end through the C-ABI host entry point ---------------
    pa = g.params_array(my_params)
    h_params = torch.from_numpy(pa).pin_memory()
    cdt = torch.complex128 if g.complex else torch.float64
    h_coef = torch.empty((Pl, r), dtype=cdt).pin_memory()
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
        lo_hi = [parallel.shard_bounds(P_all, env.world, q) for q in range(env.world)]
        maxrows = max(hi - lo for lo, hi in lo_hi)
        d_params = torch.empty_like(params_t)
        pad_coef = torch.zeros((maxrows, r), dtype=cdt, device=dev)
        pad_st = torch.zeros(maxrows, dtype=torch.int32, device=dev)
        gathered = torch.empty((maxrows * env.world, r), dtype=cdt, device=dev)
        st_all = torch.empty(maxrows * env.world, dtype=torch.int32, device=dev)
        h_all = torch.empty((maxrows * env.world, r), dtype=cdt).pin_memory()
        h_st_all = torch.empty(maxrows * env.world, dtype=torch.int32).pin_memory()

        def e2e_step():
            d_params.copy_(h_params, non_blocking=True)
            online.solve_device(plan, d_params, out, stream)
            pad_coef[:Pl].copy_(out["coef"])
            pad_st[:Pl].copy_(out["status"])
            parallel.all_gather_device(gathered, pad_coef)
            parallel.all_gather_device(st_all, pad_st)
            if env.rank == 0:
                h_all.copy_(gathered, non_blocking=True)
                h_st_all.copy_(st_all, non_blocking=True)
            torch.cuda.synchronize(dev)
            h_status.copy_(h_st_all[:Pl] if env.rank == 0 else out["status"])
        gather_rows = maxrows * env.world

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
    e2e_val = P_all * K / e2e_s
    assert int(h_status.sum().item()) == 0
    h2d = pa.nbytes
    esz = 16 if g.complex else 8
    if env.world == 1:
        d2h = h_coef.numel() * esz + h_sres.numel() * 8 + h_outv.numel() * 8 + h_status.numel() * 4
    else:  # rank 0 reads back the gathered coefficients and status of the whole sweep
        d2h = gather_rows * r * esz + gather_rows * 4

    # ---- roofline of the dominant stage -------------------------------------
    def stage(sid):
        v = stage_ms.get(sid, [])
        return (sum(v) / len(v) if v else 0.0), len(v) / K, sum(v)
    k3_ms, k3_per_step, k3_sum = stage(_capi.SAS_STAGE_GAUSS_ROWS)
    k4_ms, k4_per_step, k4_sum = stage(_capi.SAS_STAGE_LSQ)
    k2_ms, k2_per_step, k2_sum = stage(_capi.SAS_STAGE_STENCIL_ROWS)
    asm = assembly_flops(plan)
    # the compact-WY path assembles the stencil rows in its own launches (K2); every
    # other path fuses the assembly into K4
    k4_flops_p = lsq_flops(s, r, g.complex) + (0.0 if k2_per_step else asm)
    stages = {"K4_lsq": {"ms_per_launch": round(k4_ms, 4), "launches_per_step": k4_per_step,
                         "share_of_step": round(k4_sum / max(local_ms, 1e-9), 4),
                         "flops_per_p": k4_flops_p,
                         "tflops": round(k4_flops_p * Pl / max(k4_per_step, 1) / (k4_ms / 1e3) / 1e12, 3)
                         if k4_ms else None}}
    stages["K4_lsq"]["frac_dfma_peak"] = (round(stages["K4_lsq"]["tflops"] / FP64_DFMA_PEAK_TFLOPS, 4)
                                          if stages["K4_lsq"]["tflops"] else None)
    if k2_per_step:
        ld = (s + 7) // 8 * 8
        while ld % 16 != 8:
            ld += 8
        blk_bytes = ld * ((r + 1 + 7) // 8 * 8) * 8   # [M | t] block written per parameter value (HBM)
        k2_gbs = blk_bytes * Pl / k2_per_step / (k2_ms / 1e3) / 1e9
        stages["K2_stencil_rows"] = {"ms_per_launch": round(k2_ms, 4), "launches_per_step": k2_per_step,
                                     "share_of_step": round(k2_sum / max(local_ms, 1e-9), 4),
                                     "flops_per_p": asm, "bytes_written_per_p": blk_bytes,
                                     "write_gbs": round(k2_gbs, 1),
                                     "frac_hbm_peak": round(k2_gbs / HBM_PEAK_GBS, 4)}
        both = (k2_sum + k4_sum) / K
        stages["K4_lsq"]["tflops_with_assembly"] = round((asm + k4_flops_p) * Pl / (both / 1e3) / 1e12, 3)
        stages["K4_lsq"]["frac_dfma_peak_with_assembly"] = round(
            stages["K4_lsq"]["tflops_with_assembly"] / FP64_DFMA_PEAK_TFLOPS, 4)
    if k3_per_step:
        k3_flops_p = 2.0 * s * n * r
        k3_tf = k3_flops_p * Pl / k3_per_step / (k3_ms / 1e3) / 1e12
        stages["K3_gauss_rows"] = {"ms_per_launch": round(k3_ms, 4), "launches_per_step": k3_per_step,
                                   "share_of_step": round(k3_sum / max(local_ms, 1e-9), 4),
                                   "flops_per_p": k3_flops_p, "exps_per_p": s * n, "tflops": round(k3_tf, 3),
                                   "frac_dmma_peak": round(k3_tf / FP64_DMMA_PEAK_TFLOPS, 4)}
    if k3_per_step and k3_sum >= k4_sum:
        st = stages["K3_gauss_rows"]
        roofline = {"bound": "tensor", "pipe": "FP64 DMMA.8x8x4 (shared with DFMA)",
                    "kernel": "k_gauss_rows (K3; one span over its fast-exp and masked-exp launches, CUDA events "
                              "on the launching stream)", "achieved": st["tflops"], "peak": FP64_DMMA_PEAK_TFLOPS,
                    "frac": st["frac_dmma_peak"], "traffic": ncu_traffic("k_gauss_rows"),
                    "algorithmic_flops_per_p": st["flops_per_p"], "launch_ms": st["ms_per_launch"],
                    "share_of_step": st["share_of_step"]}
    else:
        st = stages["K4_lsq"]
        roofline = {"bound": "fp64", "pipe": "FP64 DFMA",
                    "kernel": ("K4 batched Householder least squares, compact-WY on DMMA (k_lsq_wy; the stencil rows "
                               "are assembled by k_wy_stencil_rows, see stages; CUDA events on the launching stream)"
                               if k2_per_step else
                               "K4 batched Householder least squares with the fused row assembly (k_lsq_*; CUDA "
                               "events on the launching stream)"), "achieved": st["tflops"],
                    "peak": FP64_DFMA_PEAK_TFLOPS, "frac": st["frac_dfma_peak"],
                    "traffic": ncu_traffic(f"k_lsq@cfg{cfg}"), "algorithmic_flops_per_p": st["flops_per_p"],
                    "launch_ms": st["ms_per_launch"], "share_of_step": st["share_of_step"]}
    roofline.update({"unit": "TFLOP/s", "peak_source": PEAK_SOURCE})

    # ---- CPU baseline (rank 0, N=1 only) ------------------------------------
    cpu = None
    if env.rank == 0 and env.world == 1 and not args.no_cpu_baseline:
        Xh = basis.basis.cpu().numpy() if hasattr(basis.basis, "cpu") else np.asarray(basis.basis)
        cref = CpuReference(prob, Xh, np.asarray(sel.indices), sel.weights, basis.singular_values)
        cpu = cref.baseline(my_params, args.cpu_seconds)

    if env.rank == 0:
        op = sysm.operator
        shape = (f"n={n} r={r} s={s}" + (f" d={op.points.shape[1]}" if hasattr(op, "points") else "")
                 + (" complex128" if g.complex else ""))
        line = {
            "metric": "SubApSnap online solves/sec (p-values/s)",
            "value": round(value, 1), "unit": "p-values/s", "n_gpus": env.world, "steps": K, "warmup": W,
            "ms_per_step": round(ms_per_step, 4), "higher_is_better": True, "scaling": args.scaling,
            "vs_baseline": None, "dtype": "c128" if g.complex else "f64",
            "data": f"synthetic (seeded, BASELINE config {cfg} definition, paper_2510_04825_b200/problems.py)",
            "config": {"workload": f"config {cfg} {prob.key}: {shape}, "
                                   + (f"{P_all} parameter values per step sharded over {env.world} GPU(s)"
                                      if args.scaling == "strong" else f"{P_all // env.world} per GPU"),
                       "P_per_step": P_all, "P_per_gpu": Pl, "l2": "flushed between steps (256 MiB write)",
                       "offline_s": round(t_off, 2), "plan_s": round(t_plan, 3),
                       "parallelism": f"p-sharded x{env.world}" + (" (shared GPU, gloo)" if shared else "")},
            "e2e": {"value": round(e2e_val, 1), "unit": "p-values/s", "h2d_bytes_per_step": int(h2d),
                    "d2h_bytes_per_step": int(d2h),
                    "api": ("sas_solve_host (C ABI, pinned host buffers)" if env.world == 1 else
                            "pinned H2D of each shard, sas_solve, all-gather of the rows, D2H on rank 0")},
            "gpu_launches": int(launches),
            "roofline": roofline,
            "stages": stages,
            "cpu_baseline": cpu,
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if env.world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def run_reference_arm(args, env):
    """--impl reference: the reference's own CPU online path (solve_batch from
    the baseline/_ref install; the oracle port if it is missing) on all host
    cores of this box.  Rank 0 alone runs and prints; other ranks exit 0."""
    if env.rank != 0:
        return
    import torch
    dev = torch.device("cuda:0") if torch.cuda.is_available() else None
    from paper_2510_04825_b200 import problems
    from paper_2510_04825_b200.offline import offline
    cfg = args.config
    prob = problems.build(cfg)
    basis, sel = offline(prob, device=dev)   # inputs only (untimed), the recipe our arm uses
    P_all = args.P or (P_TOTAL[cfg] if args.scaling == "strong" else P_PER_GPU[cfg] * env.world)
    params = prob.test_params(P_all)
    cref = CpuReference(prob, np.asarray(basis.basis), np.asarray(sel.indices), sel.weights, basis.singular_values)
    # protocol choice on a probe: workers=1 (default BLAS) vs workers=cores (1 BLAS thread)
    per1 = cref.run(params[:2], 1) / 2
    wmax = cref.max_workers()
    perw = cref.run(params[:max(2, wmax)], wmax) / max(2, wmax) if wmax > 1 else float("inf")
    workers, per = (wmax, perw) if perw < per1 else (1, per1)
    budget = max(0.5, min(6.0, 150.0 / max(args.steps + args.warmup, 1)))
    count = int(min(len(params), max(2, workers, budget / max(per, 1e-9))))
    if cref.dense_row_bytes > (4 << 30):
        count = min(count, 2)
    sample = list(params[:count])
    for _ in range(args.warmup):
        cref.run(sample[:max(1, min(len(sample), workers))], workers)
    total = 0.0
    for _ in range(args.steps):
        total += cref.run(sample, workers)
    value = count * args.steps / total
    what = ("reference online.solve_batch (baseline/_ref)" if cref.kind == "reference"
            else "oracle port oracle/online_ref.py (reference not importable)")
    line = {
        "metric": "SubApSnap online solves/sec (p-values/s)", "impl": "reference",
        "value": round(value, 3), "unit": "p-values/s", "n_gpus": env.world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": round(total / args.steps * 1e3, 3), "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "c128" if cfg == 4 else "f64",
        "data": f"synthetic (seeded, BASELINE config {cfg} definition, paper_2510_04825_b200/problems.py)",
        "config": {"workload": f"config {cfg} {prob.key}: n={prob.system.n} r={basis.rank} s={sel.size}; each step "
                               f"= the first {count} of the {P_all} parameter values",
                   "parallelism": f"solve_batch workers={workers}" + (" (1 BLAS thread each)" if workers > 1
                                                                       else " (default BLAS threads)")},
        "cpu_baseline": {"value": round(value, 3), "unit": "p-values/s", "cores": cref.cores, "kind": cref.kind,
                         "host_cores": cref.cores, "cpu_model": cpu_model(),
                         "sample": f"{count} parameter values per step through {what}, perf_counter around "
                                   f"solve_batch (cli.py:338-343); inputs X, S, w from the offline recipe "
                                   f"both arms share (untimed)"},
        "e2e": {"value": round(value, 3), "unit": "p-values/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


if __name__ == "__main__":
    main()
