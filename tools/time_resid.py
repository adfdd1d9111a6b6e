"""Time the full-residual checker (sas_residual: K5 lift + K6 stencil/affine
residual) on the first P parameter values of a config (synthetic basis).
Usage: python tools/time_resid.py <config> [P]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

from bench_configs import synthetic_basis  # noqa: E402
from paper_2510_04825_b200 import online, problems  # noqa: E402

cfg = int(sys.argv[1])
P = int(sys.argv[2]) if len(sys.argv) > 2 else 1024
prob = problems.build(cfg)
dev = torch.device("cuda:0")
basis, sel = synthetic_basis(prob, {3: 40, 4: 30, 5: 50}[cfg], complex_=(cfg == 4), device=dev)
plan = online.precompute_online(prob.system, basis, sel)
params = prob.test_params(P)
res = online.solve_params(plan, params)
online.relative_residual(plan, params[:64], res.coefficients[:64])   # operator upload + warm-up
ts = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rr, fl = online.relative_residual(plan, params, res.coefficients, return_floor=True)
    ts.append(time.perf_counter() - t0)
ts2 = []
for _ in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rr2 = online.relative_residual(plan, params, res.coefficients)
    ts2.append(time.perf_counter() - t0)
assert (rr2 == rr).all()
n = prob.system.n
print(json.dumps({"config": cfg, "P": P, "n": n, "seconds": min(ts), "seconds_without_floor": min(ts2), "ms_per_p": 1e3 * min(ts) / P,
                  "relres_first": float(rr[0]), "floor_first": float(fl[0])}))
