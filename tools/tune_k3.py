"""Time K3 variants on the config-2 workload (one process per variant because
the variant is read once from the environment).  A variant is
"pw,minb[,maxw[,ksplit]]" (SAS_K3_VARIANT; maxw -> SAS_K3_MAXW, the
warps per CTA row block; ksplit -> SAS_K3_KSPLIT, "a" = automatic).  Each line also reports the worst coefficient difference
against the CPU oracle on 4 bandwidths.   Usage: VARIANTS="..." python tools/tune_k3.py"""
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
VARIANTS = os.environ.get("VARIANTS", "4,2,10,a 4,2,10,1 3,2,10,a").split()

CHILD = r'''
import json, sys, time
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
from oracle import online_ref
from paper_2510_04825_b200 import online, problems, _capi
from paper_2510_04825_b200.offline import offline
prob = problems.gauss_krr()
basis, sel = offline(prob, device=torch.device("cuda:0"))
plan = online.precompute_online(prob.system, basis, sel)
params = prob.test_params(4096)
pt = online.device_params(plan, params)
out = online.alloc_outputs(plan, len(params))
for _ in range(3): online.solve_device(plan, pt, out)
torch.cuda.synchronize()
plan.gpu.set_timing(True)
k3 = []; k4 = []
for _ in range(10):
    online.solve_device(plan, pt, out)
    for sid, ms in plan.gpu.stage_times():
        (k3 if sid == _capi.SAS_STAGE_GAUSS_ROWS else k4).append(ms)
coef = out["coef"].cpu().numpy() if hasattr(out["coef"], "cpu") else np.asarray(out["coef"])
op = prob.system.operator
worst = 0.0
for k in (0, 1, 2049, 4095):
    p = params[k]
    fn = lambda q, rows: online_ref.gauss_rows(op.points, rows, float(q), op.ridge)
    m = online_ref.sampled_rows(fn, basis.basis, sel.indices, p)
    c, _, _ = online_ref.solve_one(m, prob.system.rhs(p, sel.indices), sel.weights)
    worst = max(worst, float(np.linalg.norm(coef[k] - c) / np.linalg.norm(c)))
print(json.dumps({"k3_ms": min(k3), "k4_ms": min(k4), "tflops": 2*80*20000*20*4096/min(k3)/1e9,
                  "max_rel_vs_oracle": worst}))
'''

for v in VARIANTS:
    f = v.split(",")
    env = dict(os.environ, SAS_K3_VARIANT=",".join(f[:2]))
    if len(f) >= 3:
        env["SAS_K3_MAXW"] = f[2]
    if len(f) >= 4 and f[3] != "a":
        env["SAS_K3_KSPLIT"] = f[3]
    r = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=env, capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-800:]
    print(v, line, flush=True)
