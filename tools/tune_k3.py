"""Time K3/K4 variants on the config-2 workload (one process per variant because
the variant is read once from SAS_K3_VARIANT).  Usage: python tools/tune_k3.py"""
import json
import os
import subprocess
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
VARIANTS = os.environ.get("VARIANTS", "4,2,1 4,2,0 2,3,1 2,3,0 3,2,1 2,2,1").split()

CHILD = r'''
import json, sys, time
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
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
ref = np.load(sys.argv[2]) if len(sys.argv) > 2 else None
print(json.dumps({"k3_ms": min(k3), "k4_ms": min(k4), "tflops": 2*80*20000*20*4096/min(k3)/1e9,
                  "coef0": out["coef"][0, :3].tolist()}))
'''

for v in VARIANTS:
    env = dict(os.environ, SAS_K3_VARIANT=v)
    r = subprocess.run([sys.executable, "-c", CHILD, str(ROOT)], env=env, capture_output=True, text=True)
    line = r.stdout.strip().splitlines()[-1] if r.stdout.strip() else r.stderr[-500:]
    print(v, line, flush=True)
