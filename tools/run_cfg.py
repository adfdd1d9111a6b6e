"""Run a few solves of one BASELINE config on cuda:0 (a short command for ncu
captures).  Usage: python tools/run_cfg.py <config> [P] [reps]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_04825_b200 import online, problems  # noqa: E402
from paper_2510_04825_b200.offline import offline  # noqa: E402

cfg = int(sys.argv[1])
P = int(sys.argv[2]) if len(sys.argv) > 2 else None
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 2
prob = problems.build(cfg)
basis, sel = offline(prob, device=torch.device("cuda:0"))
plan = online.precompute_online(prob.system, basis, sel)
params = prob.test_params(P or {1: 1000, 2: 4096, 3: 65536, 4: 100000, 5: 125000}[cfg])
pt = online.device_params(plan, params)
out = online.alloc_outputs(plan, len(params))
for _ in range(reps):
    online.solve_device(plan, pt, out)
torch.cuda.synchronize()
print("ok", cfg, len(params), int((out["status"] != 0).sum()))
