"""Run a few solves of one BASELINE config on cuda:0 (a short command for ncu
captures).  Usage: python tools/run_cfg.py <config> [P] [reps] [--synthetic]
(--synthetic: seeded orthonormal basis instead of the offline snapshot solves;
the online cost does not depend on the values of X)."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

from paper_2510_04825_b200 import online, problems  # noqa: E402
from paper_2510_04825_b200.offline import offline  # noqa: E402

argv = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = int(argv[0])
P = int(argv[1]) if len(argv) > 1 else None
reps = int(argv[2]) if len(argv) > 2 else 2
prob = problems.build(cfg)
if "--synthetic" in sys.argv and cfg != 2:
    sys.path.insert(0, str(Path(__file__).resolve().parent))
    from bench_configs import synthetic_basis
    basis, sel = synthetic_basis(prob, {1: 8, 3: 40, 4: 30, 5: 50}[cfg], complex_=(cfg == 4),
                                 device=torch.device("cuda:0"))
else:
    basis, sel = offline(prob, device=torch.device("cuda:0"))
plan = online.precompute_online(prob.system, basis, sel)
params = prob.test_params(P or {1: 1000, 2: 4096, 3: 65536, 4: 100000, 5: 125000}[cfg])
pt = online.device_params(plan, params)
out = online.alloc_outputs(plan, len(params))
for _ in range(reps):
    online.solve_device(plan, pt, out)
torch.cuda.synchronize()
print("ok", cfg, len(params), int((out["status"] != 0).sum()))
