"""Per-launch stage times of one config's sweep (sas_plan_set_timing).
Usage: python tools/stage_times.py <config> [P] [--synthetic]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

from paper_2510_04825_b200 import online, problems  # noqa: E402
from paper_2510_04825_b200.offline import offline  # noqa: E402

argv = [a for a in sys.argv[1:] if not a.startswith("--")]
cfg = int(argv[0])
P = int(argv[1]) if len(argv) > 1 else {1: 1000, 2: 4096, 3: 65536, 4: 100000, 5: 125000}[cfg]
prob = problems.build(cfg)
dev = torch.device("cuda:0")
if "--synthetic" in sys.argv and cfg != 2:
    from bench_configs import synthetic_basis
    basis, sel = synthetic_basis(prob, {1: 8, 3: 40, 4: 30, 5: 50}[cfg], complex_=(cfg == 4), device=dev)
else:
    basis, sel = offline(prob, device=dev, prefer_cg=True) if cfg in (3, 5) else offline(prob, device=dev)
plan = online.precompute_online(prob.system, basis, sel)
params = prob.test_params(P)
pt = online.device_params(plan, params)
out = online.alloc_outputs(plan, P)
online.solve_device(plan, pt, out)
torch.cuda.synchronize()
g = plan.gpu
g.set_timing(True)
for _ in range(2):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    online.solve_device(plan, pt, out)
    e1.record()
    torch.cuda.synchronize()
    st = list(g.stage_times())
    tot = {}
    for sid, ms in st:
        tot[sid] = tot.get(sid, 0.0) + ms
    print("sweep %.3f ms, launches %d, per stage id %s" % (e0.elapsed_time(e1), len(st),
                                                            {k: round(v, 3) for k, v in tot.items()}))
print("first launches:", [(sid, round(ms, 3)) for sid, ms in st[:6]])
