"""Offline pieces on the GPU kernels: the config-4 BiCGSTAB snapshot solve (sas_bicgstab_csr)
and the leverage scores of a config-5-shaped target (sas_tsqr_r + sas_range_rows) against
numpy's thin SVD on the host.  Usage: python tools/time_offline.py [--no-host-svd]"""
import json
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_04825_b200 import offline, problems  # noqa: E402

dev = torch.device("cuda:0")
torch.zeros(1, device=dev)

prob = problems.build(4)
s = prob.system
offline._affine_bicgstab(s, prob.snapshot_points[0], dev)   # warm-up
for p in prob.snapshot_points[:3]:
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = offline._affine_bicgstab(s, p, dev)
    dt = time.perf_counter() - t0
    a = s.matrix(p)
    b = np.asarray(s.full_rhs(p))
    print(json.dumps({"what": "config 4 snapshot solve, fused BiCGSTAB (incl. CSR assembly + upload)", "p": str(p),
                      "n": int(s.n), "seconds": round(dt, 3),
                      "true_relres": float(np.linalg.norm(a @ x - b) / np.linalg.norm(b))}))

rng = np.random.default_rng(0)
n, w = 10_077_696, 51
t = torch.from_numpy(rng.standard_normal((n, w)) * np.logspace(0, -5, w)).to(dev)
offline.leverage_scores_gpu(t[:100_000], device=dev)   # warm-up
torch.cuda.synchronize()
t0 = time.perf_counter()
sc, keep = offline.leverage_scores_gpu(t, device=dev)
torch.cuda.synchronize()
dt = time.perf_counter() - t0
out = {"what": "leverage scores, config-5 target shape (TSQR + range_rows, two passes)", "n": n, "w": w, "keep": keep,
       "gpu_seconds": round(dt, 3), "score_sum": float(sc.sum())}
if "--no-host-svd" not in sys.argv:
    th = t.cpu().numpy()
    t0 = time.perf_counter()
    q = offline._range_basis(th)
    hs = offline.leverage_scores(q)
    out["host_svd_seconds"] = round(time.perf_counter() - t0, 3)
    out["max_abs_diff_over_max_score"] = float(np.abs(hs - sc.cpu().numpy()).max() / hs.max())
print(json.dumps(out))
