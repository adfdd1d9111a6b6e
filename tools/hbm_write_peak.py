"""Write-only HBM bandwidth on this GPU (fill of a 1.6 GB buffer, CUDA events, best of 10):
the roofline of k_wy_stencil_rows, whose only HBM traffic is its output stream."""
import json
import torch

n = 200 * 1024 * 1024  # doubles: 1.6 GB, larger than L2
x = torch.empty(n, dtype=torch.float64, device="cuda")
best = 1e9
for _ in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    x.fill_(1.0)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1))
print(json.dumps({"test": "fill 1.6 GB (write only)", "ms": round(best, 4), "write_gbs": round(n * 8 / best / 1e6, 1)}))
