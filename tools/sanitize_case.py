"""Small end-to-end case for compute-sanitizer (one tool per gpurun call):
every kernel family once -- K3 + K4 (Gaussian rows, n=1024), K2 + K4
column-owner (2-D stencil, 48^2), K1 + K4 shared-memory kernel (complex
affine, 40^2, r'=30 via a synthetic basis), K5 lift and the K6 residual checker.
Usage: compute-sanitizer --tool memcheck python tools/sanitize_case.py"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2510_04825_b200 import online, problems  # noqa: E402
from paper_2510_04825_b200.offline import offline  # noqa: E402
from bench_configs import synthetic_basis  # noqa: E402

dev = torch.device("cuda:0")
for name, prob, mk in [("gauss", problems.gauss_krr(n=1024), None),
                       ("stencil2d", problems.diffusion2d(grid=48), None),
                       ("affine_c128", problems.convdiff_tf(grid=40), 30)]:
    if mk:
        basis, sel = synthetic_basis(prob, mk, complex_=True, device=dev)
    else:
        basis, sel = offline(prob, device=dev)
    plan = online.precompute_online(prob.system, basis, sel)
    params = prob.test_params(37)
    res = online.solve_params(plan, params)
    assert np.all(res.status == 0), (name, res.status)
    x = online.lift_batch(plan, res.coefficients[:3])
    rr = online.relative_residual(plan, params[:3], res.coefficients[:3])
    print(name, "ok", x.shape, np.round(rr, 6))
