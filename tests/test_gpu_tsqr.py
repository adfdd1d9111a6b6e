"""TSQR kernels (k_tsqr_block, sas_tsqr_r) and their caller solve_apsnap.

* R of tall real/complex matrices against numpy's qr R, up to the phases of
  its rows (the R factor is unique up to them): one block, several levels,
  m < w, the w <= 48 / w > 48 block sizes, w = 1 and w = 64;
* solve_apsnap (online.py:156-165) on it is covered by
  test_gpu_parity.py::test_solve_apsnap_matches_oracle and
  test_full_selector_equals_apsnap."""
import numpy as np
import pytest
import torch

from paper_2510_04825_b200 import online

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("m,w,cplx", [(50, 7, False), (256, 17, False), (3000, 41, False), (100_000, 51, False),
                                      (20, 30, False), (5000, 64, False), (777, 1, False), (4000, 31, True),
                                      (600, 64, True), (130, 49, False)])
def test_tsqr_r_matches_numpy_up_to_row_phases(m, w, cplx):
    rng = np.random.default_rng(m + w)
    a = rng.standard_normal((m, w)) * np.logspace(0, -6, w)
    if cplx:
        a = a + 1j * rng.standard_normal((m, w)) * np.logspace(0, -6, w)
    R = online.tsqr_r(torch.from_numpy(a).cuda()).cpu().numpy()
    Rn = np.linalg.qr(a, mode="r")
    k = min(m, w)
    assert np.all(np.tril(R, -1) == 0) and np.all(R[k:] == 0)
    Rn = np.vstack([Rn, np.zeros((w - Rn.shape[0], w))]) if Rn.shape[0] < w else Rn
    for i in range(k):
        ph = R[i, i] / Rn[i, i]
        assert abs(abs(ph) - 1) < 1e-10
        np.testing.assert_allclose(R[i, i:], ph * Rn[i, i:], rtol=0, atol=1e-12 * np.abs(Rn[i, i:]).max() + 1e-300)
