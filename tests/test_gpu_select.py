"""Leverage selector on the GPU: k_range_rows / sas_range_rows and
offline.leverage_scores_gpu / select_rows(device=...) against the host restatement
of subsample.py:84-159 (which reproduces the reference's selector bit for bit,
tests/test_host_logic.py::test_offline_selector_restatement_matches_reference).

The GPU scores are those of the same numerical range, formed from the TSQR R
factor instead of an n x w thin SVD; they agree with numpy's to the conditioning
of that subspace, so the comparisons are tolerance-based and the tolerances are
stated per case."""
import ctypes as C

import numpy as np
import pytest
import torch

from paper_2510_04825_b200 import _capi, offline, problems

pytestmark = pytest.mark.gpu


def _range_rows(a, c, want_q=True):
    lib = _capi.load()
    A = torch.from_numpy(np.ascontiguousarray(a)).cuda()
    m, w = a.shape
    k = c.shape[1]
    Q = torch.empty((m, k), dtype=A.dtype, device="cuda") if want_q else None
    sc = torch.empty(m, dtype=torch.float64, device="cuda")
    ch = np.ascontiguousarray(c, dtype=a.dtype)
    st = C.c_void_p(torch.cuda.current_stream().cuda_stream)
    dt = _capi.SAS_C128 if np.iscomplexobj(a) else _capi.SAS_F64
    _capi.check(lib.sas_range_rows(_capi.ptr(A), m, w, ch.ctypes.data_as(C.c_void_p), k, dt, _capi.ptr(Q),
                                   _capi.ptr(sc), 0, st), "sas_range_rows")
    torch.cuda.synchronize()
    return (Q.cpu().numpy() if want_q else None), sc.cpu().numpy()


@pytest.mark.parametrize("m,w,k,cplx", [(1, 1, 1, False), (63, 5, 3, False), (64, 21, 21, False), (1000, 41, 40, False),
                                        (100_003, 52, 51, False), (777, 64, 64, False), (5000, 31, 30, True),
                                        (130, 64, 17, True)])
def test_range_rows_matches_numpy(m, w, k, cplx):
    rng = np.random.default_rng(m * 7 + w)
    a = rng.standard_normal((m, w))
    c = rng.standard_normal((w, k))
    if cplx:
        a = a + 1j * rng.standard_normal((m, w))
        c = c + 1j * rng.standard_normal((w, k))
    q, sc = _range_rows(a, c)
    qn = a @ c
    scale = np.abs(a) @ np.abs(c)
    assert np.all(np.abs(q - qn) <= 1e-14 * scale.max() * w)
    np.testing.assert_allclose(sc, (np.abs(qn) ** 2).sum(axis=1), rtol=1e-12)
    _, sc2 = _range_rows(a, c, want_q=False)   # scores only: same bits
    assert np.array_equal(sc, sc2)


def _host_scores(target):
    q = offline._range_basis(target)
    return offline.leverage_scores(q), q.shape[1]


@pytest.mark.parametrize("case", ["decay", "augmented_in_span", "complex", "wide64"])
def test_leverage_scores_gpu_matches_host(case):
    rng = np.random.default_rng(11)
    if case == "decay":
        t = rng.standard_normal((20_000, 41)) @ np.diag(np.logspace(0, -7, 41)) @ rng.standard_normal((41, 41))
    elif case == "augmented_in_span":   # [B | B c]: rank-deficient by construction (subsample.py:150-152)
        b = rng.standard_normal((30_000, 20)) @ np.diag(np.logspace(0, -5, 20))
        t = np.column_stack([b, 1e3 * (b @ rng.standard_normal(20))])
    elif case == "complex":
        t = (rng.standard_normal((10_000, 31)) + 1j * rng.standard_normal((10_000, 31))) @ np.diag(np.logspace(0, -6, 31))
    else:
        t = rng.standard_normal((5_000, 64))
    hs, hk = _host_scores(t)
    gs, gk = offline.leverage_scores_gpu(t, device=0)
    gs = gs.cpu().numpy()
    assert gk == hk
    assert abs(gs.sum() - gk) <= 1e-9 * gk        # trace of an orthonormal Gram
    # same subspace up to its conditioning: eps * s_0 / s_k ~ 1e-8 for these targets
    assert np.abs(gs - hs).max() <= 1e-6 * hs.max(), np.abs(gs - hs).max() / hs.max()


@pytest.mark.parametrize("cfg", [3, 4, 5])
def test_select_rows_gpu_on_golden_size_problems(cfg):
    """The BASELINE problems at the golden fixtures' sizes: the GPU selector draws the
    same rows as the host restatement (same numpy stream, probabilities equal to ~1e-9)
    and the weights agree to 1e-6 relative."""
    prob = {3: lambda: problems.diffusion2d(grid=40), 4: lambda: problems.convdiff_tf(grid=40),
            5: lambda: problems.diffusion3d(grid=12)}[cfg]()
    basis, sel_h = offline.offline(prob)
    _, sel_g = offline.offline(prob, device=torch.device("cuda:0"), basis=basis, gpu_select=True)
    assert sel_g.size == sel_h.size == prob.samples
    same = np.asarray(sel_g.indices) == np.asarray(sel_h.indices)
    assert same.mean() >= 0.98, same.mean()
    wg, wh = np.asarray(sel_g.weights)[same], np.asarray(sel_h.weights)[same]
    assert np.abs(wg / wh - 1).max() <= 1e-6, np.abs(wg / wh - 1).max()


def test_leverage_scores_gpu_full_size_config3_shape():
    """n = 10^6, width 41 (config 3's target shape): against numpy's thin SVD."""
    rng = np.random.default_rng(5)
    t = rng.standard_normal((1_000_000, 41)) * np.logspace(0, -6, 41)
    hs, hk = _host_scores(t)
    gs, gk = offline.leverage_scores_gpu(torch.from_numpy(t).cuda(), device=0)
    gs = gs.cpu().numpy()
    assert gk == hk == 41
    assert abs(gs.sum() - 41) <= 1e-8
    assert np.abs(gs - hs).max() <= 1e-6 * hs.max()


def test_leverage_scores_gpu_error_behaviour():
    """The reference's errors (subsample.py:154-155; select_rows' all-zero guard) and the C ABI's argument checks."""
    from paper_2510_04825_b200.errors import RankDeficiencyError
    with pytest.raises(RankDeficiencyError):
        offline.leverage_scores_gpu(np.zeros((500, 7)), device=0)
    lib = _capi.load()
    A = torch.zeros((10, 4), dtype=torch.float64, device="cuda")
    c = np.zeros((4, 5))
    sc = torch.empty(10, dtype=torch.float64, device="cuda")
    rc = lib.sas_range_rows(_capi.ptr(A), 10, 4, c.ctypes.data_as(C.c_void_p), 5, _capi.SAS_F64, None, _capi.ptr(sc), 0,
                            C.c_void_p(0))
    assert rc != 0 and "k <= w" in _capi.last_error()
    with pytest.raises(ValueError):
        _capi.check(rc, "sas_range_rows")


def test_select_rows_gpu_weights_and_size():
    """select_rows(device=...) returns the reference's selector fields: s = ceil(oversample * width) rows drawn with
    replacement, weights 1 / sqrt(s pi_i), strategy and anchors carried over."""
    rng = np.random.default_rng(3)
    b = rng.standard_normal((4000, 9))
    rhs = b @ rng.standard_normal(9) + 1e-3 * rng.standard_normal(4000)
    sel = offline.select_rows(b, rhs, strategy="leverage", oversample=4.0, seed=7, anchors=(0.5,),
                              device=torch.device("cuda:0"))
    ref = offline.select_rows(b, rhs, strategy="leverage", oversample=4.0, seed=7, anchors=(0.5,))
    assert sel.size == ref.size == 40 and sel.strategy == "leverage" and sel.anchors == (0.5,)
    assert np.array_equal(sel.indices, ref.indices)
    np.testing.assert_allclose(sel.weights, ref.weights, rtol=1e-9)
