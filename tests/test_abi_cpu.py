"""CPU-side checks of the C-ABI library: it loads without a GPU, exports every
function include/dmpq.h declares, and its host-pure decision functions agree with
the oracle. No device compute is called here."""
import math
import os
import re

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2603_18742_b200 import build, _lib
    build.build()
    return _lib


def _header_functions():
    src = open(os.path.join(ROOT, "include", "dmpq.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    names = re.findall(r"^\s*[A-Za-z_][\w\s\*]*?\b([a-z_][a-z0-9_]*)\s*\(", src, flags=re.M)
    return sorted(set(n for n in names if n.startswith(("dmpq_", "tdc_"))))


def test_library_exports_every_header_symbol(L):
    lib = L.lib()
    declared = _header_functions()
    assert len(declared) >= 14
    for name in declared:
        assert hasattr(lib, name), f"libdmpq.so does not export {name}"
    assert sorted(L.exported_names()) == declared, "binding signatures out of sync with include/dmpq.h"


def test_sizing_helpers(L, orc):
    lib = L.lib()
    for m, k in [(1, 64), (128, 128), (300, 1920), (17776, 3072), (2222, 12288)]:
        assert lib.dmpq_sf_bytes(m, k) == orc.sf_swizzled_bytes(m, k)
    assert lib.dmpq_sf_bytes(0, 64) == 0
    assert lib.tdc_workspace_bytes(17776, 3072) >= 148 * 4 * 7 * 8


def test_validation_without_gpu(L):
    """Argument validation happens before any device work and reports statuses."""
    from paper_2603_18742_b200 import dmpq
    import ctypes
    lib = L.lib()
    rc = lib.dmpq_quantize_act(None, 4, 100, 100, None, None, None, None, None)
    assert rc == L.DMPQ_EINVAL
    act = L.Act(L.FMT_INT8, 4, 100, 16, None, None, 16)
    rc = lib.dmpq_quantize_act(ctypes.c_void_p(16), 4, 100, 104, None, ctypes.byref(act), None, None, None)
    assert rc == L.DMPQ_ESHAPE and b"k % 64" in lib.dmpq_last_error()
    rc = lib.tdc_step(7, None, None, None, 1, 8, None, None, None)
    assert rc == L.DMPQ_EINVAL
    cache = L.TdcNvfp4Cache(16, 16, 16)
    rc = lib.tdc_step_nvfp4(L.TDC_SKIP, None, None, ctypes.byref(cache), None, None, 4, 96, None, None, None)
    assert rc == L.DMPQ_ESHAPE and b"h % 64" in lib.dmpq_last_error()
    rc = lib.tdc_step_nvfp4(L.TDC_SKIP, None, None, None, None, None, 4, 128, None, None, None)
    assert rc == L.DMPQ_EINVAL
    rc = lib.tdc_step_nvfp4(L.TDC_REFRESH, ctypes.c_void_p(16), ctypes.c_void_p(16), ctypes.byref(cache), None, None,
                            4, 128, None, None, None)
    assert rc == L.DMPQ_EINVAL   # X_out aliases X_in
    assert lib.tdc_delta_amax(None, None, 4, 12, None, None) == L.DMPQ_ESHAPE


def test_derive_tau_matches_oracle(L, orc):
    from paper_2603_18742_b200 import dmpq
    rng = np.random.default_rng(0)
    for _ in range(500):
        a, b, tr = rng.uniform(-0.1, 2), rng.uniform(-0.01, 0.01), rng.uniform(0, 0.05)
        assert dmpq.dmpq_derive_tau(a, b, tr) == orc.derive_tau_gamma(a, b, tr)
    assert dmpq.dmpq_derive_tau(0.1, 0.001, 0.0025) == pytest.approx(0.015, rel=1e-12)


def test_predict_matches_oracle(L, orc):
    from paper_2603_18742_b200 import dmpq
    rng = np.random.default_rng(1)
    taus = [0.015, 0.01, 0.0043, 0.02, 0.0075, 0.012]
    for trial in range(2000):
        st = list(rng.uniform(0, 1, 7))
        st[1] = st[0] / rng.uniform(0.002, 0.05) if trial % 50 else 0.0
        t = int(rng.integers(0, 5))
        ps = bool(rng.integers(0, 2))
        fmts, gamma, rc = dmpq.dmpq_predict(st, taus, t, ps)
        g_or = orc.gamma_from_stats(st)
        ref = orc.route_block(g_or, taus, t, ps)
        assert fmts == ref
        if t > 0 and not ps and g_or is not None:
            assert gamma == g_or
        if st[1] == 0.0 and t > 0 and not ps:
            assert rc == L.DMPQ_EZERONORM
    # equality routes NVFP4 (Eq. 7 "<=")
    fmts, _, _ = dmpq.dmpq_predict([0.015, 1.0, 0, 0, 0, 0, 0], [0.015], 3, False)
    assert fmts == [orc.FMT_NVFP4]


@pytest.mark.parametrize("metric", ["cos", "rel_l2"])
def test_tdc_host_matches_oracle(L, orc, metric):
    from paper_2603_18742_b200 import dmpq
    rng = np.random.default_rng(2)
    for trial in range(300):
        cfg_o = orc.TdcConfig(rho=float(rng.uniform(0, 0.002)), tau=float(rng.uniform(0, 0.006)) * (30 if metric != "cos" else 1),
                              n_max=int(rng.integers(1, 4)), metric=metric)
        cfg_c = L.TdcConfig(cfg_o.rho, cfg_o.tau, cfg_o.n_max, L.TDC_METRIC_REL_L2 if metric == "rel_l2" else L.TDC_METRIC_COS)
        so, sc = orc.TdcState(), dmpq.tdc_new_state()
        for t in range(30):
            do = orc.tdc_decide(so, cfg_o, t)
            dc = dmpq.tdc_decide(sc, cfg_c, t)
            assert do == dc, (trial, t)
            # synthetic stats whose cosine error straddles tau
            cos = 1.0 - float(rng.uniform(0, 0.006))
            st = [0, 1, 0, 1, cos, 1.0, 1.0]
            e = orc.prediction_error_from_stats(st, metric)
            orc.tdc_update(so, cfg_o, t, do, e)
            dmpq.tdc_update(sc, cfg_c, t, dc, st)
            assert sc.e_acc == so.e_acc and sc.t_p == so.t_p


def test_purify_matches_oracle(L, orc):
    from paper_2603_18742_b200 import dmpq
    rng = np.random.default_rng(3)
    for _ in range(500):
        fm = [int(v) for v in rng.integers(0, 2, 6)]
        ratios = list(rng.uniform(0, 50, 6))
        ratios[int(rng.integers(0, 6))] = 25.0
        ps = bool(rng.integers(0, 2))
        got = dmpq.dmpq_purify(fm, ratios, ps, 25.0)
        assert got == [orc.purify_route(f, r, ps, 25.0) for f, r in zip(fm, ratios)]
    assert dmpq.dmpq_purify([1, 1], None, True) == [0, 0]


def test_predict_l2_metric_matches_oracle(L, orc):
    """dmpq_predict with the L2 Gamma variant (DMPQ_GAMMA_L2, R1) against the oracle's
    gamma_from_stats(metric="l2") and Eq. 7 routing; SPEC rel_l2 examples via the statistics."""
    from paper_2603_18742_b200 import dmpq
    rng = np.random.default_rng(4)
    taus = [0.015, 0.01, 0.0043, 0.02, 0.0075, 0.012]
    for trial in range(2000):
        st = list(rng.uniform(0, 1, 7))
        st[3] = st[2] / rng.uniform(0.002, 0.05) ** 2 if trial % 50 else 0.0
        t = int(rng.integers(0, 5))
        ps = bool(rng.integers(0, 2))
        fmts, gamma, rc = dmpq.dmpq_predict(st, taus, t, ps, metric=L.GAMMA_L2)
        g_or = orc.gamma_from_stats(st, "l2")
        assert fmts == orc.route_block(g_or, taus, t, ps)
        if t > 0 and not ps and g_or is not None:
            assert gamma == pytest.approx(g_or, rel=1e-15)
        if st[3] == 0.0 and t > 0 and not ps:
            assert rc == L.DMPQ_EZERONORM
    # ref [3, 4] vs other [0, 0]: sum d^2 = 25, sum x^2 = 25 -> Gamma_L2 = 1 -> INT8 at tau 0.015
    fmts, gamma, _ = dmpq.dmpq_predict([7, 7, 25, 25, 0, 0, 0], [0.015, 2.0], 3, False, metric=L.GAMMA_L2)
    assert gamma == 1.0 and fmts == [orc.FMT_INT8, orc.FMT_NVFP4]
    # the same statistics under L1 give Gamma = 1 as well; a case where they differ: L1 0.5, L2 1/sqrt(2)
    st = [1.0, 2.0, 1.0, 2.0, 0, 0, 0]
    assert dmpq.dmpq_predict(st, [0.6], 3, False)[1] == 0.5
    assert dmpq.dmpq_predict(st, [0.6], 3, False, metric=L.GAMMA_L2)[1] == pytest.approx(2 ** -0.5, rel=1e-15)
    assert dmpq.dmpq_predict(st, [0.6], 3, False, metric=L.GAMMA_L2)[0] == [orc.FMT_INT8]


def test_outlier_ratio_matches_oracle(L, orc):
    """dmpq_outlier_ratio (host-pure, P:241 R = max|X| / mean|X|) equals the oracle's ratio computed
    from the same tensor, and is 1 for an all-zero input."""
    from paper_2603_18742_b200 import dmpq
    rng = np.random.default_rng(5)
    for trial in range(50):
        x = (rng.standard_normal(777) * rng.choice([1.0, 40.0], size=777, p=[0.99, 0.01])).astype(np.float32)
        import torch
        b = torch.from_numpy(x).to(torch.bfloat16)
        bits = b.view(torch.int16).numpy().view(np.uint16)
        xf = np.abs(b.float().numpy().astype(np.float64))
        got = dmpq.dmpq_outlier_ratio(float(xf.max()), float(xf.sum()), x.size)
        assert got == pytest.approx(orc.outlier_ratio(bits), rel=1e-12)
    assert dmpq.dmpq_outlier_ratio(0.0, 0.0, 100) == 1.0
