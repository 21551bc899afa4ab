"""GPU parity of every hot-path kernel against the CPU oracle, through the C ABI.

Bars (north_star): codes, scales, INT8 int32 accumulators, INT8
GEMM fp32 outputs and TDC deltas bit-exact; NVFP4 GEMM fp32 outputs within
relative L2 1e-5 of the oracle's fp64 accumulation over identical codes; FP64
statistics within 1e-9 relative.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2603_18742_b200 import synth  # noqa: E402


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_18742_b200 import build, dmpq
    build.build()
    return dmpq


def _u16(t):
    return synth.bits(t)


def rel_l2(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


QUANT_SHAPES = [(1, 64), (7, 128), (37, 512), (300, 1920), (129, 3072), (3, 7680), (130, 12288)]


@pytest.mark.parametrize("m,k", QUANT_SHAPES)
def test_quantize_nvfp4_bit_exact(D, orc, m, k):
    x = synth.dit_activation(m, k, seed=m * 7 + k)
    xd = x.cuda()
    amax_ref = orc.amax_bf16(_u16(x))
    g = torch.tensor([orc.global_scale(amax_ref, 1344.0)], device="cuda")
    a = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g)
    a.sf.fill_(0xAB)  # poison: padding rows must be zeroed by the kernel
    amax = torch.zeros(1, device="cuda")
    D.dmpq_quantize_act(xd, out_fp4=a, amax_out=amax)
    torch.cuda.synchronize()
    codes_ref, sf_ref = orc.nvfp4_quantize(_u16(x), float(g.item()))
    assert amax.item() == amax_ref
    assert np.array_equal(a.codes.cpu().numpy(), codes_ref)
    sf_dev = a.sf.cpu().numpy()
    assert np.array_equal(orc.sf_unswizzle(sf_dev, m, k), sf_ref)
    assert np.array_equal(sf_dev, orc.sf_swizzle(sf_ref, m, k)), "padding scales must be zero"


@pytest.mark.parametrize("m,k", QUANT_SHAPES)
def test_quantize_int8_bit_exact(D, orc, m, k):
    x = synth.ffn2_activation(m, k, seed=m + k)
    a = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    D.dmpq_quantize_act(x.cuda(), out_i8=a)
    torch.cuda.synchronize()
    codes_ref, s_ref = orc.int8_quantize(_u16(x))
    assert np.array_equal(a.codes.cpu().numpy(), codes_ref)
    assert np.array_equal(a.row_scale.cpu().numpy(), s_ref)


@pytest.mark.parametrize("k", [64, 128, 1920])
def test_quantize_adversarial_rows(D, orc, k):
    """Zero / signed-zero / constant / tiny / huge rows, E4M3-subnormal block scales,
    saturating blocks (g far below amax/1344) and the R4 reciprocal tie vector."""
    x = synth.adversarial_rows(k)
    m = x.shape[0]
    # g = 1e-30 / 1e30 are outside the fast block-scale path's guard (IEEE fallback)
    for g_val in (1.0, orc.global_scale(orc.amax_bf16(_u16(x)), 1344.0), 1e-3, 1e-30, 1e30):
        g = torch.tensor([g_val], dtype=torch.float32, device="cuda")
        a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g)
        a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
        D.dmpq_quantize_act(x.cuda(), out_i8=a8, out_fp4=a4)
        torch.cuda.synchronize()
        c_ref, s_ref = orc.nvfp4_quantize(_u16(x), float(g.item()))
        assert np.array_equal(a4.codes.cpu().numpy(), c_ref)
        assert np.array_equal(orc.sf_unswizzle(a4.sf.cpu().numpy(), m, k), s_ref)
        i_ref, is_ref = orc.int8_quantize(_u16(x))
        assert np.array_equal(a8.codes.cpu().numpy(), i_ref)
        assert np.array_equal(a8.row_scale.cpu().numpy(), is_ref)


def test_device_cvt_matches_oracle_sweep(D, orc):
    """The device E2M1/E4M3 conversions (via the quantizer with g = 1 and a unit
    block scale) agree with the oracle's exhaustive nearest search on a dense
    sweep of bf16 values around every E2M1 midpoint."""
    k = 1024
    vals = []
    mags = [0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0]
    for i in range(7):
        mid = (mags[i] + mags[i + 1]) / 2
        c = torch.tensor([mid], dtype=torch.bfloat16).view(torch.int16).item()
        for d in range(-40, 41):
            vals.append(c + d)
    v = torch.tensor(vals, dtype=torch.int16).view(torch.bfloat16).float()
    v = torch.cat([v, -v])
    n = (v.numel() + 14) // 15
    rows = torch.zeros(n * 15)
    rows[: v.numel()] = v
    rows = rows.view(n, 15)
    blocks = torch.cat([torch.full((n, 1), 6.0), rows], dim=1)  # block max 6 -> scale exactly 1 (E4M3 0x38)
    x = blocks.reshape(-1)
    x = torch.cat([x, torch.zeros((-x.numel()) % k)]).view(-1, k).to(torch.bfloat16)
    m = x.shape[0]
    g = torch.ones(1, device="cuda")
    a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g)
    D.dmpq_quantize_act(x.cuda(), out_fp4=a4)
    torch.cuda.synchronize()
    c_ref, s_ref = orc.nvfp4_quantize(_u16(x), 1.0)
    assert np.array_equal(a4.codes.cpu().numpy(), c_ref)


@pytest.mark.parametrize("n,k", [(32, 64), (256, 128), (512, 1920), (1920, 256)])
def test_pack_weights_bit_exact(D, orc, n, k):
    w, b = synth.linear_weight(n, k, seed=n + k)
    pw = D.dmpq_pack_weights(w.cuda(), b)
    torch.cuda.synchronize()
    ref = orc.pack_weights(_u16(w))
    assert pw.fp4_g.item() == ref["fp4_g"]
    assert np.array_equal(pw.fp4_codes.cpu().numpy(), ref["fp4_codes"])
    assert np.array_equal(orc.sf_unswizzle(pw.fp4_sf.cpu().numpy(), n, k), ref["fp4_sf"])
    assert np.array_equal(pw.i8_codes.cpu().numpy(), ref["i8_codes"])
    assert np.array_equal(pw.i8_scale.cpu().numpy(), ref["i8_scale"])


GEMM_SHAPES = [(1, 32, 64), (100, 128, 128), (129, 256, 512), (300, 512, 1920), (257, 1920, 256), (64, 96, 3072)]


@pytest.mark.parametrize("m,n,k", GEMM_SHAPES)
def test_gemm_int8_bit_exact(D, orc, m, n, k):
    x = synth.dit_activation(m, k, seed=3 * m + k)
    w, b = synth.linear_weight(n, k, seed=n * 3 + k)
    pw = D.dmpq_pack_weights(w.cuda(), b)
    a = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    D.dmpq_quantize_act(x.cuda(), out_i8=a)
    y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    y32 = torch.empty(m, n, dtype=torch.float32, device="cuda")
    acc = torch.empty(m, n, dtype=torch.int32, device="cuda")
    D.dmpq_gemm(a, pw, Y=y, Y32=y32, acc=acc)
    torch.cuda.synchronize()
    acc_ref, y_ref = orc.gemm_int8(a.codes.cpu().numpy(), a.row_scale.cpu().numpy(), pw.i8_codes.cpu().numpy(),
                                   pw.i8_scale.cpu().numpy(), b.numpy())
    assert np.array_equal(acc.cpu().numpy(), acc_ref)
    assert np.array_equal(y32.cpu().numpy(), y_ref)
    assert torch.equal(y.cpu(), torch.from_numpy(y_ref).to(torch.bfloat16))


@pytest.mark.parametrize("fmt,m,n,k", [(0, 300, 512, 256), (1, 300, 512, 256), (0, 1029, 1920, 512),
                                       (1, 1029, 1920, 512), (0, 4133, 3072, 128), (1, 4133, 3072, 128)])
def test_gemm_gated_residual(D, orc, fmt, m, n, k):
    """Gated-residual epilogue y = fma(gate, y, residual): the TMA-staged residual (bf16 output
    path, chunks requested a tile ahead, many tiles per CTA) equals the lane-per-row residual
    path (FP32-only output) bit for bit, and the bf16 output is the RNE of the FP32 one; INT8
    against the oracle's exact epilogue within the last FP32 rounding of the fma."""
    x = synth.dit_activation(m, k, seed=m + 2 * k)
    w, b = synth.linear_weight(n, k, seed=n + 3 * k)
    pw = D.dmpq_pack_weights(w.cuda(), b)
    g = torch.tensor([0.01], device="cuda")
    a = D.QuantAct.empty(fmt, m, k, "cuda", g=g if fmt == 1 else None)
    D.dmpq_quantize_act(x.cuda(), out_fp4=a if fmt == 1 else None, out_i8=a if fmt == 0 else None)
    res = synth.dit_activation(m, n, seed=m + 7, outlier_frac=0, tail_frac=0).cuda()
    gate = (0.05 * torch.rand(n, generator=torch.Generator().manual_seed(n))).cuda()
    y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    y32_tma = torch.empty(m, n, dtype=torch.float32, device="cuda")
    y32_lane = torch.empty(m, n, dtype=torch.float32, device="cuda")
    D.dmpq_gemm(a, pw, Y=y, Y32=y32_tma, residual=res, gate=gate)
    D.dmpq_gemm(a, pw, Y32=y32_lane, residual=res, gate=gate)
    torch.cuda.synchronize()
    assert torch.equal(y32_tma.cpu(), y32_lane.cpu())
    assert torch.equal(y.cpu(), y32_tma.cpu().to(torch.bfloat16))
    gate64 = gate.cpu().numpy().astype(np.float64)[None, :]
    res64 = res.cpu().float().numpy().astype(np.float64)
    got = y32_tma.cpu().numpy().astype(np.float64)
    if fmt == 0:
        _, y_lin = orc.gemm_int8(a.codes.cpu().numpy(), a.row_scale.cpu().numpy(), pw.i8_codes.cpu().numpy(),
                                 pw.i8_scale.cpu().numpy(), b.numpy())
        ref = gate64 * y_lin.astype(np.float64) + res64
        assert np.all(np.abs(got - ref) <= np.abs(ref) * 2.0 ** -23 + 1e-30)
    else:
        # NVFP4: the plain GEMM's fp32 output is within rel-L2 1e-5 of the oracle's fp64 accumulation
        # over the same codes, and the gated-residual output is fma(gate, y, res) of exactly that y
        # (one fp32 rounding of the exact value)
        y_plain = torch.empty(m, n, dtype=torch.float32, device="cuda")
        D.dmpq_gemm(a, pw, Y32=y_plain)
        torch.cuda.synchronize()
        y64 = orc.gemm_nvfp4(a.codes.cpu().numpy(), orc.sf_unswizzle(a.sf.cpu().numpy(), m, k), g.item(),
                             pw.fp4_codes.cpu().numpy(), orc.sf_unswizzle(pw.fp4_sf.cpu().numpy(), n, k),
                             pw.fp4_g.item(), b.numpy())
        yp = y_plain.cpu().numpy().astype(np.float64)
        assert rel_l2(yp, y64) <= 1e-5
        ref = gate64 * yp + res64
        assert np.all(np.abs(got - ref) <= np.abs(ref) * 2.0 ** -23 + 1e-30)
        assert rel_l2(got - res64, gate64 * y64) <= 1e-5


@pytest.mark.parametrize("fmt,m,k,had", [(0, 300, 256, False), (1, 300, 256, False), (1, 1029, 512, True),
                                        (0, 1029, 512, True), (2, 257, 128, False)])
def test_gemm_concatenated_layers(D, orc, fmt, m, k, had):
    """Q, K, V packed side by side (dmpq_concat_weights: per-column NVFP4 g_w): one GEMM gives
    the three separate GEMMs' outputs bit for bit; the per-layer views pack what the inputs did."""
    ns = (384, 256, 512)
    packs, ws = [], []
    for j, n in enumerate(ns):
        w, b = synth.linear_weight(n, k, seed=40 + j)
        ws.append(w)
        packs.append(D.dmpq_pack_weights(w.cuda(), b, hadamard=had, keep_bf16=(fmt == 2)))
    ref = [(p.fp4_codes.clone(), p.fp4_sf.clone(), p.fp4_g.clone(), p.i8_codes.clone(), p.i8_scale.clone())
           for p in packs]
    assert len({float(p.fp4_g.item()) for p in packs}) == 3   # distinct per-layer scales
    cat, views = D.dmpq_concat_weights(packs)
    for v, r in zip(views, ref):
        for a_, b_ in zip((v.fp4_codes, v.fp4_sf, v.fp4_g, v.i8_codes, v.i8_scale), r):
            assert torch.equal(a_, b_)
    x = synth.dit_activation(m, k, seed=m + k)
    g = torch.tensor([0.01], device="cuda")
    if fmt == 2:
        a = D.QuantAct.bf16(x.cuda())
    else:
        a = D.QuantAct.empty(fmt, m, k, "cuda", g=g if fmt == 1 else None)
        D.dmpq_quantize_act(x.cuda(), out_fp4=a if fmt == 1 else None, out_i8=a if fmt == 0 else None, hadamard=had)
    y_cat = torch.empty(m, sum(ns), dtype=torch.bfloat16, device="cuda")
    y32_cat = torch.empty(m, sum(ns), dtype=torch.float32, device="cuda")
    D.dmpq_gemm(a, cat, Y=y_cat, Y32=y32_cat)
    c0 = 0
    for v, n in zip(views, ns):
        y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
        y32 = torch.empty(m, n, dtype=torch.float32, device="cuda")
        D.dmpq_gemm(a, v, Y=y, Y32=y32)
        torch.cuda.synchronize()
        assert torch.equal(y32_cat[:, c0:c0 + n].cpu(), y32.cpu())
        assert torch.equal(y_cat[:, c0:c0 + n].cpu(), y.cpu())
        c0 += n


@pytest.mark.parametrize("m,n,k", GEMM_SHAPES)
def test_gemm_nvfp4_rel_l2(D, orc, m, n, k):
    x = synth.dit_activation(m, k, seed=5 * m + k)
    w, b = synth.linear_weight(n, k, seed=n * 5 + k)
    pw = D.dmpq_pack_weights(w.cuda(), b)
    g = torch.tensor([orc.global_scale(orc.amax_bf16(_u16(x)), 2688.0)], device="cuda")
    a = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g)
    D.dmpq_quantize_act(x.cuda(), out_fp4=a)
    y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    y32 = torch.empty(m, n, dtype=torch.float32, device="cuda")
    D.dmpq_gemm(a, pw, Y=y, Y32=y32)
    torch.cuda.synchronize()
    ref = orc.gemm_nvfp4(a.codes.cpu().numpy(), orc.sf_unswizzle(a.sf.cpu().numpy(), m, k), g.item(),
                         pw.fp4_codes.cpu().numpy(), orc.sf_unswizzle(pw.fp4_sf.cpu().numpy(), n, k),
                         pw.fp4_g.item(), b.numpy())
    err = rel_l2(y32.cpu().numpy(), ref)
    assert err <= 1e-5, err
    assert torch.equal(y.cpu(), y32.cpu().to(torch.bfloat16))


@pytest.mark.parametrize("fmt,m,n,k", [(0, 300, 512, 256), (1, 300, 512, 256), (0, 1029, 1920, 512),
                                       (1, 1029, 1920, 512), (2, 257, 384, 128), (1, 1, 256, 128)])
def test_gemm_fused_tdc_refresh(D, orc, fmt, m, n, k):
    """TDC refresh fused into the gated-residual GEMM epilogue (DMPQ_EP_TDC_REFRESH, SURVEY
    NEXT-2): Y equals the unfused GEMM's Y, Delta_new = bf16(Y - X_in) bit-exact, the seven
    statistics within tdc_step's bounds of the oracle, deterministic run to run."""
    x = synth.dit_activation(max(m, 1), k, seed=m + k + 5)[:m]
    w, b = synth.linear_weight(n, k, seed=n + 7)
    pw = D.dmpq_pack_weights(w.cuda(), b, keep_bf16=(fmt == 2))
    g = torch.tensor([0.01], device="cuda")
    if fmt == 2:
        a = D.QuantAct.bf16(x.cuda())
    else:
        a = D.QuantAct.empty(fmt, m, k, "cuda", g=g if fmt == 1 else None)
        D.dmpq_quantize_act(x.cuda(), out_fp4=a if fmt == 1 else None, out_i8=a if fmt == 0 else None)
    act = lambda s_: synth.dit_activation(max(m, 1), n, seed=s_, outlier_frac=0, tail_frac=0)[:m]
    res, xin = act(m + 11).cuda(), act(m + 12).cuda()
    dp = (0.05 * act(m + 13).float()).to(torch.bfloat16)
    gate = (0.01 * torch.rand(n, generator=torch.Generator().manual_seed(n))).cuda()
    y_ref = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    D.dmpq_gemm(a, pw, Y=y_ref, residual=res, gate=gate)
    ws = torch.zeros(D.dmpq_gemm_tdc_workspace_bytes(), dtype=torch.uint8, device="cuda")
    outs = []
    for _ in range(2):
        y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
        delta = dp.cuda().clone()
        stats = torch.full((7,), -1.0, dtype=torch.float64, device="cuda")
        D.dmpq_gemm(a, pw, Y=y, residual=res, gate=gate, tdc_x_in=xin, tdc_delta=delta, tdc_stats=stats,
                    tdc_workspace=ws)
        torch.cuda.synchronize()
        outs.append((y.cpu(), delta.cpu(), stats.cpu()))
    y, delta, stats = outs[0]
    assert torch.equal(y, y_ref.cpu())
    dn_ref, st_ref = orc.block_stats(_u16(xin.cpu()), _u16(y), _u16(dp))
    assert np.array_equal(synth.bits(delta), dn_ref)
    st = stats.numpy()
    np.testing.assert_allclose(st[:4], st_ref[:4], rtol=4.2e-7, atol=0)
    np.testing.assert_allclose(st[4:], st_ref[4:], rtol=1e-12, atol=1e-300)
    assert torch.equal(outs[1][1], delta) and torch.equal(outs[1][2], stats)


@pytest.mark.parametrize("m,h", [(1, 8), (256, 128), (1000, 1920), (777, 3072)])
def test_tdc_refresh_and_skip(D, orc, m, h):
    xi = synth.dit_activation(m, h, seed=m + 1, outlier_frac=0, tail_frac=0)
    xo = (xi.float() + 0.05 * synth.dit_activation(m, h, seed=m + 2, outlier_frac=0, tail_frac=0).float()).to(torch.bfloat16)
    dp = (0.05 * synth.dit_activation(m, h, seed=m + 3, outlier_frac=0, tail_frac=0).float()).to(torch.bfloat16)
    delta = dp.cuda().clone()
    stats = torch.zeros(7, dtype=torch.float64, device="cuda")
    ws = torch.zeros(D.tdc_workspace_bytes(m, h), dtype=torch.uint8, device="cuda")
    D.tdc_step(1, xi.cuda(), xo.cuda(), delta, stats, ws)
    torch.cuda.synchronize()
    dn_ref, st_ref = orc.block_stats(_u16(xi), _u16(xo), _u16(dp))
    assert np.array_equal(synth.bits(delta.cpu()), dn_ref)
    # Gamma/L2 sums: FP32 per 8-element vector (<= 7 roundings, 4.2e-7 relative of
    # the sum of |terms|, all terms non-negative); cosine sums: FP64 per element.
    st = stats.cpu().numpy()
    np.testing.assert_allclose(st[:4], st_ref[:4], rtol=4.2e-7, atol=0)
    np.testing.assert_allclose(st[4:], st_ref[4:], rtol=1e-12, atol=1e-300)
    # determinism: a second refresh over identical inputs gives identical bits
    delta2 = dp.cuda().clone()
    stats2 = torch.zeros(7, dtype=torch.float64, device="cuda")
    D.tdc_step(1, xi.cuda(), xo.cuda(), delta2, stats2, ws)
    torch.cuda.synchronize()
    assert torch.equal(stats.cpu(), stats2.cpu())
    # SKIP, in place
    x = xi.cuda().clone()
    D.tdc_step(0, x, x, delta)
    torch.cuda.synchronize()
    assert np.array_equal(synth.bits(x.cpu()), orc.tdc_skip(_u16(xi), dn_ref))


@pytest.mark.parametrize("m,h", [(1, 64), (256, 128), (1000, 1920), (777, 3072)])
def test_tdc_nvfp4_cache(D, orc, m, h):
    """NVFP4-compressed delta cache (R16): bootstrap amax, two refreshes (the second
    against the first's compressed cache, delayed scale), skip (also in place): codes,
    scales, amax, cache scale and outputs bit-exact; statistics as the bf16 cache path."""
    act = lambda s_: synth.dit_activation(m, h, seed=s_, outlier_frac=0, tail_frac=0)
    xi1 = act(m + 1)
    xo1 = (xi1.float() + 0.05 * act(m + 2).float()).to(torch.bfloat16)
    xi2 = act(m + 3)
    xo2 = (xi2.float() + 0.04 * act(m + 4).float()).to(torch.bfloat16)
    cache = D.DeltaCacheNvfp4(m, h, "cuda")
    ws = torch.zeros(D.tdc_workspace_bytes(m, h), dtype=torch.uint8, device="cuda")
    am0 = torch.zeros(1, device="cuda")
    D.tdc_delta_amax(xi1.cuda(), xo1.cuda(), am0)
    torch.cuda.synchronize()
    d1 = xo1.float().numpy() - xi1.float().numpy()
    assert am0.item() == float(np.abs(d1).max())
    g1 = torch.tensor([orc.global_scale(am0.item(), 1344.0)], device="cuda")
    zc, zs = np.zeros((m, h // 2), np.uint8), np.zeros((m, h // 16), np.uint8)
    prev = (zc, zs, 0.0)
    for (xi, xo, g) in ((xi1, xo1, g1), (xi2, xo2, None)):
        if g is None:   # delayed policy: the previous refresh's amax
            g = torch.tensor([orc.global_scale(am.item(), 1344.0)], device="cuda")
        am = torch.zeros(1, device="cuda")
        stats = torch.zeros(7, dtype=torch.float64, device="cuda")
        D.tdc_step_nvfp4(1, xi.cuda(), xo.cuda(), cache, g_new=g, amax_out=am, stats_out=stats, workspace=ws)
        torch.cuda.synchronize()
        cn, sn, st_ref, am_ref = orc.block_stats_nvfp4(_u16(xi), _u16(xo), prev[0], prev[1], prev[2], g.item())
        assert np.array_equal(cache.codes.cpu().numpy(), cn)
        assert np.array_equal(cache.sf.cpu().numpy(), sn)
        assert cache.g.item() == g.item() and am.item() == am_ref
        st = stats.cpu().numpy()
        np.testing.assert_allclose(st[:4], st_ref[:4], rtol=4.2e-7, atol=0)
        np.testing.assert_allclose(st[4:], st_ref[4:], rtol=1e-12, atol=1e-300)
        prev = (cn, sn, g.item())
    xi3 = act(m + 5)
    out = torch.empty_like(xi3).cuda()
    D.tdc_step_nvfp4(0, xi3.cuda(), out, cache)
    x = xi3.cuda().clone()
    D.tdc_step_nvfp4(0, x, x, cache)
    torch.cuda.synchronize()
    ref = orc.tdc_skip_nvfp4(_u16(xi3), prev[0], prev[1], prev[2])
    assert np.array_equal(synth.bits(out.cpu()), ref)
    assert np.array_equal(synth.bits(x.cpu()), ref)


@pytest.mark.parametrize("m,k,ln", [(5, 128, False), (130, 3072, True), (37, 1920, False), (33, 12288, False),
                                    (19, 7680, True), (41, 640, True), (23, 9216, False), (3, 16384, True)])
def test_quantize_hadamard_bit_exact(D, orc, m, k, ln):
    """Online block Hadamard fused into the quantizer (R14): codes and scales
    equal the oracle's FP32 FHT followed by the FP32-input quantizers."""
    x = synth.dit_activation(m, k, seed=m + 3 * k)
    h = torch.empty(m, k, dtype=torch.bfloat16, device="cuda") if ln else None
    g = torch.tensor([0.01], device="cuda")
    a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g)
    a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    amax = torch.zeros(1, device="cuda")
    D.dmpq_quantize_act(x.cuda(), out_i8=a8, out_fp4=a4, amax_out=amax, layernorm=ln, h_out=h, hadamard=True)
    torch.cuda.synchronize()
    src = synth.bits(h.cpu()) if ln else synth.bits(x)
    y = orc.fht128(orc.bf16_to_f32(src).reshape(m, k))
    assert amax.item() == float(np.abs(y).max())
    c4, s4 = orc.nvfp4_quantize_f32(y, 0.01)
    assert np.array_equal(a4.codes.cpu().numpy(), c4)
    assert np.array_equal(orc.sf_unswizzle(a4.sf.cpu().numpy(), m, k), s4)
    c8, s8 = orc.int8_quantize_f32(y)
    assert np.array_equal(a8.codes.cpu().numpy(), c8)
    assert np.array_equal(a8.row_scale.cpu().numpy(), s8)


@pytest.mark.parametrize("k,ln,which", [(3072, False, "both"), (3072, True, "both"), (12288, False, "both"),
                                        (3072, True, "nvfp4"), (3072, True, "int8"), (12288, False, "int8")])
def test_quantize_hadamard_dense_rows(D, orc, k, ln, which):
    """Several thousand full rows through the Hadamard quantizer (both formats): enough
    elements that fl(y r) lands exactly on INT8 / E2M1 rounding ties many times, so a
    contracted multiply-add (one rounding instead of RNE(fl(y r))) cannot pass."""
    m = 2053   # ragged: not a multiple of the kernel's rows per CTA
    x = synth.dit_activation(m, k, seed=k + 17) if k == 3072 else synth.ffn2_activation(m, k, seed=k + 17)
    h = torch.empty(m, k, dtype=torch.bfloat16, device="cuda") if ln else None
    g = torch.tensor([0.004], device="cuda")
    a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g)
    a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    amax = torch.zeros(1, device="cuda")
    D.dmpq_quantize_act(x.cuda(), out_i8=a8 if which != "nvfp4" else None, out_fp4=a4 if which != "int8" else None,
                        amax_out=amax, layernorm=ln, h_out=h, hadamard=True)
    torch.cuda.synchronize()
    src = synth.bits(h.cpu()) if ln else synth.bits(x)
    y = orc.fht128(orc.bf16_to_f32(src).reshape(m, k))
    assert amax.item() == float(np.abs(y).max())
    if which != "nvfp4":
        c8, s8 = orc.int8_quantize_f32(y)
        assert np.array_equal(a8.row_scale.cpu().numpy(), s8)
        assert np.array_equal(a8.codes.cpu().numpy(), c8)
    if which != "int8":
        c4, s4 = orc.nvfp4_quantize_f32(y, 0.004)
        assert np.array_equal(orc.sf_unswizzle(a4.sf.cpu().numpy(), m, k), s4)
        assert np.array_equal(a4.codes.cpu().numpy(), c4)


@pytest.mark.parametrize("k", [128, 1920])
def test_quantize_hadamard_adversarial_rows(D, orc, k):
    """The Hadamard quantizer on the adversarial rows (zero, tiny, huge, constant rows,
    saturating and E4M3-subnormal blocks) with global scales inside and outside the fast
    block-scale path's guard range."""
    x = synth.adversarial_rows(k)
    m = x.shape[0]
    y = orc.fht128(orc.bf16_to_f32(synth.bits(x)).reshape(m, k))
    for g_val in (1.0, 1e-3, float(np.abs(y).max()) / 1344.0, 1e-30, 1e30):
        g = torch.tensor([g_val], dtype=torch.float32, device="cuda")
        a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g)
        a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
        D.dmpq_quantize_act(x.cuda(), out_i8=a8, out_fp4=a4, hadamard=True)
        torch.cuda.synchronize()
        c4, s4 = orc.nvfp4_quantize_f32(y, float(g.item()))
        assert np.array_equal(a4.codes.cpu().numpy(), c4)
        assert np.array_equal(orc.sf_unswizzle(a4.sf.cpu().numpy(), m, k), s4)
        c8, s8 = orc.int8_quantize_f32(y)
        assert np.array_equal(a8.codes.cpu().numpy(), c8)
        assert np.array_equal(a8.row_scale.cpu().numpy(), s8)


def test_fastmath_exhaustive(tmp_path):
    """The quantizers' guarded fast division / reciprocal (csrc/fastmath.cuh) equal
    __fdiv_rn / __frcp_rn on every float of their guard ranges (scripts/fastmath_check.cu)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    exe = str(tmp_path / "fmc")
    subprocess.check_call(["/usr/local/cuda/bin/nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "--fmad=false", "-o", exe, os.path.join(root, "scripts", "fastmath_check.cu")])
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr


@pytest.mark.parametrize("n,k", [(128, 128), (256, 1920)])
def test_pack_weights_hadamard_and_gemm(D, orc, n, k):
    """Rotated weights pack bit-exact; the rotated GEMM reproduces the unrotated layer
    (H orthogonal: (Hx).(Hw) = x.w) up to quantization."""
    w, b = synth.linear_weight(n, k, seed=n + 7 * k)
    pw = D.dmpq_pack_weights(w.cuda(), b, hadamard=True)
    torch.cuda.synchronize()
    ref = orc.pack_weights_hadamard(synth.bits(w))
    assert pw.fp4_g.item() == ref["fp4_g"]
    assert np.array_equal(pw.fp4_codes.cpu().numpy(), ref["fp4_codes"])
    assert np.array_equal(orc.sf_unswizzle(pw.fp4_sf.cpu().numpy(), n, k), ref["fp4_sf"])
    assert np.array_equal(pw.i8_codes.cpu().numpy(), ref["i8_codes"])
    assert np.array_equal(pw.i8_scale.cpu().numpy(), ref["i8_scale"])
    m = 96
    x = synth.dit_activation(m, k, seed=5)
    a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    D.dmpq_quantize_act(x.cuda(), out_i8=a8, hadamard=True)
    y = torch.empty(m, n, dtype=torch.float32, device="cuda")
    D.dmpq_gemm(a8, pw, Y32=y)
    torch.cuda.synchronize()
    exact = x.float().numpy().astype(np.float64) @ w.float().numpy().astype(np.float64).T + b.numpy()
    # the unrotated quantized layer on the same input, for comparison
    pw0 = D.dmpq_pack_weights(w.cuda(), b)
    a0 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    D.dmpq_quantize_act(x.cuda(), out_i8=a0)
    y0 = torch.empty(m, n, dtype=torch.float32, device="cuda")
    D.dmpq_gemm(a0, pw0, Y32=y0)
    torch.cuda.synchronize()
    err_rot = np.linalg.norm(y.cpu().numpy() - exact) / np.linalg.norm(exact)
    err_plain = np.linalg.norm(y0.cpu().numpy() - exact) / np.linalg.norm(exact)
    # transparent up to quantization (4-bit-derived weights): same error scale as the plain path
    assert err_rot < 0.25 and err_rot < 1.5 * err_plain, (err_rot, err_plain)


@pytest.mark.parametrize("m,n,k", [(1, 32, 64), (200, 256, 1920), (257, 512, 3072)])
def test_gemm_bf16_rel_l2(D, orc, m, n, k):
    """BF16 fallback GEMM of the PDR gate (kind::f16): rel-L2 <= 1e-5 vs fp64."""
    x = synth.dit_activation(m, k, seed=9 * m + k)
    w, b = synth.linear_weight(n, k, seed=n + 11 * k)
    pw = D.dmpq_pack_weights(w.cuda(), b, keep_bf16=True)
    a = D.QuantAct.bf16(x.cuda())
    y32 = torch.empty(m, n, dtype=torch.float32, device="cuda")
    y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    D.dmpq_gemm(a, pw, Y=y, Y32=y32)
    torch.cuda.synchronize()
    ref = orc.gemm_bf16(synth.bits(x), synth.bits(w), b.numpy())
    assert rel_l2(y32.cpu().numpy(), ref) <= 1e-5
    assert torch.equal(y.cpu(), y32.cpu().to(torch.bfloat16))


@pytest.mark.parametrize("m,k,had", [(300, 1920, False), (129, 3072, True), (5, 12288, False)])
def test_pdr_statistics(D, orc, m, k, had):
    """Per-row sum|x| (FP32, fixed order: within K * 2^-24 of the exact sum) and max|x|
    of the layer input (exact), and the FP64 fixed-order reduction."""
    x = synth.dit_activation(m, k, seed=m + k)
    a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    rs = torch.zeros(1, m, dtype=torch.float32, device="cuda")
    ain = torch.zeros(1, device="cuda")
    D.dmpq_quantize_act(x.cuda(), out_i8=a8, hadamard=had, row_abs_sum=rs[0], amax_in=ain)
    tot = torch.zeros(1, dtype=torch.float64, device="cuda")
    D.dmpq_outlier_reduce(rs, tot)
    torch.cuda.synchronize()
    xf = np.abs(x.float().numpy().astype(np.float64))
    exact = xf.sum(axis=1)
    np.testing.assert_allclose(rs[0].cpu().numpy(), exact, rtol=k * 2.0 ** -24)
    assert ain.item() == float(xf.max())
    assert tot.item() == pytest.approx(float(rs[0].cpu().numpy().astype(np.float64).sum()), rel=1e-12)
    r_gpu = ain.item() / (tot.item() / (m * k))
    assert r_gpu == pytest.approx(orc.outlier_ratio(synth.bits(x)), rel=1e-5)


@pytest.mark.parametrize("k", [3072, 12288])
@pytest.mark.parametrize("which", ["nvfp4", "int8", "both"])
def test_quantize_hadamard_layernorm_no_h(D, orc, k, which):
    """The bench's LayerNorm + Hadamard quantizer instantiations (no h output, output formats fixed
    at compile time: quant_had_kernel<LN, !PDR, !WH, FMT 1 / 2 / 3>): codes, scales, row scales and
    amax equal the oracle's FP32 FHT + quantizers applied to the LN rows of the h-writing variant."""
    m = 1029
    x = synth.dit_activation(m, k, seed=k + 31)
    xd = x.cuda()
    h = torch.empty(m, k, dtype=torch.bfloat16, device="cuda")
    a_h = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    D.dmpq_quantize_act(xd, out_i8=a_h, layernorm=True, h_out=h, hadamard=True)
    g = torch.tensor([0.004], device="cuda")
    a4 = D.QuantAct.empty(D.FMT_NVFP4, m, k, "cuda", g=g)
    a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    amax = torch.zeros(1, device="cuda")
    D.dmpq_quantize_act(xd, out_i8=a8 if which != "nvfp4" else None, out_fp4=a4 if which != "int8" else None,
                        amax_out=amax, layernorm=True, hadamard=True)
    torch.cuda.synchronize()
    y = orc.fht128(orc.bf16_to_f32(synth.bits(h.cpu())).reshape(m, k))
    assert amax.item() == float(np.abs(y).max())
    if which != "nvfp4":
        c8, s8 = orc.int8_quantize_f32(y)
        assert np.array_equal(a8.row_scale.cpu().numpy(), s8)
        assert np.array_equal(a8.codes.cpu().numpy(), c8)
    if which != "int8":
        c4, s4 = orc.nvfp4_quantize_f32(y, 0.004)
        assert np.array_equal(orc.sf_unswizzle(a4.sf.cpu().numpy(), m, k), s4)
        assert np.array_equal(a4.codes.cpu().numpy(), c4)


@pytest.mark.parametrize("had,overlap,extra", [(True, False, {}), (False, False, {}), (True, True, {}),
                                               (True, False, {"pdr": "current", "tau_outlier": 9.0}),
                                               (True, False, {"int8_cast": True, "int8_block": True}),
                                               (False, False, {"fuse_quant": True, "tau_gamma": [0.05] * 6})])
def test_graph_replay_equals_eager(D, had, overlap, extra):
    """The bench's headline pass replays one CUDA graph per (block, decision, formats) pattern.
    Six timesteps of a two-block stack replayed from graphs equal the same steps launched eagerly
    bit for bit: outputs of every step, delta caches, FP64 statistics, global scales, decisions;
    also with each block's TDC refresh overlapped with the next block on a side stream."""
    from paper_2603_18742_b200.block import DiTStack
    M, H, F, T = 1000, 128, 512, 6
    A, B = synth.trajectory_basis(M, H, seed=5)
    xs = [synth.trajectory_input(A, B, t, 50).cuda() for t in range(T)]
    runs = []
    for graphs in (False, True):
        stack = DiTStack(3 if overlap else 2, H, F, M, "cuda", seed=4, gate_scales=[0.008, 0.012, 0.006][:3 if overlap else 2],
                         hadamard=had, tdc_cfg=(0.001, 0.02, 2), overlap_refresh=overlap, **extra)
        stack.use_graphs = graphs
        outs, stats = [], []
        for t in range(T):
            outs.append(stack.step(xs[t], t).clone())
            stats.append(stack.end_step(t).copy())
        torch.cuda.synchronize()
        runs.append(dict(outs=[o.cpu() for o in outs], stats=stats, delta=[d.cpu() for d in stack.delta],
                         g=stack.g_table.cpu(), dec=[r.decisions for r in stack.records],
                         fmts=[r.fmts for r in stack.records], graphs=sum(len(g) for g in stack.graphs)))
    e, g = runs
    assert g["graphs"] > 0 and e["graphs"] == 0
    assert e["dec"] == g["dec"] and e["fmts"] == g["fmts"]
    assert any(d == 1 for ds in e["dec"] for d in ds), "the trajectory should skip at least once"
    assert {f for fs in e["fmts"] for ff in fs if ff for f in ff} >= ({0, 2} if extra.get("pdr") else {0, 1}), \
        "both formats should run"
    for a, b in zip(e["outs"], g["outs"]):
        assert torch.equal(a, b)
    for a, b in zip(e["stats"], g["stats"]):
        assert np.array_equal(a, b)
    for a, b in zip(e["delta"], g["delta"]):
        assert torch.equal(a, b)
    assert torch.equal(e["g"], g["g"])


@pytest.mark.parametrize("n,k,had", [(32, 64, False), (256, 1920, False), (384, 3072, True), (1920, 256, True)])
def test_cast_int8_bit_exact(D, orc, n, k, had):
    """On-the-fly NVFP4 -> INT8 weight cast (NEXT-4b): an NVFP4-only pack plus dmpq_cast_int8
    reproduces the pre-packed INT8 codes bit for bit (and the oracle's pack), and the INT8 GEMM
    through the cast equals the GEMM on resident codes."""
    w, b = synth.linear_weight(n, k, seed=n + 13 * k)
    w[3] = 0   # a zero row: r_w = 0, codes 0, s_w = 1
    full = D.dmpq_pack_weights(w.cuda(), b, hadamard=had)
    lean = D.dmpq_pack_weights(w.cuda(), b, hadamard=had, int8_resident=False)
    assert lean.i8_codes is None and lean.nbytes() < full.nbytes()
    scratch = torch.full((n * k + 64,), 77, dtype=torch.int8, device="cuda")
    cast = D.dmpq_cast_int8(lean, scratch)
    torch.cuda.synchronize()
    assert torch.equal(cast.i8_codes.cpu(), full.i8_codes.cpu())
    assert torch.equal(lean.i8_scale.cpu(), full.i8_scale.cpu())
    ref = orc.pack_weights_hadamard(synth.bits(w)) if had else orc.pack_weights(synth.bits(w))
    assert np.array_equal(cast.i8_codes.cpu().numpy(), ref["i8_codes"])
    m = 129
    x = synth.dit_activation(m, k, seed=k)
    a = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    D.dmpq_quantize_act(x.cuda(), out_i8=a, hadamard=had)
    y0 = torch.empty(m, n, dtype=torch.float32, device="cuda")
    y1 = torch.empty(m, n, dtype=torch.float32, device="cuda")
    D.dmpq_gemm(a, full, Y32=y0)
    D.dmpq_gemm(a, cast, Y32=y1)
    torch.cuda.synchronize()
    assert torch.equal(y0.cpu(), y1.cpu())


def test_cast_int8_concatenated(D, orc):
    """The cast of side-by-side Q | K | V packs (per-column g_w) equals each layer's own codes."""
    k = 256
    packs, fulls = [], []
    for j, n in enumerate((128, 256, 384)):
        w, b = synth.linear_weight(n, k, seed=70 + j)
        packs.append(D.dmpq_pack_weights(w.cuda(), b, int8_resident=False))
        fulls.append(D.dmpq_pack_weights(w.cuda(), b))
    cat, views = D.dmpq_concat_weights(packs)
    scratch = torch.empty(cat.n * k, dtype=torch.int8, device="cuda")
    c = D.dmpq_cast_int8(cat, scratch)
    torch.cuda.synchronize()
    assert torch.equal(c.i8_codes.cpu(), torch.cat([f.i8_codes for f in fulls]).cpu())


@pytest.mark.parametrize("m,k", [(300, 1920), (129, 3072), (5, 12288)])
def test_outlier_gate_current_input(D, orc, m, k):
    """The device-side PDR gate (R18): its FP64 sum equals dmpq_outlier_reduce's, and its
    decision equals R > tau for the oracle's outlier ratio of the same input, for thresholds just
    below and above R (strict inequality) and far from it; a predicated GEMM pair runs exactly one."""
    x = synth.dit_activation(m, k, seed=m * 3 + k)
    a8 = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda")
    rs = torch.zeros(1, m, dtype=torch.float32, device="cuda")
    ain = torch.zeros(1, device="cuda")
    D.dmpq_quantize_act(x.cuda(), out_i8=a8, hadamard=True, row_abs_sum=rs[0], amax_in=ain)
    tot = torch.zeros(1, dtype=torch.float64, device="cuda")
    D.dmpq_outlier_reduce(rs, tot)
    torch.cuda.synchronize()
    r_ref = orc.outlier_ratio(synth.bits(x))
    r_dev = D.dmpq_outlier_ratio(ain.item(), tot.item(), m * k)
    assert r_dev == pytest.approx(r_ref, rel=1e-5)
    for tau in (r_dev * (1 - 1e-9), r_dev * (1 + 1e-9), 1.0, 1e6, 25.0):
        flag = torch.full((1,), 7, dtype=torch.int32, device="cuda")
        s_out = torch.zeros(1, dtype=torch.float64, device="cuda")
        D.dmpq_outlier_gate(rs[0], ain, m * k, tau, flag, s_out)
        torch.cuda.synchronize()
        assert s_out.item() == tot.item()
        assert flag.item() == int(r_dev > tau), (tau, r_dev)
        if abs(r_ref - tau) > 1e-5 * tau:
            assert flag.item() == int(r_ref > tau)
    # predicated launches: exactly the GEMM whose run_if_value matches the flag writes its output
    w, b = synth.linear_weight(64, k, seed=3)
    pw = D.dmpq_pack_weights(w.cuda(), b, keep_bf16=True)
    flag = torch.ones(1, dtype=torch.int32, device="cuda")
    y_q = torch.full((m, 64), float("nan"), device="cuda")
    y_b = torch.full((m, 64), float("nan"), device="cuda")
    D.dmpq_gemm(a8, pw, Y32=y_q, run_if=flag, run_if_value=0)
    D.dmpq_gemm(D.QuantAct.bf16(x.cuda()), pw, Y32=y_b, run_if=flag, run_if_value=1)
    torch.cuda.synchronize()
    assert torch.isnan(y_q).all() and not torch.isnan(y_b).any()


@pytest.mark.parametrize("m,k,ln", [(5, 128, False), (1029, 3072, True), (300, 1920, False), (33, 12288, False)])
def test_quantize_int8_blocks_bit_exact(D, orc, m, k, ln):
    """Per-block symmetric INT8 over the 128-element Hadamard blocks (R17): codes and the
    [m, k/128] block scales bit-exact against the oracle on the FP32 FHT output (also with LN and
    the NVFP4 output in the same pass), adversarial rows included."""
    x = torch.cat([synth.dit_activation(m, k, seed=m + 5 * k), synth.adversarial_rows(k)])
    mm = x.shape[0]
    h = torch.empty(mm, k, dtype=torch.bfloat16, device="cuda") if ln else None
    g = torch.tensor([0.01], device="cuda")
    a4 = D.QuantAct.empty(D.FMT_NVFP4, mm, k, "cuda", g=g)
    for with_fp4 in (False, True):
        a8 = D.QuantAct.empty(D.FMT_INT8, mm, k, "cuda", scale_block=128)
        D.dmpq_quantize_act(x.cuda(), out_i8=a8, out_fp4=a4 if with_fp4 else None, layernorm=ln, h_out=h, hadamard=True)
        torch.cuda.synchronize()
        src = synth.bits(h.cpu()) if ln else synth.bits(x)
        y = orc.fht128(orc.bf16_to_f32(src).reshape(mm, k))
        c8, s8 = orc.int8_quantize_blocks_f32(y)
        assert np.array_equal(a8.row_scale.cpu().numpy(), s8)
        assert np.array_equal(a8.codes.cpu().numpy(), c8)
        if with_fp4:
            c4, s4 = orc.nvfp4_quantize_f32(y, 0.01)
            assert np.array_equal(a4.codes.cpu().numpy(), c4)


@pytest.mark.parametrize("m,n,k", [(1, 192, 128), (300, 384, 256), (257, 1920, 1920), (1029, 3072, 3072), (64, 96, 12288)])
def test_gemm_int8_blocks_rel_l2(D, orc, m, n, k):
    """Per-block INT8 GEMM (R17): exact integer partial per 128-K block, FP32 promotion with the block
    scale: fp32 output within rel-L2 1e-5 of the oracle's FP64 (exact per-block sums, FP64 scaling),
    bf16 output the RNE of it; bias, GELU and gated-residual glue as the other kinds."""
    x = synth.dit_activation(m, k, seed=7 * m + k)
    w, b = synth.linear_weight(n, k, seed=n + 9 * k)
    pw = D.dmpq_pack_weights(w.cuda(), b, hadamard=True)
    a = D.QuantAct.empty(D.FMT_INT8, m, k, "cuda", scale_block=128)
    D.dmpq_quantize_act(x.cuda(), out_i8=a, hadamard=True)
    y32 = torch.empty(m, n, dtype=torch.float32, device="cuda")
    y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    D.dmpq_gemm(a, pw, Y=y, Y32=y32)
    res = synth.dit_activation(m, n, seed=m + 1, outlier_frac=0, tail_frac=0).cuda()
    gate = (0.05 * torch.rand(n, generator=torch.Generator().manual_seed(n))).cuda()
    y32r = torch.empty(m, n, dtype=torch.float32, device="cuda")
    D.dmpq_gemm(a, pw, Y32=y32r, residual=res, gate=gate)
    torch.cuda.synchronize()
    ref = orc.gemm_int8_blocks(a.codes.cpu().numpy(), a.row_scale.cpu().numpy(), pw.i8_codes.cpu().numpy(),
                               pw.i8_scale.cpu().numpy(), b.numpy())
    assert rel_l2(y32.cpu().numpy(), ref) <= 1e-5
    assert torch.equal(y.cpu(), y32.cpu().to(torch.bfloat16))
    yp = y32.cpu().numpy().astype(np.float64)
    got = y32r.cpu().numpy().astype(np.float64)
    want = gate.cpu().numpy().astype(np.float64)[None, :] * yp + res.cpu().float().numpy().astype(np.float64)
    assert np.all(np.abs(got - want) <= np.abs(want) * 2.0 ** -23 + 1e-30)


@pytest.mark.parametrize("fmt,m,n,k,gelu", [(0, 300, 512, 256, True), (1, 300, 512, 256, True), (1, 1029, 1920, 512, True),
                                            (0, 129, 3072, 128, False), (1, 35, 768, 3072, True)])
def test_gemm_fused_nvfp4_quant(D, orc, fmt, m, n, k, gelu):
    """Producer-fused NVFP4 quantization in the GEMM epilogue (DMPQ_EP_QUANT_NVFP4, NEXT-2):
    the codes, swizzled scales (padding rows zeroed) and amax it writes equal the standalone
    quantizer's on the same GEMM's bf16 output, and the oracle's; without Y the codes are the same."""
    x = synth.dit_activation(m, k, seed=m + 11 * k)
    w, b = synth.linear_weight(n, k, seed=n + 13 * k)
    pw = D.dmpq_pack_weights(w.cuda(), b)
    g = torch.tensor([0.01], device="cuda")
    a = D.QuantAct.empty(fmt, m, k, "cuda", g=g if fmt == 1 else None)
    D.dmpq_quantize_act(x.cuda(), out_fp4=a if fmt == 1 else None, out_i8=a if fmt == 0 else None)
    gq = torch.tensor([0.003], device="cuda")
    q1 = D.QuantAct.empty(D.FMT_NVFP4, m, n, "cuda", g=gq)
    q1.sf.fill_(0xAB)
    am1 = torch.zeros(1, device="cuda")
    y = torch.empty(m, n, dtype=torch.bfloat16, device="cuda")
    D.dmpq_gemm(a, pw, Y=y, gelu=gelu, quant_out=q1, quant_amax=am1)
    q2 = D.QuantAct.empty(D.FMT_NVFP4, m, n, "cuda", g=gq)
    am2 = torch.zeros(1, device="cuda")
    D.dmpq_quantize_act(y, out_fp4=q2, amax_out=am2)
    q3 = D.QuantAct.empty(D.FMT_NVFP4, m, n, "cuda", g=gq)
    am3 = torch.zeros(1, device="cuda")
    D.dmpq_gemm(a, pw, gelu=gelu, quant_out=q3, quant_amax=am3)   # no bf16 output at all
    torch.cuda.synchronize()
    assert torch.equal(q1.codes, q2.codes) and torch.equal(q1.sf, q2.sf) and am1.item() == am2.item()
    assert torch.equal(q3.codes, q1.codes) and torch.equal(q3.sf, q1.sf) and am3.item() == am1.item()
    c, s_ = orc.nvfp4_quantize(synth.bits(y.cpu()), 0.003)
    assert np.array_equal(q1.codes.cpu().numpy(), c)
    assert np.array_equal(q1.sf.cpu().numpy(), orc.sf_swizzle(s_, m, n))
    assert am1.item() == orc.amax_bf16(synth.bits(y.cpu()))


def test_gemm_cluster4_equals_pairs(tmp_path):
    """The 4-CTA-cluster option (DMPQ_GEMM_CLUSTER=4: B quarters and SFB atoms shared by TMA multicast
    between two CTA pairs) gives the CTA-pair GEMMs' outputs bit for bit — same
    MMAs in the same K order, only the operand delivery differs (ragged M and N, plain / GELU / gated
    residual epilogues, both formats)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    outs = {}
    for c in ("2", "4"):
        f = str(tmp_path / f"cl{c}.npz")
        env = dict(os.environ, DMPQ_GEMM_CLUSTER=c)
        subprocess.run([sys.executable, os.path.join(root, "scripts", "gemm_cluster_check.py"), f], env=env, check=True,
                       timeout=600)
        outs[c] = np.load(f)
    assert sorted(outs["2"].files) == sorted(outs["4"].files) and len(outs["2"].files) == 18
    for key in outs["2"].files:
        assert np.array_equal(outs["2"][key], outs["4"][key]), key
