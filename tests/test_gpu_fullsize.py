"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times
(CogVideoX-5B layer shapes, M = 35,552 token rows), on sampled outputs the oracle
computes one by one: sampled rows spread over every 256-row tile band, including the
ragged last tile; properties that hold at any size (amax, statistics) in full."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

from paper_2603_18742_b200 import synth  # noqa: E402

M = 2 * 17776


@pytest.fixture(scope="module")
def D():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2603_18742_b200 import build, dmpq
    build.build()
    return dmpq


def sample_rows(m, n=12, seed=0):
    rng = np.random.default_rng(seed)
    rows = set(rng.integers(0, m, n).tolist()) | {0, 127, 128, 255, m - 1, m - 129, (m // 256) * 256}
    return sorted(r for r in rows if 0 <= r < m)


@pytest.mark.parametrize("n,k", [(3072, 3072), (12288, 3072), (3072, 12288)])
def test_fullsize_gemms_sampled(D, orc, n, k):
    x = synth.dit_activation(M, k, seed=k) if k == 3072 else synth.ffn2_activation(M, k, seed=k)
    xd = x.cuda()
    w, b = synth.linear_weight_device(n, k, seed=n + k, device="cuda")
    pw = D.dmpq_pack_weights(w, b)
    amax = torch.zeros(1, device="cuda")
    g = torch.zeros(1, device="cuda")
    a8 = D.QuantAct.empty(D.FMT_INT8, M, k, "cuda")
    D.dmpq_quantize_act(xd, out_i8=a8, amax_out=amax)
    D.dmpq_global_scale(amax, 1344.0, g)
    a4 = D.QuantAct.empty(D.FMT_NVFP4, M, k, "cuda", g=g)
    D.dmpq_quantize_act(xd, out_fp4=a4)
    y8 = torch.empty(M, n, dtype=torch.bfloat16, device="cuda")
    y4 = torch.empty(M, n, dtype=torch.bfloat16, device="cuda")
    D.dmpq_gemm(a8, pw, Y=y8)
    D.dmpq_gemm(a4, pw, Y=y4)
    torch.cuda.synchronize()
    xb = synth.bits(x)
    assert amax.item() == orc.amax_bf16(xb)
    assert g.item() == orc.global_scale(amax.item(), 1344.0)
    wb = synth.bits(w.cpu())
    pk = orc.pack_weights(wb)
    assert np.array_equal(pw.i8_codes.cpu().numpy(), pk["i8_codes"])
    assert pw.fp4_g.item() == pk["fp4_g"]
    bias = b.cpu().numpy()
    c8_all = a8.codes.cpu().numpy()
    s8_all = a8.row_scale.cpu().numpy()
    c4_all = a4.codes.cpu().numpy()
    sf4 = orc.sf_unswizzle(a4.sf.cpu().numpy(), M, k)
    for r in sample_rows(M):
        c8, s8 = orc.int8_quantize(xb[r:r + 1])
        assert np.array_equal(c8_all[r:r + 1], c8) and s8_all[r] == s8[0]
        c4, s4 = orc.nvfp4_quantize(xb[r:r + 1], g.item())
        assert np.array_equal(c4_all[r:r + 1], c4) and np.array_equal(sf4[r:r + 1], s4)
        _, yr8 = orc.gemm_int8(c8, s8, pk["i8_codes"], pk["i8_scale"], bias)
        assert torch.equal(y8[r:r + 1].cpu(), torch.from_numpy(yr8).to(torch.bfloat16)), r
        yr4 = orc.gemm_nvfp4(c4, s4, g.item(), pk["fp4_codes"], pk["fp4_sf"], pk["fp4_g"], bias)
        got = y4[r].float().cpu().numpy().astype(np.float64)
        # bf16 output of an fp32-accumulated GEMM: within bf16 rounding of the fp64 reference
        assert np.linalg.norm(got - yr4[0]) <= 4e-3 * np.linalg.norm(yr4[0]), r


def test_fullsize_tdc(D, orc):
    H = 3072
    xi = synth.dit_activation(M, H, seed=1, outlier_frac=0, tail_frac=0)
    xo = (xi.float() + 0.01 * synth.dit_activation(M, H, seed=2, outlier_frac=0, tail_frac=0).float()).to(torch.bfloat16)
    dp = (0.01 * synth.dit_activation(M, H, seed=3, outlier_frac=0, tail_frac=0).float()).to(torch.bfloat16)
    delta = dp.cuda()
    stats = torch.zeros(7, dtype=torch.float64, device="cuda")
    ws = torch.zeros(D.tdc_workspace_bytes(M, H), dtype=torch.uint8, device="cuda")
    D.tdc_step(1, xi.cuda(), xo.cuda(), delta, stats, ws)
    torch.cuda.synchronize()
    dn, st = orc.block_stats(synth.bits(xi), synth.bits(xo), synth.bits(dp))
    assert np.array_equal(synth.bits(delta.cpu()), dn)
    s = stats.cpu().numpy()
    np.testing.assert_allclose(s[:4], st[:4], rtol=4.2e-7)
    np.testing.assert_allclose(s[4:], st[4:], rtol=1e-12)


@pytest.mark.parametrize("n,k,ln", [(3072, 3072, True), (3072, 12288, False)])
def test_fullsize_hadamard_sampled(D, orc, n, k, ln):
    """The bench's default path at full size: LN (attention / FFN1 inputs) + online block
    Hadamard quantizer (both formats in one pass) against Hadamard-packed weights (R14)."""
    x = synth.dit_activation(M, k, seed=k + 1) if k == 3072 else synth.ffn2_activation(M, k, seed=k + 1)
    xd = x.cuda()
    w, b = synth.linear_weight_device(n, k, seed=n + k + 1, device="cuda")
    pw = D.dmpq_pack_weights(w, b, hadamard=True)
    h = torch.empty(M, k, dtype=torch.bfloat16, device="cuda") if ln else None
    g = torch.tensor([0.02], device="cuda")
    amax = torch.zeros(1, device="cuda")
    a8 = D.QuantAct.empty(D.FMT_INT8, M, k, "cuda")
    a4 = D.QuantAct.empty(D.FMT_NVFP4, M, k, "cuda", g=g)
    D.dmpq_quantize_act(xd, out_i8=a8, out_fp4=a4, amax_out=amax, layernorm=ln, h_out=h, hadamard=True)
    y8 = torch.empty(M, n, dtype=torch.bfloat16, device="cuda")
    y4 = torch.empty(M, n, dtype=torch.bfloat16, device="cuda")
    D.dmpq_gemm(a8, pw, Y=y8)
    D.dmpq_gemm(a4, pw, Y=y4)
    torch.cuda.synchronize()
    pk = orc.pack_weights_hadamard(synth.bits(w.cpu()))
    assert np.array_equal(pw.i8_codes.cpu().numpy(), pk["i8_codes"])
    assert np.array_equal(pw.i8_scale.cpu().numpy(), pk["i8_scale"])
    assert pw.fp4_g.item() == pk["fp4_g"]
    src = synth.bits(h.cpu()) if ln else synth.bits(x)
    bias = b.cpu().numpy()
    c8_all, s8_all = a8.codes.cpu().numpy(), a8.row_scale.cpu().numpy()
    c4_all, sf4 = a4.codes.cpu().numpy(), orc.sf_unswizzle(a4.sf.cpu().numpy(), M, k)
    for r in sample_rows(M, seed=1):
        y = orc.fht128(orc.bf16_to_f32(src[r:r + 1]).reshape(1, k))
        c8, s8 = orc.int8_quantize_f32(y)
        assert np.array_equal(c8_all[r:r + 1], c8) and s8_all[r] == s8[0], r
        c4, s4 = orc.nvfp4_quantize_f32(y, 0.02)
        assert np.array_equal(c4_all[r:r + 1], c4) and np.array_equal(sf4[r:r + 1], s4), r
        _, yr8 = orc.gemm_int8(c8, s8, pk["i8_codes"], pk["i8_scale"], bias)
        assert torch.equal(y8[r:r + 1].cpu(), torch.from_numpy(yr8).to(torch.bfloat16)), r
        yr4 = orc.gemm_nvfp4(c4, s4, 0.02, pk["fp4_codes"], pk["fp4_sf"], pk["fp4_g"], bias)
        got = y4[r].float().cpu().numpy().astype(np.float64)
        assert np.linalg.norm(got - yr4[0]) <= 4e-3 * np.linalg.norm(yr4[0]), r
    # the tensor amax is a property of every row: check it over all rows of the sample
    assert amax.item() >= float(np.abs(orc.fht128(orc.bf16_to_f32(src[:256]).reshape(256, k))).max())


def test_fullsize_tdc_nvfp4_cache(D, orc):
    """Compressed delta cache (R16) at full size: refresh against a compressed cache, skip."""
    H = 3072
    act = lambda s_: synth.dit_activation(M, H, seed=s_, outlier_frac=0, tail_frac=0)
    xi, xo = act(11), None
    xo = (xi.float() + 0.01 * act(12).float()).to(torch.bfloat16)
    rng = np.random.default_rng(5)
    cp = rng.integers(0, 256, size=(M, H // 2), dtype=np.uint8)
    sp = rng.integers(0x20, 0x38, size=(M, H // 16), dtype=np.uint8)   # E4M3 0.0078 .. 1.0
    cache = D.DeltaCacheNvfp4(M, H, "cuda")
    cache.codes.copy_(torch.from_numpy(cp))
    cache.sf.copy_(torch.from_numpy(sp))
    cache.g.fill_(0.01)
    g_new = torch.tensor([orc.global_scale(float((xo.float() - xi.float()).abs().max()), 1344.0)], device="cuda")
    am = torch.zeros(1, device="cuda")
    stats = torch.zeros(7, dtype=torch.float64, device="cuda")
    ws = torch.zeros(D.tdc_workspace_bytes(M, H), dtype=torch.uint8, device="cuda")
    D.tdc_step_nvfp4(1, xi.cuda(), xo.cuda(), cache, g_new=g_new, amax_out=am, stats_out=stats, workspace=ws)
    out = torch.empty(M, H, dtype=torch.bfloat16, device="cuda")
    D.tdc_step_nvfp4(0, xo.cuda(), out, cache)
    torch.cuda.synchronize()
    cn, sn, st, am_ref = orc.block_stats_nvfp4(synth.bits(xi), synth.bits(xo), cp, sp, 0.01, g_new.item())
    assert np.array_equal(cache.codes.cpu().numpy(), cn) and np.array_equal(cache.sf.cpu().numpy(), sn)
    assert am.item() == am_ref and cache.g.item() == g_new.item()
    s = stats.cpu().numpy()
    np.testing.assert_allclose(s[:4], st[:4], rtol=4.2e-7)
    np.testing.assert_allclose(s[4:], st[4:], rtol=1e-12)
    assert np.array_equal(synth.bits(out.cpu()), orc.tdc_skip_nvfp4(synth.bits(xo), cn, sn, g_new.item()))


@pytest.mark.parametrize("which", ["nvfp4", "int8", "both"])
def test_fullsize_layernorm_hadamard_no_h(D, orc, which):
    """The exact quantizer launches of the bench's attention / FFN1 inputs at full size: LN +
    Hadamard without the h output, formats fixed at compile time (quant_had_kernel<LN,!PDR,!WH,FMT>),
    sampled rows bit-exact against the oracle on the LN rows of the h-writing variant; the tensor
    amax over all rows."""
    k = 3072
    x = synth.dit_activation(M, k, seed=k + 2)
    xd = x.cuda()
    h = torch.empty(M, k, dtype=torch.bfloat16, device="cuda")
    a_h = D.QuantAct.empty(D.FMT_INT8, M, k, "cuda")
    D.dmpq_quantize_act(xd, out_i8=a_h, layernorm=True, h_out=h, hadamard=True)
    g = torch.tensor([0.02], device="cuda")
    a8 = D.QuantAct.empty(D.FMT_INT8, M, k, "cuda")
    a4 = D.QuantAct.empty(D.FMT_NVFP4, M, k, "cuda", g=g)
    amax = torch.zeros(1, device="cuda")
    D.dmpq_quantize_act(xd, out_i8=a8 if which != "nvfp4" else None, out_fp4=a4 if which != "int8" else None,
                        amax_out=amax, layernorm=True, hadamard=True)
    torch.cuda.synchronize()
    src = synth.bits(h.cpu())
    y_all = orc.fht128(orc.bf16_to_f32(src).reshape(M, k))
    assert amax.item() == float(np.abs(y_all).max())
    c8_all, s8_all = a8.codes.cpu().numpy(), a8.row_scale.cpu().numpy()
    c4_all, sf4 = a4.codes.cpu().numpy(), orc.sf_unswizzle(a4.sf.cpu().numpy(), M, k)
    for r in sample_rows(M, n=40, seed=2):
        y = y_all[r:r + 1]
        if which != "nvfp4":
            c8, s8 = orc.int8_quantize_f32(y)
            assert np.array_equal(c8_all[r:r + 1], c8) and s8_all[r] == s8[0], r
        if which != "int8":
            c4, s4 = orc.nvfp4_quantize_f32(y, 0.02)
            assert np.array_equal(c4_all[r:r + 1], c4) and np.array_equal(sf4[r:r + 1], s4), r


@pytest.mark.parametrize("fmt", [0, 1])
def test_fullsize_qkv_concat_sampled(D, orc, fmt):
    """The bench's most frequent GEMM: Q | K | V side by side (N = 9216, K = 3072, M = 35,552,
    Hadamard-packed, per-column NVFP4 g_w) on sampled rows against the oracle's GEMM with each
    layer's own packed weights and g_w (INT8 bit-exact, NVFP4 fp32 rel-L2 <= 1e-5)."""
    H = 3072
    packs, pks = [], []
    for j in range(3):
        w, b = synth.linear_weight_device(H, H, seed=900 + j, device="cuda")
        packs.append(D.dmpq_pack_weights(w, b, hadamard=True))
        pks.append((orc.pack_weights_hadamard(synth.bits(w.cpu())), b.cpu().numpy()))
    assert len({p.fp4_g.item() for p in packs}) == 3
    cat, _ = D.dmpq_concat_weights(packs)
    x = synth.dit_activation(M, H, seed=77)
    g = torch.tensor([0.02], device="cuda")
    a = D.QuantAct.empty(fmt, M, H, "cuda", g=g if fmt == 1 else None)
    D.dmpq_quantize_act(x.cuda(), out_fp4=a if fmt == 1 else None, out_i8=a if fmt == 0 else None, hadamard=True)
    y32 = torch.empty(M, 3 * H, dtype=torch.float32, device="cuda")
    y = torch.empty(M, 3 * H, dtype=torch.bfloat16, device="cuda")
    D.dmpq_gemm(a, cat, Y=y, Y32=y32)
    torch.cuda.synchronize()
    codes = a.codes.cpu().numpy()
    if fmt == 1:
        sfa = orc.sf_unswizzle(a.sf.cpu().numpy(), M, H)
    else:
        s8 = a.row_scale.cpu().numpy()
    rows = sample_rows(M, n=6, seed=3)
    for j, (pk, bias) in enumerate(pks):
        assert packs[j].fp4_g.item() == pk["fp4_g"]
        for r in rows:
            got = y32[r, j * H:(j + 1) * H].cpu().numpy()
            assert torch.equal(y[r, j * H:(j + 1) * H].cpu(), torch.from_numpy(got).to(torch.bfloat16))
            if fmt == 0:
                _, ref = orc.gemm_int8(codes[r:r + 1], s8[r:r + 1], pk["i8_codes"], pk["i8_scale"], bias)
                assert np.array_equal(got, ref[0]), (j, r)
            else:
                ref = orc.gemm_nvfp4(codes[r:r + 1], sfa[r:r + 1], 0.02, pk["fp4_codes"], pk["fp4_sf"], pk["fp4_g"],
                                     bias)[0]
                err = np.linalg.norm(got.astype(np.float64) - ref) / np.linalg.norm(ref)
                assert err <= 1e-5, (j, r, err)


@pytest.mark.parametrize("n,k,ln", [(1920, 1920, True), (1920, 7680, False)])
def test_fullsize_cogvideox2b_hadamard_sampled(D, orc, n, k, ln):
    """CogVideoX-2B layer shapes (BASELINE configs[2]: hidden 1920, FFN 7680; 15 / 60 Hadamard blocks per
    row, ragged against the quantizer's 8-thread row segments) at M = 35,552: LN + Hadamard quantizer
    and both GEMMs on sampled rows against the oracle."""
    x = synth.dit_activation(M, k, seed=k + 5) if k == 1920 else synth.ffn2_activation(M, k, seed=k + 5)
    xd = x.cuda()
    w, b = synth.linear_weight_device(n, k, seed=n + k + 5, device="cuda")
    pw = D.dmpq_pack_weights(w, b, hadamard=True)
    h = torch.empty(M, k, dtype=torch.bfloat16, device="cuda") if ln else None
    g = torch.tensor([0.02], device="cuda")
    a8 = D.QuantAct.empty(D.FMT_INT8, M, k, "cuda")
    a4 = D.QuantAct.empty(D.FMT_NVFP4, M, k, "cuda", g=g)
    D.dmpq_quantize_act(xd, out_i8=a8, out_fp4=a4, layernorm=ln, h_out=h, hadamard=True)
    y8 = torch.empty(M, n, dtype=torch.bfloat16, device="cuda")
    y4 = torch.empty(M, n, dtype=torch.bfloat16, device="cuda")
    D.dmpq_gemm(a8, pw, Y=y8)
    D.dmpq_gemm(a4, pw, Y=y4)
    torch.cuda.synchronize()
    pk = orc.pack_weights_hadamard(synth.bits(w.cpu()))
    assert np.array_equal(pw.i8_codes.cpu().numpy(), pk["i8_codes"])
    src = synth.bits(h.cpu()) if ln else synth.bits(x)
    bias = b.cpu().numpy()
    c8_all, s8_all = a8.codes.cpu().numpy(), a8.row_scale.cpu().numpy()
    c4_all, sf4 = a4.codes.cpu().numpy(), orc.sf_unswizzle(a4.sf.cpu().numpy(), M, k)
    for r in sample_rows(M, n=8, seed=4):
        y = orc.fht128(orc.bf16_to_f32(src[r:r + 1]).reshape(1, k))
        c8, s8 = orc.int8_quantize_f32(y)
        assert np.array_equal(c8_all[r:r + 1], c8) and s8_all[r] == s8[0], r
        c4, s4 = orc.nvfp4_quantize_f32(y, 0.02)
        assert np.array_equal(c4_all[r:r + 1], c4) and np.array_equal(sf4[r:r + 1], s4), r
        _, yr8 = orc.gemm_int8(c8, s8, pk["i8_codes"], pk["i8_scale"], bias)
        assert torch.equal(y8[r:r + 1].cpu(), torch.from_numpy(yr8).to(torch.bfloat16)), r
        yr4 = orc.gemm_nvfp4(c4, s4, 0.02, pk["fp4_codes"], pk["fp4_sf"], pk["fp4_g"], bias)
        got = y4[r].float().cpu().numpy().astype(np.float64)
        assert np.linalg.norm(got - yr4[0]) <= 4e-3 * np.linalg.norm(yr4[0]), r


def test_max_size_hunyuan_rows_sampled(D, orc):
    """The largest single-GPU row count of the workloads (BASELINE configs[4]: 119,056 tokens,
    hidden 3072) through the LN + Hadamard quantizer (both formats) and both GEMMs of the O shape:
    sampled rows (incl. the ragged last tile) against the oracle; the tensor amax over all rows."""
    Mh, k, n = 119056, 3072, 3072
    xd = synth.dit_activation_device(Mh, k, seed=12, device="cuda")
    w, b = synth.linear_weight_device(n, k, seed=13, device="cuda")
    pw = D.dmpq_pack_weights(w, b, hadamard=True)
    h = torch.empty(Mh, k, dtype=torch.bfloat16, device="cuda")
    g = torch.tensor([0.02], device="cuda")
    amax = torch.zeros(1, device="cuda")
    a8 = D.QuantAct.empty(D.FMT_INT8, Mh, k, "cuda")
    a4 = D.QuantAct.empty(D.FMT_NVFP4, Mh, k, "cuda", g=g)
    D.dmpq_quantize_act(xd, out_i8=a8, out_fp4=a4, amax_out=amax, layernorm=True, h_out=h, hadamard=True)
    y8 = torch.empty(Mh, n, dtype=torch.bfloat16, device="cuda")
    y4 = torch.empty(Mh, n, dtype=torch.bfloat16, device="cuda")
    D.dmpq_gemm(a8, pw, Y=y8)
    D.dmpq_gemm(a4, pw, Y=y4)
    torch.cuda.synchronize()
    pk = orc.pack_weights_hadamard(synth.bits(w.cpu()))
    bias = b.cpu().numpy()
    rows = sample_rows(Mh, n=8, seed=6)
    hb = synth.bits(h[rows].cpu())
    c8_all, s8_all = a8.codes[rows].cpu().numpy(), a8.row_scale[rows].cpu().numpy()
    c4_all = a4.codes[rows].cpu().numpy()
    sf4 = orc.sf_unswizzle(a4.sf.cpu().numpy(), Mh, k)[rows]
    ymax = 0.0
    for i, r in enumerate(rows):
        y = orc.fht128(orc.bf16_to_f32(hb[i:i + 1]).reshape(1, k))
        ymax = max(ymax, float(np.abs(y).max()))
        c8, s8 = orc.int8_quantize_f32(y)
        assert np.array_equal(c8_all[i:i + 1], c8) and s8_all[i] == s8[0], r
        c4, s4 = orc.nvfp4_quantize_f32(y, 0.02)
        assert np.array_equal(c4_all[i:i + 1], c4) and np.array_equal(sf4[i:i + 1], s4), r
        _, yr8 = orc.gemm_int8(c8, s8, pk["i8_codes"], pk["i8_scale"], bias)
        assert torch.equal(y8[r:r + 1].cpu(), torch.from_numpy(yr8).to(torch.bfloat16)), r
        yr4 = orc.gemm_nvfp4(c4, s4, 0.02, pk["fp4_codes"], pk["fp4_sf"], pk["fp4_g"], bias)
        got = y4[r].float().cpu().numpy().astype(np.float64)
        assert np.linalg.norm(got - yr4[0]) <= 4e-3 * np.linalg.norm(yr4[0]), r
    assert amax.item() >= ymax


@pytest.mark.parametrize("k,ln,which", [(12288, False, "int8"), (3072, False, "int8"), (3072, True, "int8"),
                                        (3072, False, "nvfp4"), (3072, True, "nvfp4")])
def test_fullsize_hadamard_dense_all_rows(D, orc, k, ln, which):
    """Every row, every code of the bench's Hadamard quantizer launches at full size (M = 35,552:
    15-60 row sets per CTA through the TMA ring), three launches on different inputs, against the
    oracle: a guard against rare shared-memory reuse races (round-2b: a TMA refill
    overtaking shared loads lost whole 128-blocks ~3 times in 10^4), which sampled rows would miss.
    LN variants: the h-writing launch gives the LN rows, the bench's launch (no h) the codes."""
    g = torch.tensor([0.02], device="cuda")
    for rep in range(3):
        xd = synth.dit_activation_device(M, k, 31 + rep, "cuda")
        if k != 3072:   # FFN2 input: GELU-tanh of an FFN1-like tensor (synth.ffn2_activation's recipe)
            xd = torch.nn.functional.gelu(xd.float(), approximate="tanh").to(torch.bfloat16)
        x = xd.cpu()
        h = None
        if ln:
            h = torch.empty(M, k, dtype=torch.bfloat16, device="cuda")
            D.dmpq_quantize_act(xd, out_i8=D.QuantAct.empty(D.FMT_INT8, M, k, "cuda"), layernorm=True, h_out=h,
                                hadamard=True)
        a = D.QuantAct.empty(D.FMT_INT8 if which == "int8" else D.FMT_NVFP4, M, k, "cuda",
                             g=g if which == "nvfp4" else None)
        D.dmpq_quantize_act(xd, out_i8=a if which == "int8" else None, out_fp4=a if which == "nvfp4" else None,
                            layernorm=ln, hadamard=True)
        torch.cuda.synchronize()
        y = orc.fht128(orc.bf16_to_f32(synth.bits(h.cpu() if ln else x)).reshape(M, k))
        if which == "int8":
            c8, s8 = orc.int8_quantize_f32(y)
            assert np.array_equal(a.row_scale.cpu().numpy(), s8), rep
            bad = np.argwhere(a.codes.cpu().numpy() != c8)
        else:
            c4, s4 = orc.nvfp4_quantize_f32(y, 0.02)
            assert np.array_equal(orc.sf_unswizzle(a.sf.cpu().numpy(), M, k), s4), rep
            bad = np.argwhere(a.codes.cpu().numpy() != c4)
        assert len(bad) == 0, f"launch {rep}: {len(bad)} codes differ, first at {bad[:4].tolist()}"
