"""Pins for the CPU oracle: checks against what the paper and the mathematics fix,
never against the oracle's own formula retyped.

Each pin is chosen so that a plausible mistake (dropped term, wrong sign/index,
transposed operand, wrong tie rule, wrong scale step) fails at least one test.
"""
import json
import math
import os
from fractions import Fraction

import numpy as np
import pytest
import torch

GOLDEN = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))


def bf16_bits(vals):
    """float values -> bf16 bit patterns via torch's RNE conversion (library routine)."""
    t = torch.tensor(np.asarray(vals, dtype=np.float32)).to(torch.bfloat16)
    return t.view(torch.int16).numpy().view(np.uint16).copy()


def round_f32(fr: Fraction) -> np.float32:
    """Correctly rounded (nearest-even) binary32 value of an exact rational."""
    f = np.float32(float(fr))
    best = f
    for c in (np.nextafter(f, np.float32(np.inf)), np.nextafter(f, np.float32(-np.inf))):
        dc, db = abs(Fraction(float(c)) - fr), abs(Fraction(float(best)) - fr)
        if dc < db or (dc == db and (int(np.float32(c).view(np.uint32)) & 1) == 0):
            best = c
    return np.float32(best)


def bf16_vals(bits):
    return torch.from_numpy(np.asarray(bits, dtype=np.uint16).view(np.int16)).view(torch.bfloat16).float().numpy()


# ---------------------------------------------------------------------------- formats

def test_e4m3_decode_matches_torch_all_codes(orc):
    """E4M3 decode of all 256 codes vs torch.float8_e4m3fn (independent library)."""
    codes = torch.arange(256, dtype=torch.int32).to(torch.uint8)
    ref = codes.view(torch.float8_e4m3fn).to(torch.float64).numpy()
    got = np.array([orc.e4m3_decode(c) for c in range(256)])
    nan = np.isnan(ref)
    assert np.array_equal(nan, np.isnan(got))
    assert np.array_equal(ref[~nan], got[~nan])
    assert orc.e4m3_decode(0x7E) == 448.0 and orc.e4m3_decode(0x01) == 2.0 ** -9


def _neighbourhood(centres, ulps=3):
    c = np.asarray(centres, dtype=np.float32)
    bits = c.view(np.int32)
    out = [c]
    for d in range(1, ulps + 1):
        out.append((bits + d).view(np.float32))
        out.append((bits - d).view(np.float32))
    v = np.concatenate(out)
    return v[np.isfinite(v) & (v >= 0)]


def test_e4m3_encode_matches_torch_rne(orc):
    """Nearest-even E4M3 (R3) vs torch's RNE float->e4m3fn conversion on every
    representable value and every midpoint +-3 ulp, plus random values; above the
    RNE overflow point (464) torch gives NaN and satfinite gives 448."""
    vals = np.array([orc.e4m3_decode(c) for c in range(0x7F)], dtype=np.float64)
    mids = (vals[:-1] + vals[1:]) / 2
    rng = np.random.default_rng(0)
    probes = np.concatenate([
        _neighbourhood(vals), _neighbourhood(mids),
        np.exp(rng.uniform(np.log(1e-4), np.log(460), 20000)).astype(np.float32),
    ])
    probes = probes[probes <= 464.0]
    ref = torch.from_numpy(probes).to(torch.float8_e4m3fn).view(torch.uint8).numpy()
    got = np.array([orc.e4m3_encode(float(v)) for v in probes], dtype=np.uint8)
    assert np.array_equal(ref, got)
    for big in (465.0, 1000.0, 3e38):
        assert orc.e4m3_encode(big) == 0x7E


def _e2m1_by_thresholds(v):
    """Independent E2M1 cast: comparisons against the midpoints between the
    representable magnitudes; at an exact midpoint take the even code."""
    mags = GOLDEN["e2m1_magnitudes"]["values"]
    a = abs(v)
    code = 7
    for i in range(7):
        mid = (mags[i] + mags[i + 1]) / 2
        if a < mid or (a == mid and i % 2 == 0):
            code = i
            break
    return code | (8 if math.copysign(1.0, v) < 0 else 0)


def test_e2m1_paper_examples(orc):
    mags = GOLDEN["e2m1_magnitudes"]["values"]
    # decode derived from the bit format (1 sign, 2 exponent, 1 mantissa; bias 1)
    for nib in range(16):
        e, m = (nib >> 1) & 3, nib & 1
        mag = (m * 0.5) if e == 0 else (1 + m / 2) * 2.0 ** (e - 1)
        assert orc.e2m1_decode(nib) == (-mag if nib & 8 else mag)
        assert abs(orc.e2m1_decode(nib)) == mags[nib & 7]
    for v, expect in GOLDEN["e2m1_cast_examples"]["cases"]:
        c = orc.e2m1_encode(v)
        assert orc.e2m1_decode(c) == expect and math.copysign(1, orc.e2m1_decode(c)) == math.copysign(1, expect)


def test_e2m1_encode_matches_threshold_impl(orc):
    mags = GOLDEN["e2m1_magnitudes"]["values"]
    mids = [(mags[i] + mags[i + 1]) / 2 for i in range(7)]
    rng = np.random.default_rng(1)
    probes = np.concatenate([_neighbourhood(mags + mids, 4), rng.uniform(0, 8, 20000).astype(np.float32),
                             np.float32([1e-30, 0.0, 6.0, 6.5, 1e30])])
    probes = np.concatenate([probes, -probes])
    for v in probes:
        assert orc.e2m1_encode(float(v)) == _e2m1_by_thresholds(float(v)), v


def test_bf16_rne_matches_torch(orc):
    rng = np.random.default_rng(2)
    bits = rng.integers(0, 2 ** 32, 200000, dtype=np.uint64).astype(np.uint32)
    # ties: low 16 bits exactly 0x8000
    bits[:5000] = (bits[:5000] & 0xFFFF0000) | 0x8000
    f = bits.view(np.float32)
    f = f[np.isfinite(f) & (np.abs(f) < 3.3e38)]
    ref = bf16_bits(f)
    got = np.array([orc.f32_to_bf16(float(v)) for v in f[:60000]], dtype=np.uint16)
    assert np.array_equal(ref[:60000], got)


# ---------------------------------------------------------------------------- NVFP4

@pytest.mark.parametrize("div", [2688.0, 1344.0])
def test_nvfp4_constant_block_paper_example(orc, div):
    """16 copies of 3.0 -> every code is +6.0 and dequantizes to exactly 3.0;
    holds for the tensor's own amax (2688) and the x2-headroom policy (1344)."""
    v = GOLDEN["nvfp4_block_examples"]["const_block_value"]
    x = bf16_bits(np.full((1, 16), v, np.float32))
    g = orc.global_scale(v, div)
    codes, sf = orc.nvfp4_quantize(x, g)
    assert np.all(codes == 0x77)
    assert np.all(orc.nvfp4_dequantize(codes, sf, g) == v)


def test_nvfp4_zero_block(orc):
    x = bf16_bits(np.zeros((2, 32), np.float32))
    x[1, :] = 0x8000  # -0.0: sign kept (R5)
    codes, sf = orc.nvfp4_quantize(x, 1.0)
    assert np.all(sf == 0)
    assert np.all(codes[0] == 0) and np.all(codes[1] == 0x88)
    assert np.all(orc.nvfp4_dequantize(codes, sf, 1.0) == 0)


def test_nvfp4_exact_representables_roundtrip(orc):
    """A block whose values are E2M1 magnitudes times a power-of-two scale, with
    the block max = 6*scale, quantizes to exactly those codes."""
    rng = np.random.default_rng(3)
    mags = np.array(GOLDEN["e2m1_magnitudes"]["values"])
    for trial in range(50):
        e = int(rng.integers(-8, 6))
        idx = rng.integers(0, 8, 16)
        idx[rng.integers(0, 16)] = 7
        sign = rng.integers(0, 2, 16)
        vals = np.where(sign == 1, -1, 1) * mags[idx] * 2.0 ** e
        x = bf16_bits(vals[None, :].astype(np.float32))
        codes, sf = orc.nvfp4_quantize(x, 1.0)
        dq = orc.nvfp4_dequantize(codes, sf, 1.0)
        assert np.array_equal(dq[0], vals)


def test_nvfp4_error_bound_and_max_maps_to_six(orc):
    """|x - x^| <= 1 * eff per element (half the widest E2M1 gap, 4..6), and each
    non-zero block's largest element maps to magnitude 6."""
    rng = np.random.default_rng(4)
    x32 = (rng.standard_normal((8, 256)) * np.exp(rng.uniform(-3, 3, (8, 1)))).astype(np.float32)
    x32[:, 7] *= 40
    x = bf16_bits(x32)
    xf = bf16_vals(x).astype(np.float64)
    amax = float(np.abs(xf).max())
    g = orc.global_scale(amax, 2688.0)
    codes, sf = orc.nvfp4_quantize(x, g)
    dq = orc.nvfp4_dequantize(codes, sf, g)
    # eff = fl32(dec(s_b) * g), the effective block scale of Eq. 2
    eff = (np.repeat(np.array([[orc.e4m3_decode(s) for s in row] for row in sf], dtype=np.float32), 16, axis=1)
           * np.float32(g)).astype(np.float64)
    assert np.all(np.abs(xf - dq) <= eff * (1 + 1e-6))
    blocks = np.abs(dq).reshape(8, -1, 16).max(axis=2)
    effb = eff.reshape(8, -1, 16)[:, :, 0]
    assert np.all(blocks == 6 * effb)


def test_nvfp4_reciprocal_reading_tie_vector(orc):
    """Reading R4 pin: eff = 0.029296875 (E4M3 0x0F, g = 1), x = 1.25*eff.
    x/eff would be the exact tie 1.25 -> 1.0, but x*fl(1/eff) = 1.2500001 -> 1.5."""
    blk = np.zeros((1, 16), np.float32)
    blk[0, 0] = 0.17578125          # 6 * eff -> block scale 0x0F
    blk[0, 1] = 0.03662109375       # 1.25 * eff (exactly representable in bf16)
    x = bf16_bits(blk)
    assert bf16_vals(x)[0, 1] == np.float32(0.03662109375)
    codes, sf = orc.nvfp4_quantize(x, 1.0)
    assert sf[0, 0] == 0x0F
    assert codes[0, 0] >> 4 == 3   # element 1 in the high nibble: code 1.5


def test_sf_layout_is_a_bijection(orc):
    m, k = 300, 320
    sf = np.arange(m * (k // 16), dtype=np.int64).reshape(m, k // 16) % 251
    sw = orc.sf_swizzle(sf.astype(np.uint8), m, k)
    assert sw.size == 384 * 20
    assert np.array_equal(orc.sf_unswizzle(sw, m, k), sf.astype(np.uint8))
    offs = {orc.sf_offset(r, c, k) for r in range(m) for c in range(k // 16)}
    assert len(offs) == m * (k // 16)


# ---------------------------------------------------------------------------- INT8

def test_int8_hand_example(orc):
    """Per-token symmetric INT8: row [-2, 1, 0.5, 0]: s = 2/127; 1.0*127/2
    = 63.5 exactly -> 64 (half to even); 0.5 -> 31.75 -> 32; -2 -> -127."""
    x = bf16_bits(np.array([[-2.0, 1.0, 0.5, 0.0]], np.float32))
    codes, s = orc.int8_quantize(x)
    assert list(codes[0]) == [-127, 64, 32, 0]
    assert s[0] == np.float32(2.0) / np.float32(127.0)
    z, s0 = orc.int8_quantize(bf16_bits(np.zeros((1, 8), np.float32)))
    assert s0[0] == 1.0 and np.all(z == 0)


def test_int8_bound_and_extremum(orc):
    rng = np.random.default_rng(5)
    x32 = (rng.standard_normal((16, 192)) * np.exp(rng.uniform(-4, 4, (16, 1)))).astype(np.float32)
    x = bf16_bits(x32)
    xf = bf16_vals(x).astype(np.float64)
    codes, s = orc.int8_quantize(x)
    err = np.abs(xf - codes.astype(np.float64) * s[:, None].astype(np.float64))
    assert np.all(err <= s[:, None] * (0.5 + 1e-5))
    am = np.argmax(np.abs(xf), axis=1)
    assert np.all(np.abs(codes[np.arange(16), am]) == 127)


# ---------------------------------------------------------------------------- weights

def test_pack_weights_consistency(orc):
    rng = np.random.default_rng(6)
    w = bf16_bits((rng.standard_normal((48, 128)) / np.sqrt(128)).astype(np.float32))
    pk = orc.pack_weights(w)
    amax = float(np.abs(bf16_vals(w)).max())
    assert pk["fp4_g"] == orc.global_scale(amax, 2688.0)
    c2, s2 = orc.nvfp4_quantize(w, pk["fp4_g"])
    assert np.array_equal(c2, pk["fp4_codes"]) and np.array_equal(s2, pk["fp4_sf"])
    # the INT8 form quantizes the DEQUANTIZED NVFP4 weights within s_w/2
    what = orc.nvfp4_dequantize(pk["fp4_codes"], pk["fp4_sf"], pk["fp4_g"])
    err = np.abs(what - pk["i8_codes"] * pk["i8_scale"][:, None].astype(np.float64))
    assert np.all(err <= pk["i8_scale"][:, None] * (0.5 + 1e-5))
    assert np.all(np.abs(pk["i8_codes"]).max(axis=1) == 127)


# ---------------------------------------------------------------------------- GEMMs

def test_gemm_int8_brute_force(orc):
    rng = np.random.default_rng(7)
    m, n, k = 5, 7, 64
    a = rng.integers(-128, 128, (m, k)).astype(np.int8)
    w = rng.integers(-128, 128, (n, k)).astype(np.int8)
    sa = rng.uniform(0.001, 0.1, m).astype(np.float32)
    sw = rng.uniform(0.001, 0.1, n).astype(np.float32)
    b = rng.standard_normal(n).astype(np.float32)
    acc, y = orc.gemm_int8(a, sa, w, sw, b)
    for i in range(m):
        for j in range(n):
            exact = sum(int(a[i, t]) * int(w[j, t]) for t in range(k))
            assert acc[i, j] == exact
            # R8: fma(fl(acc * s_a), s_w, bias) -- the fused step checked in exact rationals
            t = Fraction(float(np.float32(np.float32(exact) * sa[i])))
            yy = round_f32(t * Fraction(float(sw[j])) + Fraction(float(b[j])))
            assert y[i, j] == yy
    acc2, _ = orc.gemm_int8(a, sa, w, sw, b, rows=(2, 4))
    assert np.array_equal(acc2, acc[2:4])


def test_gemm_nvfp4_exact_fractions(orc):
    rng = np.random.default_rng(8)
    m, n, k = 3, 4, 64
    ac = rng.integers(0, 256, (m, k // 2)).astype(np.uint8)
    wc = rng.integers(0, 256, (n, k // 2)).astype(np.uint8)
    asf = rng.integers(0x20, 0x50, (m, k // 16)).astype(np.uint8)
    wsf = rng.integers(0x20, 0x50, (n, k // 16)).astype(np.uint8)
    ga, gw = np.float32(0.37), np.float32(1.9)
    b = rng.standard_normal(n).astype(np.float32)
    y = orc.gemm_nvfp4(ac, asf, ga, wc, wsf, gw, b)

    def dec(codes, sf, r, t):
        byte = int(codes[r, t // 2])
        nib = (byte >> 4) if t & 1 else (byte & 15)
        return Fraction(orc.e2m1_decode(nib)) * Fraction(orc.e4m3_decode(int(sf[r, t // 16])))

    gg = Fraction(float(np.float32(ga * gw)))
    for i in range(m):
        for j in range(n):
            s = sum(dec(ac, asf, i, t) * dec(wc, wsf, j, t) for t in range(k))
            exact = s * gg + Fraction(float(b[j]))
            assert abs(Fraction(y[i, j]) - exact) <= abs(exact) * Fraction(1, 2 ** 50) + Fraction(1, 2 ** 80)


def test_gemm_nvfp4_identity_weights(orc):
    """W with one-hot rows of code +1.0 and unit block scales (0x38), g_w = 1:
    Y = dequant(A) restricted to the selected columns (transposition check)."""
    rng = np.random.default_rng(9)
    m, k = 4, 32
    x = bf16_bits(rng.standard_normal((m, k)).astype(np.float32))
    ga = orc.global_scale(float(np.abs(bf16_vals(x)).max()), 2688.0)
    ac, asf = orc.nvfp4_quantize(x, ga)
    n = k
    wc = np.zeros((n, k // 2), np.uint8)
    for j in range(n):
        wc[j, j // 2] = 0x02 << (4 * (j & 1))
    wsf = np.full((n, k // 16), 0x38, np.uint8)
    y = orc.gemm_nvfp4(ac, asf, ga, wc, wsf, 1.0, None)
    # the block scales act inside the sum, g_a*g_w outside it (R3): Y = dec(a)*dec(sf_a)*g_a exactly
    assert np.array_equal(y, orc.nvfp4_dequantize(ac, asf, 1.0) * float(ga))


# ---------------------------------------------------------------------------- stats / TDC

def test_block_stats_paper_examples(orc):
    ones, twos = bf16_bits(np.ones(8, np.float32)), bf16_bits(2 * np.ones(8, np.float32))
    _, st = orc.block_stats(ones, twos)
    assert st[0] / st[1] == 1.0
    _, st = orc.block_stats(bf16_bits([1, -1]), bf16_bits([1.5, -0.5]))
    assert st[0] / st[1] == 0.5
    d = bf16_bits([0.5, -1.0, 2.0, 0.25])
    z = bf16_bits(np.zeros(4))
    for dp, e in [(d, 0.0), (bf16_bits([-0.5, 1.0, -2.0, -0.25]), 2.0),
                  (bf16_bits([2.0, 1.0, 0.0, 0.0]), 1.0), (bf16_bits([1.0, -2.0, 4.0, 0.5]), 0.0)]:
        dn, st = orc.block_stats(z, d, dp)
        assert np.array_equal(dn, d)
        assert orc.cosine_error_from_stats(st[4], st[5], st[6]) == pytest.approx(e, abs=1e-15)


def test_block_stats_vs_numpy(orc):
    rng = np.random.default_rng(10)
    xi = bf16_bits(rng.standard_normal(50000).astype(np.float32))
    xo = bf16_bits((bf16_vals(xi) + 0.05 * rng.standard_normal(50000)).astype(np.float32))
    dp = bf16_bits(0.05 * rng.standard_normal(50000).astype(np.float32))
    dn, st = orc.block_stats(xi, xo, dp)
    x, y, p = (bf16_vals(v).astype(np.float64) for v in (xi, xo, dp))
    d = (bf16_vals(xo) - bf16_vals(xi)).astype(np.float32).astype(np.float64)
    assert np.array_equal(dn, bf16_bits(d.astype(np.float32)))
    n = bf16_vals(dn).astype(np.float64)
    ref = [np.abs(d).sum(), np.abs(x).sum(), (d * d).sum(), (x * x).sum(), (n * p).sum(), (n * n).sum(), (p * p).sum()]
    np.testing.assert_allclose(st, ref, rtol=1e-12)


def test_tdc_skip_matches_torch_bf16_add(orc):
    rng = np.random.default_rng(11)
    xi = bf16_bits(rng.standard_normal(20000).astype(np.float32))
    d = bf16_bits(0.1 * rng.standard_normal(20000).astype(np.float32))
    out = orc.tdc_skip(xi, d)
    ref = (torch.from_numpy(xi.view(np.int16)).view(torch.bfloat16) + torch.from_numpy(d.view(np.int16)).view(torch.bfloat16))
    assert np.array_equal(out, ref.view(torch.int16).numpy().view(np.uint16))
    assert np.array_equal(orc.tdc_skip(xi, bf16_bits(np.zeros(20000))), xi)


# ---------------------------------------------------------------------------- decisions

def test_threshold_and_routing_examples(orc):
    g = GOLDEN["threshold_inversion"]
    assert orc.derive_tau_gamma(g["alpha"], g["beta"], g["tau_rel"]) == pytest.approx(g["tau_gamma"], rel=1e-12)
    assert orc.derive_tau_gamma(0.0, 0.001, 0.0025) == -math.inf
    r = GOLDEN["routing_examples"]
    for gamma, fmt in r["cases"]:
        got = orc.route_block(gamma, [r["tau_gamma"]], t=5, prev_skipped=False)[0]
        assert got == (orc.FMT_INT8 if fmt == "INT8" else orc.FMT_NVFP4)
    assert orc.route_block(0.0, [0.015], t=0, prev_skipped=False) == [orc.FMT_INT8]
    assert orc.route_block(0.0, [0.015], t=3, prev_skipped=True) == [orc.FMT_INT8]
    assert orc.route_block(None, [0.015], t=3, prev_skipped=False) == [orc.FMT_INT8]
    rng = np.random.default_rng(12)
    for _ in range(1000):
        a, b, tr = rng.uniform(0.01, 2), rng.uniform(-0.01, 0.01), rng.uniform(0, 0.05)
        assert a * orc.derive_tau_gamma(a, b, tr) + b == pytest.approx(tr, abs=1e-15)


def _run_trace(orc, cfg, etps, T):
    st = orc.TdcState()
    seq = []
    for t in range(T):
        dcs = orc.tdc_decide(st, cfg, t)
        seq.append(dcs)
        orc.tdc_update(st, cfg, t, dcs, etps[t] if dcs == 0 else None)
    return seq, st


def test_tdc_golden_trace(orc):
    g = GOLDEN["tdc_golden_trace"]
    cfg = orc.TdcConfig(rho=g["rho"], tau=g["tau"], n_max=g["n_max"])
    st = orc.TdcState()
    for t in range(2):   # warm-up computes
        assert orc.tdc_decide(st, cfg, t) == 0
        orc.tdc_update(st, cfg, t, 0, g["e_tp"])
    accs = [st.e_acc]
    decs = []
    for t in range(2, 5):
        d = orc.tdc_decide(st, cfg, t)
        decs.append("SKIP" if d else "COMPUTE")
        orc.tdc_update(st, cfg, t, d, g["e_tp"])
        accs.append(st.e_acc)
    assert decs == g["decisions_after_compute"]
    assert accs[:3] == pytest.approx(g["e_acc_sequence"], rel=1e-12)


def test_tdc_properties(orc):
    rng = np.random.default_rng(13)
    T = 50
    # tau = 0 with e_tp > 0: never skips
    seq, _ = _run_trace(orc, orc.TdcConfig(tau=0.0), rng.uniform(1e-6, 1e-2, T), T)
    assert sum(seq) == 0
    # tau = inf: exactly N_max skips between computes after warm-up
    seq, _ = _run_trace(orc, orc.TdcConfig(tau=math.inf, n_max=2), rng.uniform(0, 1, T), T)
    assert seq[:8] == [0, 0, 1, 1, 0, 1, 1, 0]
    # never more than N_max consecutive skips
    for trial in range(200):
        n_max = int(rng.integers(1, 5))
        seq, _ = _run_trace(orc, orc.TdcConfig(tau=float(rng.uniform(0, 0.01)), n_max=n_max),
                            rng.uniform(0, 0.004, T), T)
        run = best = 0
        for s in seq:
            run = run + 1 if s else 0
            best = max(best, run)
        assert best <= n_max


# ---------------------------------------------------------------------------- block Hadamard (R14)

def _sylvester(n):
    h = np.array([[1.0]])
    while h.shape[0] < n:
        h = np.block([[h, h], [h, -h]])
    return h


def test_fht_one_hot_is_a_hadamard_row(orc):
    """Sylvester H[i][j] = (-1)^popcount(i & j); a one-hot block maps to the +-1 row
    exactly (every butterfly adds a value to zero)."""
    s = np.float32(1.0)
    for j in (0, 1, 5, 64, 127):
        x = np.zeros((1, 128), np.float32)
        x[0, j] = 1.0
        y = orc.fht128(x)[0]
        ref = np.array([(-1.0) ** bin(i & j).count("1") for i in range(128)], np.float32) * s
        assert np.array_equal(y, ref)


def test_fht_matches_dense_transform_and_is_an_involution(orc):
    rng = np.random.default_rng(21)
    x = rng.standard_normal((6, 384)).astype(np.float32)
    x[:, 7] *= 80.0
    y = orc.fht128(x)
    H = _sylvester(128)
    dense = (x.astype(np.float64).reshape(6, 3, 128) @ H.T).reshape(6, 384)
    assert np.max(np.abs(y - dense)) <= 1e-5 * np.max(np.abs(dense))
    # Parseval for the unnormalized transform: ||Hx||^2 = 128 ||x||^2
    np.testing.assert_allclose(np.linalg.norm(y, axis=1), np.sqrt(128.0) * np.linalg.norm(x.astype(np.float64), axis=1),
                               rtol=1e-6)
    assert np.max(np.abs(orc.fht128(y) / 128.0 - x)) <= 1e-5 * np.max(np.abs(x))   # H H = 128 I (S:209 involution)
    # linear-layer transparency: (Hx).(2^-7 Hw) == x.w
    w = rng.standard_normal((4, 384)).astype(np.float32)
    np.testing.assert_allclose(orc.fht128(x).astype(np.float64) @ (orc.fht128(w) / 128.0).T.astype(np.float64),
                               x.astype(np.float64) @ w.T.astype(np.float64), rtol=1e-5, atol=1e-4)


def test_fht_smooths_channel_outliers_for_int8(orc):
    """P:187 / S:220: block-Hadamard smoothing redistributes activation outliers; with
    a few large outlier channels, the per-token INT8 error (scale set by the row max)
    drops after the rotation (the error is measured back in the original basis)."""
    rng = np.random.default_rng(22)
    e_plain, e_fht = [], []
    for trial in range(40):
        x = rng.standard_normal((4, 256)).astype(np.float32)
        x[:, rng.integers(0, 256, 2)] *= 60.0
        xb = torch.tensor(x).to(torch.bfloat16).float().numpy()
        c, s = orc.int8_quantize_f32(xb)
        e_plain.append(np.linalg.norm(c * s[:, None] - xb) / np.linalg.norm(xb))
        y = orc.fht128(xb)
        c2, s2 = orc.int8_quantize_f32(y)
        back = orc.fht128((c2 * s2[:, None]).astype(np.float32)) / 128.0
        e_fht.append(np.linalg.norm(back - xb) / np.linalg.norm(xb))
    assert np.mean(e_fht) < 0.5 * np.mean(e_plain)


def test_f32_quantizers_agree_with_bf16_ones_on_bf16_values(orc):
    rng = np.random.default_rng(23)
    x = torch.tensor(rng.standard_normal((5, 128)).astype(np.float32)).to(torch.bfloat16)
    xb, xf = bf16_bits(x.float().numpy()), x.float().numpy()
    c1, s1 = orc.nvfp4_quantize(xb, 0.01)
    c2, s2 = orc.nvfp4_quantize_f32(xf, 0.01)
    assert np.array_equal(c1, c2) and np.array_equal(s1, s2)
    i1, t1 = orc.int8_quantize(xb)
    i2, t2 = orc.int8_quantize_f32(xf)
    assert np.array_equal(i1, i2) and np.array_equal(t1, t2)


def test_pack_weights_hadamard(orc):
    rng = np.random.default_rng(24)
    w = bf16_bits((rng.standard_normal((32, 256)) / 16).astype(np.float32))
    pk = orc.pack_weights_hadamard(w)
    wr = orc.fht128(bf16_vals(w)) * np.float32(2.0 ** -7)
    assert pk["fp4_g"] == orc.global_scale(float(np.abs(wr).max()), 2688.0)
    c, s = orc.nvfp4_quantize_f32(wr, pk["fp4_g"])
    assert np.array_equal(c, pk["fp4_codes"]) and np.array_equal(s, pk["fp4_sf"])
    what = orc.nvfp4_dequantize(pk["fp4_codes"], pk["fp4_sf"], pk["fp4_g"])
    err = np.abs(what - pk["i8_codes"] * pk["i8_scale"][:, None].astype(np.float64))
    assert np.all(err <= pk["i8_scale"][:, None] * (0.5 + 1e-5))


# ---------------------------------------------------------------------------- Purified Cache Refresh (R15)

def test_outlier_ratio_spec_examples(orc):
    """constant magnitude -> 1; [50, 2, 2, 2] -> 50/14; one spike 1000 among
    999 ones -> 1000 / (1999/1000); all-zero -> 1."""
    assert orc.outlier_ratio(bf16_bits(np.full(64, -3.0, np.float32))) == 1.0
    assert orc.outlier_ratio(bf16_bits([50.0, 2.0, 2.0, 2.0])) == pytest.approx(50.0 / 14.0, rel=1e-15)
    x = np.ones(1000, np.float32)
    x[17] = 1000.0
    assert orc.outlier_ratio(bf16_bits(x)) == pytest.approx(1000.0 / (1999.0 / 1000.0), rel=1e-15)
    assert orc.outlier_ratio(bf16_bits(np.zeros(8, np.float32))) == 1.0
    # strided sampling: every 2nd element of [50, 9, 2, 9, 2, 9] -> [50, 2, 2]
    assert orc.outlier_ratio(bf16_bits([50.0, 9.0, 2.0, 9.0, 2.0, 9.0]), stride=2) == pytest.approx(50.0 / 18.0)


def test_purify_route_precedence(orc):
    """ratio exactly tau keeps the base decision (strict '>');
    after a skip (ratio <= tau) every layer is INT8; ratio 500 -> BF16 regardless;
    precedence outlier > post-skip > base."""
    B, I, N = orc.FMT_BF16, orc.FMT_INT8, orc.FMT_NVFP4
    assert orc.purify_route(N, 25.0, False, 25.0) == N
    assert orc.purify_route(N, 24.0, True, 25.0) == I
    assert orc.purify_route(N, 500.0, False, 25.0) == B
    assert orc.purify_route(I, 500.0, True, 25.0) == B
    assert orc.purify_route(N, None, False, 25.0) == N


def test_gemm_bf16_exact_fractions(orc):
    rng = np.random.default_rng(25)
    x = bf16_bits(rng.standard_normal((3, 64)).astype(np.float32))
    w = bf16_bits(rng.standard_normal((5, 64)).astype(np.float32))
    b = rng.standard_normal(5).astype(np.float32)
    y = orc.gemm_bf16(x, w, b)
    xf, wf = bf16_vals(x), bf16_vals(w)
    for i in range(3):
        for j in range(5):
            exact = sum(Fraction(float(xf[i, t])) * Fraction(float(wf[j, t])) for t in range(64)) + Fraction(float(b[j]))
            assert abs(Fraction(y[i, j]) - exact) <= abs(exact) * Fraction(1, 2 ** 50) + Fraction(1, 2 ** 80)


# ----------------------------------------------------------------------------- compressed delta cache (R16)

E2M1_GRID = np.array([0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0])


def _exact_cache_case(m, h, seed):
    """x_in on a 2^-4 grid in [-4, 4] and a delta on the E2M1 grid x 2^-3 with +-0.75
    (= 6 x 2^-3) in every 16-block: y = x + delta is exactly bf16, d = delta exactly,
    and NVFP4(d; g = 1) is lossless (block scale 2^-3 is an exact E4M3 value)."""
    rng = np.random.default_rng(seed)
    x = rng.integers(-64, 65, size=(m, h)) / 16.0
    mag = E2M1_GRID[rng.integers(0, 8, size=(m, h))] * 0.125
    d = mag * rng.choice([-1.0, 1.0], size=(m, h))
    d.reshape(m, h // 16, 16)[:, :, 0] = 0.75 * rng.choice([-1.0, 1.0], size=(m, h // 16))
    xt = torch.tensor(x, dtype=torch.float32).to(torch.bfloat16)
    yt = torch.tensor(x + d, dtype=torch.float32).to(torch.bfloat16)
    assert torch.equal(yt.float() - xt.float(), torch.tensor(d, dtype=torch.float32))
    return xt, yt, d


def test_cache_lossless_deltas_reduce_to_the_uncompressed_cache(orc):
    """R16 pinned against the uncompressed TDC functions: with NVFP4-representable deltas
    the compressed cache stores them exactly, so skip output and refresh statistics equal
    oracle_tdc_skip / oracle_block_stats with a bf16 cache (independent code paths)."""
    from paper_2603_18742_b200 import synth
    m, h = 6, 64
    xi, xo, d = _exact_cache_case(m, h, 1)
    _, xp, dp = _exact_cache_case(m, h, 2)      # an earlier delta, also exactly representable
    cp, sp = orc.nvfp4_quantize_f32(dp.astype(np.float32), 1.0)
    assert np.array_equal(orc.cache_dequant(cp, sp, 1.0), dp.astype(np.float32))
    cn, sn, st, am = orc.block_stats_nvfp4(synth.bits(xi), synth.bits(xo), cp, sp, 1.0, 1.0)
    dp_bf16 = synth.bits(torch.tensor(dp, dtype=torch.float32).to(torch.bfloat16))
    _, st_ref = orc.block_stats(synth.bits(xi), synth.bits(xo), dp_bf16)
    np.testing.assert_array_equal(st, st_ref)
    assert am == float(np.abs(d).max())
    assert np.array_equal(orc.cache_dequant(cn, sn, 1.0), d.astype(np.float32))
    d_bf16 = synth.bits(torch.tensor(d, dtype=torch.float32).to(torch.bfloat16))
    assert np.array_equal(orc.tdc_skip_nvfp4(synth.bits(xi), cn, sn, 1.0), orc.tdc_skip(synth.bits(xi), d_bf16))


def _dequant_numpy(codes, sf, g):
    """dec(code) * fl32(dec(s) * g) written out with numpy float32 (SPEC S:370's
    codec-composition oracle): nibble -> sign x E2M1 grid, E4M3 via torch."""
    m = codes.shape[0]
    nib = np.stack([codes & 15, codes >> 4], axis=-1).reshape(m, -1)
    val = E2M1_GRID[nib & 7] * np.where(nib & 8, -1.0, 1.0)
    s = torch.tensor(sf.reshape(-1)).view(torch.float8_e4m3fn).float().numpy().reshape(m, -1)
    eff = (s.astype(np.float32) * np.float32(g)).astype(np.float32)
    return (val.astype(np.float32) * np.repeat(eff, 16, axis=1)).astype(np.float32)


def test_cache_skip_is_codec_composition(orc):
    """Skip output equals x_in + dequant(quant_nvfp4(Delta)), composed by hand
    (numpy float32 add, torch RNE to bf16); refresh amax and dequant error bound."""
    from paper_2603_18742_b200 import synth
    m, h = 5, 128
    xi = synth.dit_activation(m, h, seed=11)
    xo = (xi.float() + 0.05 * synth.dit_activation(m, h, seed=12).float()).to(torch.bfloat16)
    d = (xo.float() - xi.float()).numpy()
    g = orc.global_scale(float(np.abs(d).max()), 1344.0)
    zc, zs = np.zeros((m, h // 2), np.uint8), np.zeros((m, h // 16), np.uint8)
    cn, sn, st, am = orc.block_stats_nvfp4(synth.bits(xi), synth.bits(xo), zc, zs, 0.0, g)
    assert am == float(np.abs(d).max())
    assert st[4] == 0.0 and st[6] == 0.0           # an empty (zero) cache contributes nothing
    dq = _dequant_numpy(cn, sn, g)
    np.testing.assert_array_equal(orc.cache_dequant(cn, sn, g), dq)
    eff = np.repeat((torch.tensor(sn.reshape(-1)).view(torch.float8_e4m3fn).float().numpy() * np.float32(g))
                    .astype(np.float32).reshape(m, -1), 16, axis=1)
    assert np.all(np.abs(dq.astype(np.float64) - d) <= eff)      # one E2M1 step at most
    ref = (xi.float() + torch.tensor(dq)).to(torch.bfloat16)
    assert np.array_equal(orc.tdc_skip_nvfp4(synth.bits(xi), cn, sn, g), synth.bits(ref))


# ---------------------------------------------------------------------------- round-2 pins
# (functions the round-1 pins only used as checkers; each pinned to an independent source)

def test_amax_bf16_vs_numpy(orc):
    """Tensor amax max|x| (R3's delayed global scale) against numpy's reduction over the widened
    bf16 values; rows whose largest magnitude is negative, signed zeros and huge/tiny values."""
    rng = np.random.default_rng(21)
    cases = [rng.standard_normal((37, 64)).astype(np.float32),
             np.array([[0.5, -7.25, 3.0, -0.0]], np.float32),           # max magnitude is negative
             np.array([[-0.0, -0.0, 0.0]], np.float32),                 # all zeros -> 0
             np.array([[1e-38, -3e-39, 2e-40]], np.float32),            # bf16 subnormals
             np.array([[-3.0e38, 1.0, 2.5e38]], np.float32)]
    for c in cases:
        b = bf16_bits(c)
        assert orc.amax_bf16(b) == float(np.abs(bf16_vals(b)).max())
    assert orc.amax_bf16(bf16_bits([[-7.25, 7.0]])) == 7.25


def test_global_scale_floor_and_division(orc):
    """g = max(fl(amax / div), FLT_MIN) (R3): IEEE single division (numpy float32) above the
    floor; amax 0 and quotients below FLT_MIN (subnormal or zero) give exactly FLT_MIN."""
    flt_min = float(np.finfo(np.float32).tiny)
    for div in (1344.0, 2688.0):
        assert orc.global_scale(0.0, div) == flt_min
        assert orc.global_scale(1e-40, div) == flt_min          # denormal amax
        assert orc.global_scale(flt_min, div) == flt_min        # quotient underflows below the floor
        assert orc.global_scale(div, div) == 1.0
        rng = np.random.default_rng(int(div))
        for a in np.concatenate([10.0 ** rng.uniform(-30, 30, 2000), [448.0 * 6, 1.0, 3.0]]).astype(np.float32):
            q = np.float32(a) / np.float32(div)
            assert orc.global_scale(float(a), div) == float(max(q, np.float32(flt_min)))


def test_gamma_l2_spec_examples(orc):
    """Eq. 4's normalized L2 distance as the L2 variant of Gamma (R1), from the statistics the
    refresh produces: SPEC rel_l2 examples and the identity case."""
    ex = GOLDEN["rel_l2_examples"]["cases"]
    for case in ex:
        _, st = orc.block_stats(bf16_bits(case["ref"]), bf16_bits(case["other"]))
        want = math.sqrt(2.0) if case["value"] == "sqrt2" else case["value"]
        assert orc.gamma_from_stats(st, "l2") == pytest.approx(want, rel=1e-15)
    x = bf16_bits([0.5, -2.0, 3.0])
    _, st = orc.block_stats(x, x)
    assert orc.gamma_from_stats(st, "l2") == 0.0
    _, st = orc.block_stats(bf16_bits([0.0, 0.0]), bf16_bits([1.0, 1.0]))
    assert orc.gamma_from_stats(st, "l2") is None                  # zero-norm reference
    # L1 and L2 differ where they should: ref [1, 1], other [2, 1] -> L1 0.5, L2 1/sqrt(2)
    _, st = orc.block_stats(bf16_bits([1.0, 1.0]), bf16_bits([2.0, 1.0]))
    assert orc.gamma_from_stats(st, "l1") == 0.5
    assert orc.gamma_from_stats(st, "l2") == pytest.approx(1 / math.sqrt(2), rel=1e-15)


# Scale-factor placement of the tcgen05 block-scaled MMA, written from the hardware's data path
# rather than from the oracle's formula: a 128-row x 4-scale-column chunk (128 rows x 64 K elements
# at scale_vec::4X) is one 512-byte smem atom, copied to TMEM by tcgen05.cp .32x128b.warpx4 as 32
# rows of 16 bytes, row l going to TMEM lane l of every 32-lane quarter q; the MMA row m = 32 q + l
# reads its four K-block scales from bytes 4q .. 4q+3 of that 16-byte row. Atoms are stored
# K-fastest (all K chunks of a 128-row tile, then the next 128 rows). Each entry: (r, c, k) -> byte.
SF_HAND_TABLE = [
    ((0, 0, 64), 0),            # first scale of the first atom
    ((0, 3, 64), 3),            # 4th K-block of row 0: same 16-byte row, byte 3
    ((1, 0, 64), 16),           # row 1 -> smem row 1 (lane 1 of quarter 0)
    ((31, 0, 64), 496),         # last smem row
    ((32, 0, 64), 4),           # row 32 = lane 0 of quarter 1 -> bytes 4..7 of smem row 0
    ((33, 2, 64), 22),          # lane 1, quarter 1, K-block 2: 16 + 4 + 2
    ((96, 1, 64), 13),          # quarter 3: bytes 12..15 of smem row 0
    ((127, 3, 64), 511),        # last byte of the atom
    ((128, 0, 64), 512),        # second 128-row tile (k = 64: one atom per row tile)
    ((0, 4, 128), 512),         # k = 128: the second K chunk of row tile 0 comes next (K-fastest)
    ((128, 0, 128), 1024),      # then row tile 1
    ((128, 5, 128), 1537),      # row tile 1, K chunk 1, K-block 1
    ((200, 117, 1920), 30345),  # k = 1920: 30 K chunks per row tile; (1*30 + 29)*512 + 8*16 + 2*4 + 1
]


def test_sf_offset_hand_table(orc):
    for (r, c, k), byte in SF_HAND_TABLE:
        assert orc.sf_offset(r, c, k) == byte, (r, c, k)
        # the gather used by the tests agrees with the table too
        dev = np.zeros(orc.sf_swizzled_bytes(r + 1, k), np.uint8)
        dev[byte] = 0x5A
        logical = orc.sf_unswizzle(dev, r + 1, k)
        assert logical[r, c] == 0x5A and int((logical == 0x5A).sum()) == 1


def test_sf_offset_hierarchical_layout(orc):
    """The same placement from CuTe's hierarchical layout notation of the SF atom,
    Shape ((32, 4), (16, 4)) : Stride ((16, 4), (0, 1)) over (row, K element) of a 128 x 64 tile,
    evaluated by a generic colexicographic shape/stride evaluator, tiled K-fastest."""
    def evaluate(coord, shape, stride):
        off = 0
        for x, sh, st in zip(coord, shape, stride):
            if isinstance(sh, tuple):
                for s_, t_ in zip(sh, st):
                    off += (x % s_) * t_
                    x //= s_
            else:
                off += x * st
        return off
    shape, stride = ((32, 4), (16, 4)), ((16, 4), (0, 1))
    for k in (64, 192, 1920, 3072):
        kc4 = k // 64
        for r in (0, 5, 31, 32, 77, 127, 128, 300, 1000):
            for c in sorted({0, 1, 3, 4, k // 16 - 1, (k // 16) // 2}):
                ke = c * 16 + 7          # any K element of the 16-element block
                inner = evaluate(((r % 128), ke % 64), shape, stride)
                atom = (r // 128) * kc4 + (ke // 64)
                assert orc.sf_offset(r, c, k) == atom * 512 + inner, (r, c, k)


# ---------------------------------------------------------------------------- per-block INT8 (R17, NEXT-1)

def test_int8_blocks_hand_example(orc):
    """Two 128-blocks of one row with different maxima get their own scales s = max/127 (P:187:
    per-block symmetric INT8): block 0 max 2 -> s = fl(2/127), 1.0 -> code 64 (63.5 ties to even);
    block 1 max 0.5 -> s = fl(0.5/127), 0.25 -> 64 (63.5), -0.5 -> -127; a zero block -> s = 1."""
    x = np.zeros((1, 384), np.float32)
    x[0, 0], x[0, 1] = -2.0, 1.0
    x[0, 128], x[0, 129], x[0, 130] = 0.5, 0.25, -0.5
    c, s = orc.int8_quantize_blocks_f32(x)
    assert s[0, 0] == np.float32(2.0) / np.float32(127.0) and s[0, 1] == np.float32(0.5) / np.float32(127.0)
    assert s[0, 2] == 1.0
    assert list(c[0, :2]) == [-127, 64] and list(c[0, 128:131]) == [127, 64, -127]
    assert not c[0, 256:].any()


def test_int8_blocks_reduce_to_per_token(orc):
    """With B = K the per-block quantizer is the per-token one (same codes and scales); with every
    block of a row sharing its maximum the block scales all equal the row's."""
    rng = np.random.default_rng(30)
    x = (rng.standard_normal((17, 256)) * np.exp(rng.standard_normal((17, 1)))).astype(np.float32)
    c1, s1 = orc.int8_quantize_blocks_f32(x, block=256)
    c0, s0 = orc.int8_quantize_f32(x)
    assert np.array_equal(c1, c0) and np.array_equal(s1[:, 0], s0)
    y = x.copy()
    y[:, 0] = y[:, 128] = np.abs(y).max(axis=1) * 2   # same block maxima in both blocks
    cb, sb = orc.int8_quantize_blocks_f32(y)
    ct, st = orc.int8_quantize_f32(y)
    assert np.array_equal(cb, ct) and np.array_equal(sb[:, 0], st) and np.array_equal(sb[:, 1], st)


def test_int8_blocks_error_bound(orc):
    rng = np.random.default_rng(31)
    x = (rng.standard_normal((9, 512)) * rng.choice([1e-3, 1.0, 50.0], size=(9, 512))).astype(np.float32)
    c, s = orc.int8_quantize_blocks_f32(x)
    deq = c.astype(np.float64).reshape(9, 4, 128) * s.astype(np.float64)[:, :, None]
    err = np.abs(deq - x.astype(np.float64).reshape(9, 4, 128))
    assert np.all(err <= 0.5 * s.astype(np.float64)[:, :, None] * (1 + 1e-6))
    for r in range(9):   # every block maximum maps to +-127
        for b in range(4):
            blk = x[r, b * 128:(b + 1) * 128]
            assert abs(int(c[r, b * 128 + int(np.abs(blk).argmax())])) == 127


def test_gemm_int8_blocks_exact_fractions(orc):
    """sum_b (sum_{k in b} a w) s_a[b] s_w + bias against exact rationals on small random inputs;
    and a GEMM whose blocks all share one scale equals the per-token INT8 GEMM's exact value."""
    rng = np.random.default_rng(32)
    m, n, k = 3, 5, 384
    a = rng.integers(-128, 128, size=(m, k), dtype=np.int8)
    w = rng.integers(-128, 128, size=(n, k), dtype=np.int8)
    sa = rng.uniform(1e-3, 1, size=(m, 3)).astype(np.float32)
    sw = rng.uniform(1e-3, 1, size=n).astype(np.float32)
    bias = rng.uniform(-1, 1, size=n).astype(np.float32)
    y = orc.gemm_int8_blocks(a, sa, w, sw, bias)
    for i in range(m):
        for j in range(n):
            t = sum(Fraction(int(np.dot(a[i, b * 128:(b + 1) * 128].astype(np.int64),
                                        w[j, b * 128:(b + 1) * 128].astype(np.int64)))) * Fraction(float(sa[i, b]))
                    for b in range(3))
            exact = t * Fraction(float(sw[j])) + Fraction(float(bias[j]))
            assert abs(Fraction(y[i, j]) - exact) <= abs(exact) * Fraction(1, 2 ** 50)
    sa_eq = np.repeat(sa[:, :1], 3, axis=1)
    y_eq = orc.gemm_int8_blocks(a, sa_eq, w, sw, None)
    acc = a.astype(np.int64) @ w.astype(np.int64).T
    ref = acc.astype(np.float64) * sa[:, :1].astype(np.float64) * sw.astype(np.float64)[None, :]
    np.testing.assert_allclose(y_eq, ref, rtol=1e-15)


def test_rel_l2_prediction_error(orc):
    """Eq. 9 with D = relative-L2 distance (R19) from the refresh statistics: SPEC rel_l2
    examples with Delta_prev as the reference, numpy's norm of the difference on random
    deltas, zero reference -> +inf; and it differs from 1 - cos where it should."""
    z = bf16_bits(np.zeros(2, np.float32))
    for dn, dp, want in (([0.0, 0.0], [3.0, 4.0], 1.0), ([0.0, 1.0], [1.0, 0.0], math.sqrt(2.0)),
                         ([2.0, 2.0], [1.0, 1.0], 1.0), ([1.5, -0.5], [1.5, -0.5], 0.0)):
        _, st = orc.block_stats(z, bf16_bits(dn), bf16_bits(dp))
        assert orc.prediction_error_from_stats(st, "rel_l2") == pytest.approx(want, abs=1e-15)
    _, st = orc.block_stats(z, bf16_bits([2.0, 2.0]), bf16_bits([1.0, 1.0]))
    assert orc.prediction_error_from_stats(st, "cos") == pytest.approx(0.0, abs=1e-15)   # scaled: cos blind
    _, st = orc.block_stats(z, bf16_bits([1.0, 1.0]), bf16_bits([0.0, 0.0]))
    assert orc.prediction_error_from_stats(st, "rel_l2") == math.inf
    rng = np.random.default_rng(33)
    n = 4096
    xi = bf16_bits(rng.standard_normal(n).astype(np.float32))
    xo = bf16_bits((bf16_vals(xi) + 0.05 * rng.standard_normal(n)).astype(np.float32))
    dp = bf16_bits((0.05 * rng.standard_normal(n)).astype(np.float32))
    dn, st = orc.block_stats(xi, xo, dp)
    a, b = bf16_vals(dn).astype(np.float64), bf16_vals(dp).astype(np.float64)
    assert orc.prediction_error_from_stats(st, "rel_l2") == pytest.approx(np.linalg.norm(a - b) / np.linalg.norm(b),
                                                                          rel=1e-12)
