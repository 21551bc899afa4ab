/*
 * dmpq_oracle.c — plain, slow, obviously-correct CPU oracle for the DMPQ + TDC
 * hot path of "6Bit-Diffusion" (arxiv 2603.18742, /root/reference/PAPER.md).
 *
 * TEST INFRASTRUCTURE ONLY. Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs may load this library. It shares no code,
 * header, table or constant generator with the CUDA path
 * (paper_2603_18742_b200/csrc/), and must never be reached from the product path.
 *
 * Citation format: P:<line> = /root/reference/PAPER.md line; S:<line> = SPEC.md
 * line; "reading Rn" = a numbered reading in DESIGN.md §3 where the paper is
 * silent or ambiguous.
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off -fno-fast-math -fexcess-precision=standard
 *        -fPIC -shared  (no FMA contraction: every float op below is one IEEE-754
 *        binary32 operation rounded to nearest-even, as written).
 *
 * Every conversion is done by exhaustive nearest search over the finite value set
 * of the target format (the plain definition of round-to-nearest with
 * saturation); ties go to the even code.  Nothing here is blocked, fused or
 * reordered beyond what the definitions state.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#include <float.h>

/* ------------------------------------------------------------------------ */
/* bf16 <-> fp32 (storage format of activations/weights; not part of the paper) */
/* ------------------------------------------------------------------------ */

float oracle_bf16_to_f32(uint16_t h) {
    uint32_t u = (uint32_t)h << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* Round-to-nearest-even fp32 -> bf16, by comparing the two bf16 neighbours of v
 * (truncation and truncation+1ulp) in exact (double) arithmetic. Finite v only. */
uint16_t oracle_f32_to_bf16(float v) {
    uint32_t u;
    memcpy(&u, &v, 4);
    uint16_t lo = (uint16_t)(u >> 16);           /* toward zero */
    uint16_t hi = (uint16_t)(lo + 1);            /* away from zero (next magnitude) */
    if ((u & 0xFFFFu) == 0) return lo;           /* exactly representable */
    double dv = (double)v;
    double dlo = (double)oracle_bf16_to_f32(lo);
    double dhi = (double)oracle_bf16_to_f32(hi);  /* may be inf: then |v-dhi| = inf */
    double elo = fabs(dv - dlo), ehi = fabs(dv - dhi);
    if (elo < ehi) return lo;
    if (ehi < elo) return hi;
    return (lo & 1u) ? hi : lo;                  /* tie: even mantissa */
}

/* ------------------------------------------------------------------------ */
/* FP8 E4M3 (e4m3fn): the NVFP4 block-scale format ("shared FP8 scaling   */
/* factor"; reading R3 fixes E4M3).  1 sign, 4 exponent (bias 7), 3 mantissa;  */
/* exponent 0 is subnormal; 0x7F/0xFF are NaN; largest finite = 448.           */
/* ------------------------------------------------------------------------ */

double oracle_e4m3_decode(uint8_t code) {
    int s = code >> 7, e = (code >> 3) & 0xF, m = code & 7;
    double mag;
    if (e == 0xF && m == 7) return NAN;
    if (e == 0) mag = ldexp((double)m / 8.0, -6);
    else        mag = ldexp(1.0 + (double)m / 8.0, e - 7);
    return s ? -mag : mag;
}

/* Nearest finite non-negative E4M3 value to v >= 0 (exhaustive scan over codes
 * 0x00..0x7E), ties to the even code; values beyond 448 saturate to 448
 * ("satfinite", reading R3). */
uint8_t oracle_e4m3_encode_nonneg(float v) {
    /* Beyond 512 every candidate is farther than 448 and, in floating point, the
     * distances |c - v| would all round to |v|; clamping first keeps the scan exact
     * (below 512 each distance is exact in double). */
    double dv = (double)v > 512.0 ? 512.0 : (double)v;
    uint8_t best = 0;
    double best_err = INFINITY;
    for (int c = 0; c <= 0x7E; ++c) {
        double err = fabs(oracle_e4m3_decode((uint8_t)c) - dv);
        if (err < best_err || (err == best_err && (c & 1) == 0 && (best & 1) != 0)) {
            best = (uint8_t)c;
            best_err = err;
        }
    }
    return best;
}

/* ------------------------------------------------------------------------ */
/* FP4 E2M1 ("1 sign bit, 2 exponent bits, and 1 mantissa bit",    */
/* max 6.0, "CastToFP4 maps normalized values to the nearest representable FP4 */
/* magnitude").  Nibble: bit3 = sign, bits0..2 index into the magnitudes.       */
/* ------------------------------------------------------------------------ */

static const double E2M1_MAG[8] = {0.0, 0.5, 1.0, 1.5, 2.0, 3.0, 4.0, 6.0};

double oracle_e2m1_decode(uint8_t nib) {
    double mag = E2M1_MAG[nib & 7];
    return (nib & 8) ? -mag : mag;
}

/* CastToFP4 (Eq. 2): nearest magnitude, ties to the even code (even
 * mantissa bit), saturating at 6; the sign bit is kept even when the magnitude
 * rounds to zero (reading R5). */
uint8_t oracle_e2m1_encode(float v) {
    /* clamp as in the E4M3 scan: above 8 the nearest magnitude is 6 */
    double a = fabs((double)v) > 8.0 ? 8.0 : fabs((double)v);
    int best = 0;
    double best_err = INFINITY;
    for (int c = 0; c < 8; ++c) {
        double err = fabs(E2M1_MAG[c] - a);
        if (err < best_err || (err == best_err && (c & 1) == 0 && (best & 1) != 0)) {
            best = c;
            best_err = err;
        }
    }
    return (uint8_t)(best | (signbit(v) ? 8 : 0));
}

/* ------------------------------------------------------------------------ */
/* NVFP4 quantization, Eq. 2 with the two-level scale of reading   */
/* R3: per 16-element block b of a row,                                       */
/*   a_b  = max |x|                                                           */
/*   raw  = fl(fl(a_b / 6) / g)            (s = max|X|/6.0, relative to g) */
/*   s_b  = E4M3(raw)                      (stored FP8 block scale)           */
/*   eff  = fl(dec(s_b) * g)               (effective scale s of Eq. 2)        */
/*   r    = eff > 0 ? fl(1 / eff) : 0      (reading R4: X/s as X * (1/s))     */
/*   code = sign(x) | E2M1(|fl(x * r)|)                                        */
/* x: bf16 [m x k] row-major (leading dim ldx elements), k % 16 == 0.          */
/* codes: [m x k/2] bytes, element 2i in the low nibble (reading R6).           */
/* sf: logical [m x k/16] E4M3 bytes, row-major (the swizzled device layout is  */
/* a separate index map, oracle_sf_offset()).                                  */
/* ------------------------------------------------------------------------ */

void oracle_nvfp4_quantize(const uint16_t* x, int m, int k, int ldx, float g,
                           uint8_t* codes, uint8_t* sf) {
    for (int r = 0; r < m; ++r) {
        for (int b = 0; b < k / 16; ++b) {
            const uint16_t* xb = x + (size_t)r * ldx + (size_t)b * 16;
            float a_b = 0.0f;
            for (int i = 0; i < 16; ++i) {
                float v = fabsf(oracle_bf16_to_f32(xb[i]));
                if (v > a_b) a_b = v;
            }
            float raw = (a_b / 6.0f) / g;
            uint8_t s_b = oracle_e4m3_encode_nonneg(raw);
            float eff = (float)oracle_e4m3_decode(s_b) * g;
            float rcp = eff > 0.0f ? 1.0f / eff : 0.0f;
            sf[(size_t)r * (k / 16) + b] = s_b;
            for (int i = 0; i < 16; i += 2) {
                float q0 = oracle_bf16_to_f32(xb[i]) * rcp;
                float q1 = oracle_bf16_to_f32(xb[i + 1]) * rcp;
                uint8_t c0 = oracle_e2m1_encode(q0), c1 = oracle_e2m1_encode(q1);
                codes[(size_t)r * (k / 2) + (size_t)b * 8 + i / 2] = (uint8_t)(c0 | (c1 << 4));
            }
        }
    }
}

/* Dequantize NVFP4 (Eq. 2, "Dequant: X^ = X_q * s"): x^ = dec(code) *
 * fl(dec(s_b) * g), returned in fp64 (the product is exact in fp64). */
void oracle_nvfp4_dequantize(const uint8_t* codes, const uint8_t* sf, int m, int k,
                             float g, double* out) {
    for (int r = 0; r < m; ++r)
        for (int j = 0; j < k; ++j) {
            uint8_t byte = codes[(size_t)r * (k / 2) + j / 2];
            uint8_t nib = (j & 1) ? (byte >> 4) : (byte & 15);
            float eff = (float)oracle_e4m3_decode(sf[(size_t)r * (k / 16) + j / 16]) * g;
            out[(size_t)r * k + j] = oracle_e2m1_decode(nib) * (double)eff;
        }
}

/* Global (per-tensor) scale of reading R3: g = max(fl(amax / div), FLT_MIN).
 * div = 6*448 = 2688 for a tensor's own amax (weights; standalone layer sweep),
 * div = 1344 (x2 headroom) for the delayed policy (amax of the same activation
 * at t-1). */
float oracle_global_scale(float amax, float div) {
    float g = amax / div;
    return g < FLT_MIN ? FLT_MIN : g;
}

/* The swizzled device layout of the block scales (reading R6): byte offset of
 * scale (row r, scale-column c) for a K/16-column scale matrix. Rows padded to
 * 128, scale columns padded to a multiple of 4; 128x4 "atoms" of 512 bytes laid
 * out K-fastest.  This is the layout the tcgen05 block-scaled MMA consumes. */
long long oracle_sf_offset(int r, int c, int k) {
    int kc = ((k / 16) + 3) / 4 * 4;
    return ((long long)(r / 128) * (kc / 4) + c / 4) * 512 + (r % 32) * 16 + ((r % 128) / 32) * 4 + (c % 4);
}

/* ------------------------------------------------------------------------ */
/* Online block Hadamard smoothing ("we apply a Fast Hadamard Transform  */
/* (FHT) over local activation blocks (B=128)").  Reading R14: the   */
/* Sylvester-ordered transform y = H_128 x per 128-block (entries +-1, no       */
/* normalization on the activation side), evaluated as the fast transform in   */
/* FP32 exactly in this order: stages h = 1, 2, 4, ..., 64; within a stage     */
/* every pair (i, i+h) with (i & h) == 0 becomes (fl(a + b), fl(a - b)).  The   */
/* normalization H^T H = 128 I is carried by the weights as the exact power of  */
/* two 2^-7 (oracle_pack_weights_hadamard), so (H x) . (2^-7 H w) = x . w.     */
/* ------------------------------------------------------------------------ */

void oracle_fht128_f32(const float* x, float* y, long long n) {
    for (long long b0 = 0; b0 < n; b0 += 128) {
        float v[128];
        for (int i = 0; i < 128; ++i) v[i] = x[b0 + i];
        for (int h = 1; h < 128; h <<= 1)
            for (int i = 0; i < 128; ++i)
                if ((i & h) == 0) {
                    float a = v[i], b = v[i + h];
                    v[i] = a + b;
                    v[i + h] = a - b;
                }
        for (int i = 0; i < 128; ++i) y[b0 + i] = v[i];
    }
}

/* NVFP4 quantization of FP32 rows (the Hadamard-smoothed path): identical steps to
 * oracle_nvfp4_quantize, the inputs being fp32 values instead of bf16 ones. */
void oracle_nvfp4_quantize_f32(const float* x, int m, int k, float g, uint8_t* codes, uint8_t* sf) {
    for (int r = 0; r < m; ++r) {
        for (int b = 0; b < k / 16; ++b) {
            const float* xb = x + (size_t)r * k + (size_t)b * 16;
            float a_b = 0.0f;
            for (int i = 0; i < 16; ++i)
                if (fabsf(xb[i]) > a_b) a_b = fabsf(xb[i]);
            float raw = (a_b / 6.0f) / g;
            uint8_t s_b = oracle_e4m3_encode_nonneg(raw);
            float eff = (float)oracle_e4m3_decode(s_b) * g;
            float rcp = eff > 0.0f ? 1.0f / eff : 0.0f;
            sf[(size_t)r * (k / 16) + b] = s_b;
            for (int i = 0; i < 16; i += 2) {
                uint8_t c0 = oracle_e2m1_encode(xb[i] * rcp), c1 = oracle_e2m1_encode(xb[i + 1] * rcp);
                codes[(size_t)r * (k / 2) + (size_t)b * 8 + i / 2] = (uint8_t)(c0 | (c1 << 4));
            }
        }
    }
}

/* Per-token symmetric INT8 of FP32 rows (same steps as oracle_int8_quantize_rows). */
void oracle_int8_quantize_rows_f32(const float* x, int m, int k, int8_t* codes, float* scale) {
    for (int r = 0; r < m; ++r) {
        const float* xr = x + (size_t)r * k;
        float a = 0.0f;
        for (int j = 0; j < k; ++j)
            if (fabsf(xr[j]) > a) a = fabsf(xr[j]);
        if (a == 0.0f) {
            scale[r] = 1.0f;
            for (int j = 0; j < k; ++j) codes[(size_t)r * k + j] = 0;
            continue;
        }
        scale[r] = a / 127.0f;
        float rcp = 127.0f / a;
        for (int j = 0; j < k; ++j) {
            double rq = nearbyint((double)(xr[j] * rcp));
            if (rq > 127.0) rq = 127.0;
            if (rq < -128.0) rq = -128.0;
            codes[(size_t)r * k + j] = (int8_t)rq;
        }
    }
}

/* Per-block symmetric INT8 of FP32 rows (after the block Hadamard, activations are
 * quantized "using either the NVFP4 format or per-block symmetric INT8"; NEXT-1). Reading R17:
 * the blocks are the B = 128 consecutive elements of a row along K that one Hadamard block
 * covers; each block is quantized exactly as a per-token row is (Eq. 1 with z = 0, R4):
 *   a = max|x| over the block;  a == 0: s = 1, codes 0;
 *   else s = fl(a / 127), code = clip(RNE(fl(x * fl(127 / a))), -128, 127).
 * scale is [m x k/B], row-major. */
void oracle_int8_quantize_blocks_f32(const float* x, int m, int k, int B, int8_t* codes, float* scale) {
    for (int r = 0; r < m; ++r)
        for (int b = 0; b < k / B; ++b) {
            const float* xb = x + (size_t)r * k + (size_t)b * B;
            int8_t* cb = codes + (size_t)r * k + (size_t)b * B;
            float a = 0.0f;
            for (int j = 0; j < B; ++j)
                if (fabsf(xb[j]) > a) a = fabsf(xb[j]);
            if (a == 0.0f) {
                scale[(size_t)r * (k / B) + b] = 1.0f;
                for (int j = 0; j < B; ++j) cb[j] = 0;
                continue;
            }
            scale[(size_t)r * (k / B) + b] = a / 127.0f;
            float rcp = 127.0f / a;
            for (int j = 0; j < B; ++j) {
                double rq = nearbyint((double)(xb[j] * rcp));
                if (rq > 127.0) rq = 127.0;
                if (rq < -128.0) rq = -128.0;
                cb[j] = (int8_t)rq;
            }
        }
}

/* GEMM over per-block INT8 activations (R17): each K block's integer dot product is exact,
 *   acc_b[m][n] = sum_{k in block b} a * w  (int64),
 * and the block scales multiply it in exact FP64 (|acc_b| < 2^22, s_a a float: exact product):
 *   Y64 = (sum_b acc_b * s_a[m][b]) * s_w[n] + bias[n]   (FP64 sum over b in order). */
void oracle_gemm_int8_blocks(const int8_t* a, const float* s_a, int B, const int8_t* w, const float* s_w,
                             const float* bias, int m, int n, int k, int row0, int row1, double* y_out) {
    (void)m;
    const int nbk = k / B;
    for (int i = row0; i < row1; ++i)
        for (int j = 0; j < n; ++j) {
            double t = 0.0;
            for (int b = 0; b < nbk; ++b) {
                int64_t acc = 0;
                for (int e = b * B; e < (b + 1) * B; ++e)
                    acc += (int64_t)a[(size_t)i * k + e] * (int64_t)w[(size_t)j * k + e];
                t += (double)acc * (double)s_a[(size_t)i * nbk + b];
            }
            double y = t * (double)s_w[j];
            if (bias) y += (double)bias[j];
            y_out[(size_t)(i - row0) * n + j] = y;
        }
}

/* ------------------------------------------------------------------------ */
/* Symmetric INT8: "maps values to [-128, 127] with s = max(|X|)/127",  */
/* Eq. 1 with z = 0: X_q = clip(round(X/s), -128, 127).  Granularity: one scale */
/* per token (row), reading R2.  X/s evaluated as fl(x * fl(127/a)) (R4);       */
/* round = half to even.  All-zero row: s = 1, codes 0.                */
/* ------------------------------------------------------------------------ */

void oracle_int8_quantize_rows(const uint16_t* x, int m, int k, int ldx,
                               int8_t* codes, float* scale) {
    for (int r = 0; r < m; ++r) {
        const uint16_t* xr = x + (size_t)r * ldx;
        float a = 0.0f;
        for (int j = 0; j < k; ++j) {
            float v = fabsf(oracle_bf16_to_f32(xr[j]));
            if (v > a) a = v;
        }
        if (a == 0.0f) {
            scale[r] = 1.0f;
            for (int j = 0; j < k; ++j) codes[(size_t)r * k + j] = 0;
            continue;
        }
        scale[r] = a / 127.0f;
        float rcp = 127.0f / a;
        for (int j = 0; j < k; ++j) {
            float q = oracle_bf16_to_f32(xr[j]) * rcp;
            double rq = nearbyint((double)q);   /* default rounding mode: half to even */
            if (rq > 127.0) rq = 127.0;
            if (rq < -128.0) rq = -128.0;
            codes[(size_t)r * k + j] = (int8_t)rq;
        }
    }
}

/* ------------------------------------------------------------------------ */
/* Weight packing: "all weights are quantized to NVFP4 offline ... if a  */
/* layer's A_bits is routed to INT8, its corresponding weights are cast to INT8 */
/* on-the-fly".  Reading R7: both forms are pre-packed; the INT8 form is the     */
/* symmetric per-output-channel INT8 quantization of the DEQUANTIZED NVFP4      */
/* weights: W^ = fl32(dec(code) * eff);  s_w[n] = fl(max|W^_n|/127);           */
/* code = RNE(fl(W^ * fl(127/max))).                                            */
/* W: bf16 [n x k] (nn.Linear layout).                                         */
/* ------------------------------------------------------------------------ */

void oracle_pack_weights(const uint16_t* w, int n, int k,
                         uint8_t* fp4_codes, uint8_t* fp4_sf, float* fp4_g,
                         int8_t* i8_codes, float* i8_scale) {
    float amax = 0.0f;
    for (size_t i = 0; i < (size_t)n * k; ++i) {
        float v = fabsf(oracle_bf16_to_f32(w[i]));
        if (v > amax) amax = v;
    }
    float g = oracle_global_scale(amax, 2688.0f);
    *fp4_g = g;
    oracle_nvfp4_quantize(w, n, k, k, g, fp4_codes, fp4_sf);
    for (int r = 0; r < n; ++r) {
        float a = 0.0f;
        for (int j = 0; j < k; ++j) {
            uint8_t byte = fp4_codes[(size_t)r * (k / 2) + j / 2];
            uint8_t nib = (j & 1) ? (byte >> 4) : (byte & 15);
            float eff = (float)oracle_e4m3_decode(fp4_sf[(size_t)r * (k / 16) + j / 16]) * g;
            float wh = (float)oracle_e2m1_decode(nib) * eff;
            if (fabsf(wh) > a) a = fabsf(wh);
        }
        if (a == 0.0f) {
            i8_scale[r] = 1.0f;
            for (int j = 0; j < k; ++j) i8_codes[(size_t)r * k + j] = 0;
            continue;
        }
        i8_scale[r] = a / 127.0f;
        float rcp = 127.0f / a;
        for (int j = 0; j < k; ++j) {
            uint8_t byte = fp4_codes[(size_t)r * (k / 2) + j / 2];
            uint8_t nib = (j & 1) ? (byte >> 4) : (byte & 15);
            float eff = (float)oracle_e4m3_decode(fp4_sf[(size_t)r * (k / 16) + j / 16]) * g;
            float wh = (float)oracle_e2m1_decode(nib) * eff;
            double rq = nearbyint((double)(wh * rcp));
            if (rq > 127.0) rq = 127.0;
            if (rq < -128.0) rq = -128.0;
            i8_codes[(size_t)r * k + j] = (int8_t)rq;
        }
    }
}

/* Weight pack with the offline Hadamard rotation (reading R14): every row of W
 * (nn.Linear [n x k]) gets the same block FHT along k as the activations, times the
 * exact power of two 2^-7 = 1/128, so (H x) . (2^-7 H w) = x . w; then the two packed
 * forms of oracle_pack_weights from the rotated FP32 weights (g_w from their amax). */
void oracle_pack_weights_hadamard(const uint16_t* w, int n, int k,
                                  uint8_t* fp4_codes, uint8_t* fp4_sf, float* fp4_g,
                                  int8_t* i8_codes, float* i8_scale, float* w_rot /* [n x k] scratch/out */) {
    for (size_t i = 0; i < (size_t)n * k; ++i) w_rot[i] = oracle_bf16_to_f32(w[i]);
    oracle_fht128_f32(w_rot, w_rot, (long long)n * k);
    for (size_t i = 0; i < (size_t)n * k; ++i) w_rot[i] = w_rot[i] * 0.0078125f;   /* 2^-7, exact */
    float amax = 0.0f;
    for (size_t i = 0; i < (size_t)n * k; ++i)
        if (fabsf(w_rot[i]) > amax) amax = fabsf(w_rot[i]);
    float g = oracle_global_scale(amax, 2688.0f);
    *fp4_g = g;
    oracle_nvfp4_quantize_f32(w_rot, n, k, g, fp4_codes, fp4_sf);
    for (int r = 0; r < n; ++r) {
        float a = 0.0f;
        float* wr = w_rot + (size_t)r * k;  /* reuse the scratch for W^ of this row */
        for (int j = 0; j < k; ++j) {
            uint8_t byte = fp4_codes[(size_t)r * (k / 2) + j / 2];
            uint8_t nib = (j & 1) ? (byte >> 4) : (byte & 15);
            float eff = (float)oracle_e4m3_decode(fp4_sf[(size_t)r * (k / 16) + j / 16]) * g;
            wr[j] = (float)oracle_e2m1_decode(nib) * eff;
            if (fabsf(wr[j]) > a) a = fabsf(wr[j]);
        }
        (void)a;
    }
    oracle_int8_quantize_rows_f32(w_rot, n, k, i8_codes, i8_scale);
}

/* ------------------------------------------------------------------------ */
/* GEMMs ("GEMM data type requirements"; north_star: dequant/bias       */
/* epilogue).  Rows [row0, row1) only, so a caller may sample rows.           */
/* ------------------------------------------------------------------------ */

/* INT8: acc[m][n] = sum_k a*w exactly (int64, then checked to fit int32);
 * Y = fma(fl(float(acc) * s_a[m]), s_w[n], bias[n])  (reading R8: the per-token
 * scale, then the per-channel scale fused with the bias; without bias the last
 * step is fl(. * s_w[n])). */
int oracle_gemm_int8(const int8_t* a, const float* s_a, const int8_t* w, const float* s_w,
                     const float* bias, int m, int n, int k, int row0, int row1,
                     int32_t* acc_out, float* y_out) {
    int overflow = 0;
    for (int i = row0; i < row1; ++i)
        for (int j = 0; j < n; ++j) {
            int64_t acc = 0;
            for (int t = 0; t < k; ++t)
                acc += (int64_t)a[(size_t)i * k + t] * (int64_t)w[(size_t)j * k + t];
            if (acc > INT32_MAX || acc < INT32_MIN) overflow = 1;
            size_t o = (size_t)(i - row0) * n + j;
            if (acc_out) acc_out[o] = (int32_t)acc;
            float y = (float)acc * s_a[i];
            y = bias ? fmaf(y, s_w[j], bias[j]) : y * s_w[j];
            if (y_out) y_out[o] = y;
        }
    (void)m;
    return overflow;
}

/* NVFP4: Y64 = sum_k (dec(a)*dec(sfa)) * (dec(w)*dec(sfw))  in fp64 (each
 * product is exact), then Y = Y64 * fl(g_a * g_w) + bias  (fp64 result).
 * The per-block E4M3 scales multiply inside the sum; the per-tensor FP32 scales
 * factor out of it (reading R3). sfa/sfw are LOGICAL [rows x k/16]. */
void oracle_gemm_nvfp4(const uint8_t* a_codes, const uint8_t* a_sf, float g_a,
                       const uint8_t* w_codes, const uint8_t* w_sf, float g_w,
                       const float* bias, int m, int n, int k, int row0, int row1,
                       double* y_out) {
    float gg = g_a * g_w;
    (void)m;
    for (int i = row0; i < row1; ++i)
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int t = 0; t < k; ++t) {
                uint8_t ab = a_codes[(size_t)i * (k / 2) + t / 2];
                uint8_t wb = w_codes[(size_t)j * (k / 2) + t / 2];
                double av = oracle_e2m1_decode((t & 1) ? (ab >> 4) : (ab & 15)) *
                            oracle_e4m3_decode(a_sf[(size_t)i * (k / 16) + t / 16]);
                double wv = oracle_e2m1_decode((t & 1) ? (wb >> 4) : (wb & 15)) *
                            oracle_e4m3_decode(w_sf[(size_t)j * (k / 16) + t / 16]);
                acc += av * wv;
            }
            double y = acc * (double)gg;
            if (bias) y += (double)bias[j];
            y_out[(size_t)(i - row0) * n + j] = y;
        }
}

/* BF16 full-precision fallback GEMM ("uses full precision (FP16/BF16)",
 * reading R15): Y = sum_k x*w + bias with bf16 x, w, in fp64 (bf16 products are exact). */
void oracle_gemm_bf16(const uint16_t* x, const uint16_t* w, const float* bias, int m, int n, int k,
                      int row0, int row1, double* y_out) {
    (void)m;
    for (int i = row0; i < row1; ++i)
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int t = 0; t < k; ++t)
                acc += (double)oracle_bf16_to_f32(x[(size_t)i * k + t]) * (double)oracle_bf16_to_f32(w[(size_t)j * k + t]);
            if (bias) acc += (double)bias[j];
            y_out[(size_t)(i - row0) * n + j] = acc;
        }
}

/* Outlier ratio of the Purified Cache Refresh gate: R = max|X| / mean|X|
 * over every `stride`-th element (stride 1 = exact). An all-zero sample has
 * ratio 1. */
double oracle_outlier_ratio(const uint16_t* x, long long count, long long stride) {
    double mx = 0.0;
    long double s = 0.0L;
    long long n = 0;
    for (long long i = 0; i < count; i += stride) {
        double v = fabs((double)oracle_bf16_to_f32(x[i]));
        if (v > mx) mx = v;
        s += v;
        ++n;
    }
    if (s == 0.0L) return 1.0;
    return mx / (double)(s / (long double)n);
}

/* ------------------------------------------------------------------------ */
/* Block statistics for the predictor and TDC (one pass definitions).          */
/*   d_i = fl32(y_i - x_i)                         (Eq. 8: X_out = X_in + Delta) */
/*   Delta_new_i = bf16(d_i)                       (cached delta)         */
/*   st[0] = sum |d|        st[1] = sum |x|        (Eq. 3 numerator/denominator) */
/*   st[2] = sum d^2        st[3] = sum x^2        (L2 variant, reading R1)     */
/*   st[4] = sum Dn*Dp      st[5] = sum Dn^2   st[6] = sum Dp^2  (Eq. 9, cosine) */
/* Sums in long double (x87 80-bit) — an accuracy margin over the device's     */
/* fp64 accumulation.  delta_prev may be NULL (then st[4..6] use zeros).        */
/* ------------------------------------------------------------------------ */

void oracle_block_stats(const uint16_t* x_in, const uint16_t* x_out, const uint16_t* delta_prev,
                        long long count, uint16_t* delta_new, double* st) {
    long double s[7] = {0, 0, 0, 0, 0, 0, 0};
    for (long long i = 0; i < count; ++i) {
        float x = oracle_bf16_to_f32(x_in[i]);
        float y = oracle_bf16_to_f32(x_out[i]);
        float d = y - x;
        uint16_t dn = oracle_f32_to_bf16(d);
        if (delta_new) delta_new[i] = dn;
        long double dnv = oracle_bf16_to_f32(dn);
        long double dpv = delta_prev ? oracle_bf16_to_f32(delta_prev[i]) : 0.0L;
        s[0] += fabsl((long double)d);
        s[1] += fabsl((long double)x);
        s[2] += (long double)d * (long double)d;
        s[3] += (long double)x * (long double)x;
        s[4] += dnv * dpv;
        s[5] += dnv * dnv;
        s[6] += dpv * dpv;
    }
    for (int j = 0; j < 7; ++j) st[j] = (double)s[j];
}

/* TDC skip: X_out = X_in + Delta_{t_p}, evaluated as
 * bf16(fl32(x + delta)). */
void oracle_tdc_skip(const uint16_t* x_in, const uint16_t* delta, long long count, uint16_t* x_out) {
    for (long long i = 0; i < count; ++i)
        x_out[i] = oracle_f32_to_bf16(oracle_bf16_to_f32(x_in[i]) + oracle_bf16_to_f32(delta[i]));
}

/* tensor amax: max |x| (feeds the delayed global scale of reading R3) */
float oracle_amax_bf16(const uint16_t* x, long long count) {
    float a = 0.0f;
    for (long long i = 0; i < count; ++i) {
        float v = fabsf(oracle_bf16_to_f32(x[i]));
        if (v > a) a = v;
    }
    return a;
}

/* ------------------------------------------------------------------------ */
/* NVFP4-compressed delta cache ("Caching these residual deltas        */
/* introduces only a small memory overhead, as they can be quantized to ultra- */
/* low precision formats such as NVFP4"; SPEC S:330 cache_compress = nvfp4,    */
/* S:365).  Reading R16: the cache of a block holds NVFP4(d) of the     */
/* FP32 delta d = fl(y - x) of its last compute, quantized exactly as the      */
/* FP32-input activation quantizer (oracle_nvfp4_quantize_f32, Eq. 2 with the  */
/* two-level scale) with the cache's global scale g; codes [m x h/2] (element  */
/* 2i in the low nibble), E4M3 scales [m x h/16] plain row-major.  The cached   */
/* value it stands for is dq = fl(dec(code) * eff), eff = fl(dec(s_b) * g).     */
/* ------------------------------------------------------------------------ */

/* dq of every element of a compressed cache (FP32, one rounding per element) */
void oracle_cache_dequant(const uint8_t* codes, const uint8_t* sf, float g, long long count, float* out) {
    for (long long i = 0; i < count; ++i) {
        uint8_t byte = codes[i / 2];
        uint8_t nib = (i & 1) ? (byte >> 4) : (byte & 15);
        float eff = (float)oracle_e4m3_decode(sf[i / 16]) * g;
        out[i] = (float)oracle_e2m1_decode(nib) * eff;
    }
}

/* TDC skip with the compressed cache ("X_out = X_in + Delta_tp"):
 * x_out = bf16(fl(x + dq)). */
void oracle_tdc_skip_nvfp4(const uint16_t* x_in, const uint8_t* codes, const uint8_t* sf, float g,
                           long long count, uint16_t* x_out) {
    for (long long i = 0; i < count; ++i) {
        uint8_t byte = codes[i / 2];
        uint8_t nib = (i & 1) ? (byte >> 4) : (byte & 15);
        float eff = (float)oracle_e4m3_decode(sf[i / 16]) * g;
        float dq = (float)oracle_e2m1_decode(nib) * eff;
        x_out[i] = oracle_f32_to_bf16(oracle_bf16_to_f32(x_in[i]) + dq);
    }
}

/* Refresh with the compressed cache: the statistics of oracle_block_stats with the
 * previous delta Dp = dq of the cache as it stands (g_prev), then the cache is
 * rewritten with NVFP4(d; g_new) (h % 16 == 0 elements per row) and amax = max |d|. */
void oracle_block_stats_nvfp4(const uint16_t* x_in, const uint16_t* x_out, const uint8_t* codes_prev,
                              const uint8_t* sf_prev, float g_prev, int m, int h, float g_new,
                              uint8_t* codes_new, uint8_t* sf_new, double* st, float* amax) {
    long long count = (long long)m * h;
    long double s[7] = {0, 0, 0, 0, 0, 0, 0};
    float a = 0.0f;
    float d[16];
    for (long long r = 0; r < m; ++r) {
        for (int b = 0; b < h / 16; ++b) {
            long long i0 = r * h + (long long)b * 16;
            for (int i = 0; i < 16; ++i) {
                long long e = i0 + i;
                float x = oracle_bf16_to_f32(x_in[e]);
                float y = oracle_bf16_to_f32(x_out[e]);
                d[i] = y - x;
                uint8_t byte = codes_prev[e / 2];
                uint8_t nib = (e & 1) ? (byte >> 4) : (byte & 15);
                float eff = (float)oracle_e4m3_decode(sf_prev[e / 16]) * g_prev;
                long double dpv = (float)oracle_e2m1_decode(nib) * eff;
                long double dnv = oracle_bf16_to_f32(oracle_f32_to_bf16(d[i]));
                s[0] += fabsl((long double)d[i]);
                s[1] += fabsl((long double)x);
                s[2] += (long double)d[i] * (long double)d[i];
                s[3] += (long double)x * (long double)x;
                s[4] += dnv * dpv;
                s[5] += dnv * dnv;
                s[6] += dpv * dpv;
                if (fabsf(d[i]) > a) a = fabsf(d[i]);
            }
        }
    }
    /* the previous cache is fully read above before it is overwritten */
    for (long long r = 0; r < m; ++r) {
        float row[h];
        for (int j = 0; j < h; ++j)
            row[j] = oracle_bf16_to_f32(x_out[r * h + j]) - oracle_bf16_to_f32(x_in[r * h + j]);
        oracle_nvfp4_quantize_f32(row, 1, h, g_new, codes_new + r * (h / 2), sf_new + r * (h / 16));
    }
    (void)count;
    for (int j = 0; j < 7; ++j) st[j] = (double)s[j];
    *amax = a;
}
