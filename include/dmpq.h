/*
 * dmpq.h — C ABI of libdmpq: the B200 (sm_100a) hot path of 6Bit-Diffusion
 * (arxiv 2603.18742): Dynamic Mixed-Precision Quantization (DMPQ, §4.1)
 * and the Temporal Delta Cache (TDC, §4.2).
 *
 * Citations: P:<line> = PAPER.md line (the method's authority); Rn = reading n
 * of DESIGN.md §3 (where the paper is silent or ambiguous).
 *
 * Conventions (all entry points)
 *  - Every buffer is caller-owned. The library never allocates device memory and
 *    never synchronises the device, except the host-pure helpers, which touch no
 *    device state at all.
 *  - Device work is enqueued on the caller's stream `s` (a cudaStream_t; NULL =
 *    legacy default stream). Arguments are validated synchronously, before
 *    anything is enqueued; a validation failure returns a status and enqueues
 *    nothing. Device faults are asynchronous and surface at the caller's next
 *    synchronisation.
 *  - No exceptions cross the ABI. dmpq_last_error() describes the most recent
 *    non-OK status of the calling thread.
 *  - bf16 tensors are passed as `const uint16_t*` (their bit patterns), row
 *    major. Device pointers must be 16-byte aligned and leading dimensions
 *    multiples of 8 elements (DMPQ_EALIGN otherwise).
 *  - Inputs must not alias outputs, except where stated (tdc_step SKIP).
 *  - Stateless and re-entrant: calls on different streams may run concurrently.
 */
#ifndef DMPQ_H_
#define DMPQ_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#pragma GCC visibility push(default) /* the ABI is the only exported surface of libdmpq */
#endif
#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* dmpq_stream_t; /* == cudaStream_t */

typedef enum {
    DMPQ_OK = 0,
    DMPQ_EINVAL = 1,       /* bad argument (NULL pointer, unknown enum, ...)      */
    DMPQ_ESHAPE = 2,       /* unsupported or inconsistent dimensions              */
    DMPQ_EALIGN = 3,       /* pointer / leading dimension alignment                */
    DMPQ_EZERONORM = 4,    /* Eq. 3 undefined (||X||_1 == 0): routed INT8         */
    DMPQ_ECUDA = 5,        /* a CUDA runtime call failed (launch, attribute, ...) */
    DMPQ_EUNSUPPORTED = 6  /* no sm_100a device / feature not built               */
} dmpq_status;

/* Activation precision of one linear layer: Eq. 7 routes INT8 / NVFP4;
 * the Purified Cache Refresh outlier gate (R15) routes BF16 (unquantised). */
typedef enum { DMPQ_FMT_INT8 = 0, DMPQ_FMT_NVFP4 = 1, DMPQ_FMT_BF16 = 2 } dmpq_fmt;

const char* dmpq_last_error(void);
const char* dmpq_version(void);

/* Set the per-kernel launch attributes (dynamic shared memory) on the current device
 * ahead of time, so that later calls may be captured into CUDA graphs. Optional:
 * every call sets what it needs on first use. */
dmpq_status dmpq_prepare(void);

/* ========================================================================== */
/* Sizing helpers                                                             */
/* ========================================================================== */

/* Bytes of an NVFP4 block-scale buffer for a [rows x k] tensor in the device
 * ("swizzled") layout consumed by the tcgen05 block-scaled MMA (R6): one E4M3
 * byte per 16 elements, rows padded to a multiple of 128, scale columns to a
 * multiple of 4, in 512-byte atoms of 128 rows x 4 scales, K-fastest. Byte of
 * (row r, scale column c) = ((r/128)*(Kc/4) + c/4)*512 + (r%32)*16 +
 * ((r%128)/32)*4 + c%4 with Kc = ceil(k/16 / 4)*4. */
size_t dmpq_sf_bytes(int rows, int k);

/* Workspace bytes tdc_step(REFRESH) needs for its deterministic two-stage
 * reduction of an [m x h] tensor. */
size_t tdc_workspace_bytes(int m, int h);

/* ========================================================================== */
/* Packed operands                                                            */
/* ========================================================================== */

/* Offline weight pack of one linear layer, P:184 ("all weights are quantized to
 * NVFP4 offline"; INT8 weights for INT8-routed layers), reading R7: both forms
 * are pre-packed; the INT8 form is the per-output-channel symmetric INT8
 * quantization of the DEQUANTIZED NVFP4 weights. All pointers are device memory
 * owned by the caller. */
typedef struct {
    int n, k;              /* out_features, in_features (nn.Linear W is [n x k]) */
    uint8_t* fp4_codes;    /* [n x k/2]: E2M1 nibbles, element 2i in the low nibble */
    uint8_t* fp4_sf;       /* dmpq_sf_bytes(n, k): E4M3 block scales, device layout */
    float* fp4_g;          /* [1]: FP32 per-tensor scale g_w = max(amax/2688, FLT_MIN) */
    int8_t* i8_codes;      /* [n x k] */
    float* i8_scale;       /* [n]: per-output-channel scale */
    const float* bias;     /* [n] or NULL (may point at caller memory) */
    const uint16_t* bf16_w;/* [n x k] original bf16 weights for the BF16 fallback (R15), or NULL */
    const float* fp4_g_col;/* [n] per-output-column g_w, or NULL (fp4_g for every column): several
                              layers packed side by side along n (e.g. Q, K, V over the same input)
                              keep their own per-tensor scales; the NVFP4 epilogue then uses
                              fl(g_a * fp4_g_col[n]) per column, bit-identical to separate GEMMs */
    float* i8_rcp;         /* [n] or NULL: r_w[n] = fl(127 / max_k|W^|) (0 for a zero row), written by the
                              pack when non-NULL; lets dmpq_cast_int8 rebuild the INT8 codes on the fly */
} dmpq_weights;

/* A quantized activation tensor, as written by dmpq_quantize_act. */
typedef struct {
    dmpq_fmt fmt;
    int m, k;
    void* codes;           /* NVFP4: uint8 [m x k/2]; INT8: int8 [m x k]; BF16: the bf16 activation [m x k] (row-major, dense) */
    uint8_t* sf;           /* NVFP4: dmpq_sf_bytes(m, k) block scales; INT8: unused */
    const float* g;        /* NVFP4: device FP32 per-tensor scale g_a (input of the quantizer) */
    float* row_scale;      /* INT8: [m] per-token scale s = amax_row/127 (R2), or with scale_block == 128:
                              [m x k/128] per-block scales s = amax_block/127, row-major (R17) */
    int scale_block;       /* INT8: 0 = per-token (R2); 128 = per-block symmetric INT8 over the 128-element
                              Hadamard blocks (R17; needs DMPQ_QF_HADAMARD in the quantizer) */
} dmpq_act;

/* ========================================================================== */
/* 1. dmpq_pack_weights                                                       */
/* ========================================================================== */

/* Quantize W (bf16 [n x k], row stride k) into both packed forms (R7):
 *   g_w = max(fl(amax(W)/2688), FLT_MIN);
 *   NVFP4 codes/scales per Eq. 2 with that g (see dmpq_quantize_act);
 *   W^ = fl(dec(code) * fl(dec(s_b) * g_w)),  s_w[n] = fl(max_k|W^|/127),
 *   i8 = RNE(fl(W^ * fl(127/max_k|W^|)))   (s_w = 1, codes 0 for a zero row).
 * `out` holds the caller's buffers; out->n, out->k must equal n, k.
 * Shapes: k % 64 == 0, n % 16 == 0, n, k > 0. */
dmpq_status dmpq_pack_weights(const uint16_t* W, int n, int k, dmpq_weights* out, dmpq_stream_t s);

#define DMPQ_PACK_HADAMARD 1u  /* rotate every row by the block FHT first (offline half of P:187's smoothing, R14) */

/* With out->i8_rcp != NULL the pack also writes r_w; out->i8_codes may then be NULL (NVFP4-only
 * residency: the INT8 form is rebuilt per GEMM by dmpq_cast_int8). out->i8_scale is always written. */

/* On-the-fly NVFP4 -> INT8 weight cast ("all weights are quantized to NVFP4 offline ... for
 * layers routed to INT8, the NVFP4 weights are cast to INT8 on-the-fly"; R7, NEXT-4b): writes the
 * INT8 codes of W into i8_out (device, [W->n x W->k], row-major, caller-owned scratch, 16-byte
 * aligned) from W's NVFP4 codes / scales / g_w and r_w (W->i8_rcp, from the pack):
 *   i8[n][k] = RNE(fl(fl(dec(code) * fl(dec(s_b) * g_w)) * r_w[n]))  (clamped to [-128, 127]),
 * bit-identical to the pre-packed codes dmpq_pack_weights writes. Per-column g_w (fp4_g_col) is
 * honoured. Pair it with W->i8_scale for the INT8 GEMM (a dmpq_weights whose i8_codes = i8_out).
 * One HBM pass: 0.5625 B read + 1 B written per weight. Errors: EINVAL (NULL / no i8_rcp),
 * EALIGN, ESHAPE (k % 64, n % 16). */
dmpq_status dmpq_cast_int8(const dmpq_weights* W, int8_t* i8_out, dmpq_stream_t s);

/* dmpq_pack_weights with options: DMPQ_PACK_HADAMARD packs W~ = 2^-7 W . blockdiag(H_128)
 * (Sylvester, entries +-1; g_w from amax(W~)), so (H x) . W~^T = x . W^T for activations
 * quantised with DMPQ_QF_HADAMARD (R14). k % 128 == 0 then. */
dmpq_status dmpq_pack_weights_ex(const uint16_t* W, int n, int k, uint32_t flags, dmpq_weights* out, dmpq_stream_t s);

/* ========================================================================== */
/* 2. dmpq_predict  (host-pure)                                               */
/* ========================================================================== */

/* Global (all ranks, all tokens) statistics of one block at the end of a step.
 * The device writes them with tdc_step(REFRESH); the sums of Eq. 3 and Eq. 9. */
typedef struct {
    double sum_abs_d;  /* sum |Y - X|    (Eq. 3 numerator)   */
    double sum_abs_x;  /* sum |X|        (Eq. 3 denominator) */
    double sum_d2;     /* sum (Y - X)^2  (L2 variant, R1)     */
    double sum_x2;     /* sum X^2                             */
    double dot_dd;     /* sum Delta_t * Delta_prev  (Eq. 9)   */
    double sum_dn2;    /* sum Delta_t^2                       */
    double sum_dp2;    /* sum Delta_prev^2                    */
} dmpq_block_stats;
#define DMPQ_STATS_LEN 7

typedef enum { DMPQ_GAMMA_L1 = 0, DMPQ_GAMMA_L2 = 1 } dmpq_gamma_metric;

/* Eq. 6: tau_Gamma = (tau_rel - beta) / alpha; alpha <= eps_slope has no
 * usable inversion and returns -INFINITY, which routes every Gamma to INT8. */
double dmpq_derive_tau(double alpha, double beta, double tau_rel, double eps_slope);

/* Routing of one block's n_layers linear layers for step t (Eq. 7):
 *   Gamma_{t-1} = sum_abs_d / sum_abs_x  (Eq. 3; L2: sqrt(sum_d2)/sqrt(sum_x2)),
 *   fmt_j = INT8  if t == 0 (no Gamma_{t-1}, R9) or prev_skipped (Gamma
 *           missing after a Skip) or Gamma > tau_gamma[j];
 *   fmt_j = NVFP4 otherwise (equality routes NVFP4).
 * `st` is the block's statistics from step t-1 (ignored when t == 0 or
 * prev_skipped). Writes fmt_out[0..n_layers) and *gamma_out (NAN if
 * undefined). Returns DMPQ_EZERONORM, with every layer INT8, when the
 * denominator is 0 and a Gamma was needed. */
dmpq_status dmpq_predict(const dmpq_block_stats* st, const double* tau_gamma, int n_layers, int t,
                         int prev_skipped, dmpq_gamma_metric metric, uint8_t* fmt_out, double* gamma_out);

/* Purified Cache Refresh gate (R15), host-pure, applied after
 * dmpq_predict: for each layer j, ratio[j] > tau_outlier (strict; 25) routes
 * BF16 (no quantization); else prev_skipped routes INT8; else fmt_inout[j] stays.
 * ratio may be NULL (no outlier gate). */
void dmpq_purify(const double* ratio, int n_layers, int prev_skipped, double tau_outlier, uint8_t* fmt_inout);

/* Outlier ratio of the PDR gate ("R_outlier = max|X| / mean|X|"), host-pure:
 * R = max_abs / (sum_abs / count) in FP64; an all-zero input (sum_abs == 0) has R = 1 (no
 * outliers, never BF16). The delayed gate (R15) evaluates it on the all-rank statistics of the
 * block's last computed step. */
double dmpq_outlier_ratio(double max_abs, double sum_abs, double count);

/* ========================================================================== */
/* 3. dmpq_quantize_act                                                       */
/* ========================================================================== */

#define DMPQ_QF_LAYERNORM 1u  /* normalise each row first: h = (x - mean)/sqrt(var + eps), no affine (block glue) */
#define DMPQ_QF_WRITE_H   2u  /* also store the bf16 values that were quantised into h_out (before any rotation) */
#define DMPQ_QF_HADAMARD  4u  /* rotate every 128-element block by the Sylvester FHT (entries +-1, FP32 butterflies)
                                 before quantising (P:187 online block Hadamard, R14); pair with weights packed
                                 with DMPQ_PACK_HADAMARD, which carry the 2^-7 normalization */

typedef struct {
    uint32_t flags;
    float ln_eps;          /* DMPQ_QF_LAYERNORM epsilon (e.g. 1e-6) */
    uint16_t* h_out;       /* DMPQ_QF_WRITE_H: bf16 [m x k], row stride ldh */
    int ldh;
    float* row_abs_sum;    /* optional [m]: sum_k |x| per row of the layer input (after LN, before any
                              rotation), FP32 in a fixed order -- PDR outlier statistics (R15) */
    float* amax_in;        /* optional device scalar: max(*amax_in, max |x|) of that input (R15) */
} dmpq_quant_opts;

/* Online activation quantization of X (bf16 [m x k], row stride ldx) into one or
 * both formats in a single HBM pass.
 *  NVFP4 (Eq. 2, R3/R4), per row and 16-element block b:
 *    a_b = max|x|; s_b = E4M3_rn_satfinite(fl(fl(a_b/6)/g)); eff = fl(dec(s_b)*g);
 *    r = eff > 0 ? fl(1/eff) : 0; code = E2M1_rn_satfinite(fl(x*r)) (sign kept).
 *    g is read from out_fp4->g (device FP32; the delayed policy of R3 sets it to
 *    max(fl(amax_{t-1}/1344), FLT_MIN)). Scale rows in [m, ceil128(m)) are zeroed.
 *  INT8 per token (R2): a = max_k|x|; s = fl(a/127); code =
 *    RNE(fl(x*fl(127/a))); a == 0 gives s = 1 and zero codes.
 *  Either output may be NULL; both may be NULL when opts asks for h_out or the PDR
 *  statistics only (a BF16-routed tensor, R15), or for an amax-only pass (the "current"
 *  global-scale policy, R3: amax first, then g = max(fl(amax/2688), FLT_MIN), then quantize).
 *  out->m/k must equal m/k.
 *  amax_out: if non-NULL, device FP32 that receives max(*amax_out, max|x|)
 *  (atomic; the caller zeroes it once per step). With DMPQ_QF_LAYERNORM the
 *  quantised (and amax'd) values are the bf16-rounded normalised rows.
 *  With DMPQ_QF_HADAMARD the values quantised (and amax'd) are the FP32 FHT outputs
 *  y = H_128 x per 128-block (Sylvester, entries +-1, no normalization on the activation side:
 *  the 2^-7 rides on the Hadamard-packed weights), butterflies h = 1..64 in FP32 (R14).
 *  Shapes: k % 64 == 0 (k % 128 == 0 with DMPQ_QF_HADAMARD), 0 < k <= 16384, m >= 0. */
dmpq_status dmpq_quantize_act(const uint16_t* X, int m, int k, int ldx, const dmpq_quant_opts* opts,
                              dmpq_act* out_i8, dmpq_act* out_fp4, float* amax_out, dmpq_stream_t s);

/* FP64 totals of per-row sums for the PDR outlier ratio (R15): out[s] = sum_r
 * row_sums[s*m + r] for s < segments, fixed order (deterministic). */
dmpq_status dmpq_outlier_reduce(const float* row_sums, int m, int segments, double* out, dmpq_stream_t s);

/* The paper-literal (current-input) PDR gate on the device (reading R18): from the
 * per-row sums |x| (row_abs_sum [m], FP32, as dmpq_quantize_act writes them) and max|x|
 * (*amax_in) of THIS step's layer input, one CTA computes
 *   sum = dmpq_outlier_reduce's FP64 total (same order),  R = dmpq_outlier_ratio(max, sum, count),
 *   *flag_out = R > tau_outlier ? 1 : 0,  *sum_out = sum (if non-NULL),
 * so the GEMMs of that input can be chosen on the device (dmpq_epilogue.run_if) with no host
 * round trip. count = the number of elements the statistics cover (m * k). */
dmpq_status dmpq_outlier_gate(const float* row_abs_sum, int m, const float* amax_in, double count, double tau_outlier,
                              double* sum_out, int* flag_out, dmpq_stream_t s);

/* Device-side global scale for the next NVFP4 quantization (R3):
 * g_out[i] = max(fl(amax[i] / div), FLT_MIN) for i < count (div = 2688 for a
 * tensor's own amax, 1344 for the delayed policy). */
dmpq_status dmpq_global_scale(const float* amax, float div, float* g_out, int count, dmpq_stream_t s);

/* ========================================================================== */
/* 4. dmpq_gemm                                                               */
/* ========================================================================== */

#define DMPQ_EP_BIAS      1u  /* + bias[n] (W->bias)                                   */
#define DMPQ_EP_GELU_TANH 2u  /* y = gelu_tanh(y)  (block glue)                        */
#define DMPQ_EP_RESIDUAL  4u  /* y = residual[m,n] + gate[n] * y (gated residual glue) */
#define DMPQ_EP_TDC_REFRESH 8u /* fused TDC refresh of the stored bf16 Y (= X_out), below */
#define DMPQ_EP_QUANT_NVFP4 16u /* producer-fused NVFP4 quantization of bf16(Y) for the next layer, below */

typedef struct {
    uint32_t flags;
    const float* gate;         /* [n] (DMPQ_EP_RESIDUAL) */
    const uint16_t* residual;  /* bf16 [m x n], row stride ldr (DMPQ_EP_RESIDUAL); may alias Y */
    int ldr;
    /* DMPQ_EP_TDC_REFRESH: tdc_step(TDC_REFRESH, tdc_x_in, Y, tdc_delta, m, n, ...) fused into
     * the epilogue of the GEMM that produces the block output X_out = Y (Eq. 8; SURVEY
     * NEXT-2): Delta_new = bf16(fl(bf16(y) - x_in)) overwrites tdc_delta (Delta_prev on entry)
     * and tdc_stats[0..7) receives the seven dmpq_block_stats sums over the m x n elements, with
     * tdc_step's arithmetic (FP32 per 8-element vector, then FP64; cosine sums exact products in
     * FP64) in a fixed order for a given grid (deterministic; not the same order as tdc_step).
     * Needs the bf16 output Y; tdc_x_in and tdc_delta are dense (row stride n); neither may
     * alias Y or the residual. tdc_workspace: device, dmpq_gemm_tdc_workspace_bytes() bytes,
     * zero-filled once before first use (the kernel leaves it ready for the next call). */
    const uint16_t* tdc_x_in;
    uint16_t* tdc_delta;
    double* tdc_stats;
    void* tdc_workspace;
    /* Device-predicated launch (R18): when run_if != NULL the kernel does nothing unless
     * *run_if == run_if_value (read on the device at kernel start), so a BF16 and a quantized
     * GEMM of one layer can both be enqueued (or captured in one CUDA graph) and the device-side
     * outlier gate (dmpq_outlier_gate) picks the one that runs. */
    const int* run_if;
    int run_if_value;
    /* DMPQ_EP_QUANT_NVFP4 (quantization "fused directly into the preceding layers"; NEXT-2):
     * the epilogue also quantizes the bf16 output it produces, v = bf16(y) after every glue step,
     * to NVFP4 exactly as dmpq_quantize_act does without the Hadamard option (Eq. 2, R3/R4: block
     * scale E4M3(fl(fl(a_b/6)/g)), codes E2M1(fl(v fl(1/eff)))): codes and swizzled scales go to
     * q_out (NVFP4 descriptor with q_out->m == m, q_out->k == n, its g = the consumer's global scale;
     * scale rows m..ceil128(m) are zeroed) and max|v| is max-reduced into *q_amax (device, caller
     * zeroes). Y may then be NULL (the bf16 tensor is not stored). n % 64 == 0. */
    const dmpq_act* q_out;
    float* q_amax;
} dmpq_epilogue;

/* Workspace bytes of the fused TDC refresh (DMPQ_EP_TDC_REFRESH) on the current device. */
size_t dmpq_gemm_tdc_workspace_bytes(void);

/* Y = A @ W^T with the dequant/bias epilogue (north_star), on tcgen05.
 *  BF16  (kind::f16, R15): acc = sum_k a*w in the tensor core's FP32 accumulator;
 *        y = fl(acc + bias[n]); needs W->bf16_w.
 *  INT8  (kind::i8): acc = sum_k a*w exactly in int32 (TMEM);
 *        y = fma(fl(float(acc) * s_a[m]), s_w[n], bias[n])             (R8)
 *  NVFP4 (kind::mxf4nvf4.block_scale.scale_vec::4X): acc = sum_k
 *        (dec(a)*s_a,b)(dec(w)*s_w,b) in the tensor core's FP32 accumulator;
 *        y = fma(acc, fl(g_a*g_w), bias[n])  (one rounding)
 *  then the optional GELU (tanh form, hardware tanh.approx) / gated residual
 *  y = fma(gate[n], y, residual[m,n]) (block glue, tolerance-checked),
 *  stored as bf16 into Y (row stride
 *  ldy) and/or as FP32 into Y32 (row stride n; NULL to skip). acc_or_null
 *  (INT8 only) receives the raw int32 accumulators [m x n] (parity tests).
 *  A->fmt selects the path and must match the packed operand used.
 *  Shapes: A->k == W->k, k % 64 == 0, W->n % 32 == 0, m >= 0. */
dmpq_status dmpq_gemm(const dmpq_act* A, const dmpq_weights* W, const dmpq_epilogue* ep,
                      uint16_t* Y, int ldy, float* Y32, int32_t* acc_or_null, dmpq_stream_t s);

/* ========================================================================== */
/* 5. tdc_step  (+ host-pure TDC helpers)                                      */
/* ========================================================================== */

typedef enum { TDC_SKIP = 0, TDC_REFRESH = 1 } tdc_mode;
typedef enum { TDC_COMPUTE = 0, TDC_DECIDE_SKIP = 1 } tdc_decision;

/* Device part of TDC for one block (Eq. 8):
 *  SKIP:    X_out = bf16(fl(X_in + Delta_{t_p}))  (X_out may alias X_in; Delta is
 *           read from delta_cache; stats/workspace unused, may be NULL).
 *  REFRESH: d = fl(X_out - X_in); Delta_new = bf16(d) overwrites delta_cache
 *           (which held Delta_prev on entry); stats_out[0..7) receives, in FP64
 *           (products exact in FP32, summed per 8-element vector in FP32, then
 *           in FP64, fixed two-stage order: deterministic), the dmpq_block_stats
 *           sums over the m x h elements. X_out is read-only here.
 *  All tensors bf16 [m x h], dense (row stride h). workspace: device,
 *  tdc_workspace_bytes(m, h). */
dmpq_status tdc_step(tdc_mode mode, const uint16_t* X_in, uint16_t* X_out, uint16_t* delta_cache, int m, int h,
                     double* stats_out, void* workspace, dmpq_stream_t s);

/* NVFP4-compressed delta cache of one block ("they can be quantized to ultra-low
 * precision formats such as NVFP4"; SPEC S:330 cache_compress = nvfp4; R16).
 * Caller-owned device buffers; zero-initialise all three before the first refresh. */
typedef struct {
    uint8_t* codes;   /* [m x h/2]  E2M1 codes of the cached delta, element 2i in the low nibble */
    uint8_t* sf;      /* [m x h/16] E4M3 block scales, plain row-major (not the MMA atom layout) */
    float* g;         /* device scalar: the FP32 global scale the cache was written with */
} tdc_nvfp4_cache;

/* tdc_step with the compressed cache (R16). dq = fl(dec(code) * fl(dec(s_b) * g)).
 *  SKIP:    X_out = bf16(fl(X_in + dq))  (X_out may alias X_in; g_new, amax_out,
 *           stats_out and workspace unused, may be NULL).
 *  REFRESH: d = fl(X_out - X_in); statistics as tdc_step(REFRESH) with Delta_new =
 *           bf16(d) and Delta_prev = dq of the cache as it stands on entry; then the
 *           cache is overwritten with NVFP4(d) under the global scale *g_new (the
 *           FP32-input activation quantizer of Eq. 2: a_b, raw = fl(fl(a_b/6)/g),
 *           E4M3, r = fl(1/eff), E2M1(d * r)), *cache->g = *g_new once every CTA has
 *           read the old value, and max|d| is max-reduced into *amax_out (device,
 *           non-negative floats; caller zeroes it). g_new: device scalar, normally the
 *           delayed policy of R3 on the previous refresh's amax (dmpq_global_scale,
 *           div 1344); tdc_delta_amax bootstraps the first refresh.
 *  bf16 tensors [m x h], dense; h % 64 == 0. Memory: 0.5625 B per cached element
 *  instead of 2 (bf16). */
dmpq_status tdc_step_nvfp4(tdc_mode mode, const uint16_t* X_in, uint16_t* X_out, const tdc_nvfp4_cache* cache,
                           const float* g_new, float* amax_out, int m, int h, double* stats_out, void* workspace,
                           dmpq_stream_t s);

/* max |fl(X_out - X_in)| over [m x h] max-reduced into *amax_out (device; caller zeroes
 * it): the current amax that bootstraps a compressed cache's first global scale. */
dmpq_status tdc_delta_amax(const uint16_t* X_in, const uint16_t* X_out, int m, int h, float* amax_out,
                           dmpq_stream_t s);

/* Host-side per-block TDC state. */
typedef struct {
    int t_p;          /* last fully computed step (-1: none)           */
    double e_tp;      /* E_{t_p}: prediction error measured at t_p     */
    double e_acc;     /* E_acc                                         */
    int last;         /* tdc_decision of the previous step (-1: none)  */
    int n_computed;   /* computed deltas so far (warm-up needs two)    */
} tdc_state;

typedef enum { TDC_METRIC_COS = 0, TDC_METRIC_REL_L2 = 1 } tdc_metric;

typedef struct {
    double rho;       /* 0.001 */
    double tau;       /* 0.003 */
    int n_max;        /* 2     */
    int metric;       /* the distance D of Eq. 9: TDC_METRIC_COS = 1 - CosSim (the paper's
                         default, 0 when zero-initialised) or TDC_METRIC_REL_L2 ("relative-L2
                         distance", R19): ||Delta_t - Delta_prev||_2 / ||Delta_prev||_2 */
} tdc_config;

void tdc_init(tdc_state* st);

/* Eq. 11: Skip iff e_acc <= tau and t - t_p <= n_max; the first two
 * computes are forced (Eq. 9 needs two deltas, R10). */
tdc_decision tdc_decide(const tdc_state* st, const tdc_config* cfg, int t);

/* Eq. 10 at the end of step t. After a Compute, `st_global` holds the
 * block's global statistics from tdc_step(REFRESH) and
 * E_{t_p} = 1 - dot_dd / sqrt(sum_dn2 * sum_dp2) (Eq. 9; +INF when a norm
 * is zero or this is the first compute), or with TDC_METRIC_REL_L2
 * E_{t_p} = sqrt(max(sum_dn2 - 2 dot_dd + sum_dp2, 0)) / sqrt(sum_dp2) (+INF when
 * sum_dp2 is zero or this is the first compute); e_acc = E_{t_p}; t_p = t. After a
 * Skip, e_acc = (e_acc + e_tp) + rho (st_global ignored, may be NULL). */
void tdc_update(tdc_state* st, const tdc_config* cfg, int t, tdc_decision d, const dmpq_block_stats* st_global);

#ifdef __cplusplus
}
#endif
#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#endif /* DMPQ_H_ */
