// quant.cu — dmpq_quantize_act: online NVFP4 / per-token INT8 activation
// quantization (Eq. 2; R2-R6), optionally
// with a fused row LayerNorm prologue (block glue), and dmpq_global_scale.
//
// This file holds the entry point (argument validation) and the small reduction kernels;
// the quantizer kernel itself is in quant_tma.cu.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "quant.cuh"

namespace dmpq {

// Deterministic fixed-order FP64 sum of per-row sums: one CTA per segment.
__global__ void __launch_bounds__(256) outlier_reduce_kernel(const float* rows, int m, double* out) {
    __shared__ double red[8];
    const float* r = rows + (size_t)blockIdx.x * m;
    double s = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) s = __dadd_rn(s, (double)r[i]);
    s = warp_sum_d(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = __dadd_rn(t, red[w]);
        out[blockIdx.x] = t;
    }
}

// PDR current-input gate (R18): the outlier_reduce_kernel total (same order), then R and the flag
__global__ void __launch_bounds__(256) outlier_gate_kernel(const float* rows, int m, const float* amax_in, double count,
                                                           double tau, double* sum_out, int* flag_out) {
    __shared__ double red[8];
    double s = 0.0;
    for (int i = threadIdx.x; i < m; i += blockDim.x) s = __dadd_rn(s, (double)rows[i]);
    s = warp_sum_d(s);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = __dadd_rn(t, red[w]);
        if (sum_out) *sum_out = t;
        const double r = t > 0.0 ? __ddiv_rn((double)*amax_in, __ddiv_rn(t, count)) : 1.0;
        *flag_out = r > tau ? 1 : 0;
    }
}

__global__ void global_scale_kernel(const float* amax, float div, float* g_out, int count) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        float g = __fdiv_rn(amax[i], div);
        g_out[i] = g < 1.17549435e-38f ? 1.17549435e-38f : g;
    }
}

}  // namespace dmpq

using namespace dmpq;

extern "C" dmpq_status dmpq_quantize_act(const uint16_t* X, int m, int k, int ldx, const dmpq_quant_opts* opts,
                                         dmpq_act* out_i8, dmpq_act* out_fp4, float* amax_out, dmpq_stream_t s) {
    DMPQ_REQUIRE(out_i8 || out_fp4 || amax_out ||
                     (opts && ((opts->flags & DMPQ_QF_WRITE_H) || opts->row_abs_sum || opts->amax_in)),
                 DMPQ_EINVAL, "dmpq_quantize_act: nothing to produce (no output, amax, h_out or statistics)");
    DMPQ_REQUIRE(m >= 0 && k > 0 && k % 64 == 0 && k <= 16384, DMPQ_ESHAPE,
                 "dmpq_quantize_act: need k %% 64 == 0, 0 < k <= 16384, m >= 0 (m=%d k=%d)", m, k);
    DMPQ_REQUIRE(ldx >= k && ldx % 8 == 0, DMPQ_EALIGN, "dmpq_quantize_act: ldx=%d must be >= k and a multiple of 8", ldx);
    DMPQ_REQUIRE(X && aligned16(X), DMPQ_EALIGN, "dmpq_quantize_act: X must be a 16-byte aligned device pointer");
    if (out_i8) {
        DMPQ_REQUIRE(out_i8->fmt == DMPQ_FMT_INT8 && out_i8->m == m && out_i8->k == k, DMPQ_ESHAPE,
                     "dmpq_quantize_act: INT8 output descriptor mismatch");
        DMPQ_REQUIRE(out_i8->codes && out_i8->row_scale && aligned16(out_i8->codes), DMPQ_EALIGN,
                     "dmpq_quantize_act: INT8 output pointers");
        DMPQ_REQUIRE(out_i8->scale_block == 0 || out_i8->scale_block == 128, DMPQ_EINVAL,
                     "dmpq_quantize_act: INT8 scale_block must be 0 (per token) or 128 (per block)");
        DMPQ_REQUIRE(out_i8->scale_block == 0 || (opts && (opts->flags & DMPQ_QF_HADAMARD)), DMPQ_EUNSUPPORTED,
                     "dmpq_quantize_act: per-block INT8 (scale_block 128) is built for the Hadamard quantizer");
    }
    if (out_fp4) {
        DMPQ_REQUIRE(out_fp4->fmt == DMPQ_FMT_NVFP4 && out_fp4->m == m && out_fp4->k == k, DMPQ_ESHAPE,
                     "dmpq_quantize_act: NVFP4 output descriptor mismatch");
        DMPQ_REQUIRE(out_fp4->codes && out_fp4->sf && out_fp4->g && aligned16(out_fp4->codes) && aligned16(out_fp4->sf),
                     DMPQ_EALIGN, "dmpq_quantize_act: NVFP4 output pointers");
    }
    QuantParams p{};
    p.X = X; p.m = m; p.k = k; p.ldx = ldx;
    p.flags = opts ? opts->flags : 0u;
    DMPQ_REQUIRE(!(p.flags & DMPQ_QF_HADAMARD) || k % 128 == 0, DMPQ_ESHAPE,
                 "dmpq_quantize_act: DMPQ_QF_HADAMARD needs k %% 128 == 0 (k=%d)", k);
    p.ln_eps = opts ? opts->ln_eps : 0.0f;
    if (p.flags & DMPQ_QF_WRITE_H) {
        DMPQ_REQUIRE(opts->h_out && aligned16(opts->h_out) && opts->ldh >= k && opts->ldh % 8 == 0, DMPQ_EALIGN,
                     "dmpq_quantize_act: h_out / ldh");
        p.h_out = opts->h_out; p.ldh = opts->ldh;
    }
    p.i8_codes = out_i8 ? reinterpret_cast<int8_t*>(out_i8->codes) : nullptr;
    p.i8_scale = out_i8 ? out_i8->row_scale : nullptr;
    p.i8_block = out_i8 ? out_i8->scale_block : 0;
    p.fp4_codes = out_fp4 ? reinterpret_cast<uint8_t*>(out_fp4->codes) : nullptr;
    p.fp4_sf = out_fp4 ? out_fp4->sf : nullptr;
    p.g = out_fp4 ? out_fp4->g : nullptr;
    p.amax_out = amax_out;
    p.row_abs_sum = opts ? opts->row_abs_sum : nullptr;
    p.amax_in = opts ? opts->amax_in : nullptr;
    p.kc4 = ((k / 16) + 3) / 4;
    p.m_pad = (m + 127) / 128 * 128;
    if (m == 0) return DMPQ_OK;
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_quantize_act: needs an sm_100 device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    if (p.flags & DMPQ_QF_HADAMARD) {
        // DMPQ_QUANT_HAD_CHUNK=1 selects the previous 64-element-chunk kernel (A/B measurements)
        static const bool chunk = [] { const char* e = getenv("DMPQ_QUANT_HAD_CHUNK"); return e && e[0] == '1'; }();
        if (!chunk || p.i8_block) return launch_quant_had(p, st);
    }
    return launch_quant_tma(p, (p.flags & DMPQ_QF_HADAMARD) != 0, st);
}

extern "C" dmpq_status dmpq_outlier_reduce(const float* row_sums, int m, int segments, double* out, dmpq_stream_t s) {
    DMPQ_REQUIRE(row_sums && out && m >= 0 && segments >= 0, DMPQ_EINVAL, "dmpq_outlier_reduce: bad arguments");
    if (segments == 0) return DMPQ_OK;
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_outlier_reduce: needs an sm_100 device");
    outlier_reduce_kernel<<<segments, 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(row_sums, m, out);
    return check_launch("dmpq_outlier_reduce");
}

extern "C" dmpq_status dmpq_outlier_gate(const float* row_abs_sum, int m, const float* amax_in, double count,
                                         double tau_outlier, double* sum_out, int* flag_out, dmpq_stream_t s) {
    DMPQ_REQUIRE(row_abs_sum && amax_in && flag_out && m >= 0 && count > 0.0, DMPQ_EINVAL,
                 "dmpq_outlier_gate: bad arguments");
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_outlier_gate: needs an sm_100 device");
    outlier_gate_kernel<<<1, 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(row_abs_sum, m, amax_in, count, tau_outlier,
                                                                          sum_out, flag_out);
    return check_launch("dmpq_outlier_gate");
}

extern "C" dmpq_status dmpq_global_scale(const float* amax, float div, float* g_out, int count, dmpq_stream_t s) {
    DMPQ_REQUIRE(amax && g_out && count >= 0 && div > 0.0f, DMPQ_EINVAL, "dmpq_global_scale: bad arguments");
    if (count == 0) return DMPQ_OK;
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_global_scale: needs an sm_100 device");
    global_scale_kernel<<<(count + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(s)>>>(amax, div, g_out, count);
    return check_launch("dmpq_global_scale");
}
