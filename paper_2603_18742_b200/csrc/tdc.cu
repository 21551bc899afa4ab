// tdc.cu — tdc_step: the device half of the Temporal Delta Cache (§4.2).
//   SKIP:        X_out = bf16(fl(X_in + Delta_tp))
//   REFRESH (Eq. 8): Delta_new = bf16(fl(X_out - X_in)) into the cache, fused
//            with the FP64 statistics of Eq. 3 (Gamma) and Eq. 9 (cosine of the
//            two most recent computed deltas).
// HBM-bound streaming kernels: 16-byte vectors, persistent grid-stride loop.
// Statistics: the Gamma/L2 sums are FP32 over each 8-element
// vector, then FP64; the three cosine sums are exact bf16 products accumulated in
// FP64 per element (DFMA: an exact product, one rounding per term). Per-thread
// FP64 accumulators are reduced warp -> CTA in fixed order and the per-CTA
// partials are summed in CTA order by the last CTA (deterministic for a given m x h).
#include "fastmath.cuh"
#include "quant.cuh"

namespace dmpq {

constexpr int kTdcThreads = 256;

// stats_out[j] = sum over the n per-CTA partials[b * 7 + j], fixed order: warp j (< 7) lets
// lane l sum partials l, l + 32, ... and then combines the lanes with a fixed butterfly
// (called by the last CTA; replaces a serial 7-thread sum, which took ~3 us at 592 partials).
__device__ __forceinline__ void sum_partials(const double* partials, unsigned n, double* stats_out) {
    const unsigned w = threadIdx.x >> 5, l = threadIdx.x & 31;
    if (w < 7) {
        double v = 0.0;
        for (unsigned b = l; b < n; b += 32) v = __dadd_rn(v, __ldcg(partials + (size_t)b * 7 + w));
        v = warp_sum_d(v);
        if (l == 0) stats_out[w] = v;
    }
}
constexpr int kTdcCtasPerSm = 4;

static int tdc_grid(long long nvec) {
    long long g = (long long)num_sms() * kTdcCtasPerSm;
    long long need = (nvec + kTdcThreads - 1) / kTdcThreads;
    if (g > need) g = need;
    return (int)(g < 1 ? 1 : g);
}

__global__ void __launch_bounds__(kTdcThreads) tdc_skip_kernel(const uint16_t* x_in, const uint16_t* delta,
                                                               uint16_t* x_out, long long nvec) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
        const uint4 x = ldg_stream(x_in + i * 8);
        const uint4 d = ldg_stream(delta + i * 8);
        const uint32_t xw[4] = {x.x, x.y, x.z, x.w}, dw[4] = {d.x, d.y, d.z, d.w};
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            o[j] = pack_bf16x2(__fadd_rn(bf16lo(xw[j]), bf16lo(dw[j])), __fadd_rn(bf16hi(xw[j]), bf16hi(dw[j])));
        *reinterpret_cast<uint4*>(x_out + i * 8) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

__global__ void __launch_bounds__(kTdcThreads) tdc_refresh_kernel(const uint16_t* __restrict__ x_in,
                                                                  const uint16_t* __restrict__ x_out,
                                                                  uint16_t* delta, long long nvec,
                                                                  double* partials, unsigned int* counter,
                                                                  double* stats_out) {
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
        const uint4 x = ldg_stream(x_in + i * 8);
        const uint4 y = ldg_stream(x_out + i * 8);
        const uint4 p = *reinterpret_cast<const uint4*>(delta + i * 8);
        const uint32_t xw[4] = {x.x, x.y, x.z, x.w}, yw[4] = {y.x, y.y, y.z, y.w}, pw[4] = {p.x, p.y, p.z, p.w};
        // Gamma / L2 sums: FP32 over the 8-element vector, then FP64 (<= 7 roundings
        // per vector: relative error <= 4.2e-7, inside the 1e-6 decision exemption).
        // Cosine sums (Eq. 9): bf16 x bf16 products are exact; FP64 per element.
        float s[4] = {0, 0, 0, 0};
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float xa = bf16lo(xw[j]), xb = bf16hi(xw[j]);
            const float da = __fsub_rn(bf16lo(yw[j]), xa), db = __fsub_rn(bf16hi(yw[j]), xb);
            o[j] = pack_bf16x2(da, db);
            const double na = (double)bf16lo(o[j]), nb = (double)bf16hi(o[j]);
            const double pa = (double)bf16lo(pw[j]), pb = (double)bf16hi(pw[j]);
            s[0] = __fadd_rn(s[0], __fadd_rn(fabsf(da), fabsf(db)));
            s[1] = __fadd_rn(s[1], __fadd_rn(fabsf(xa), fabsf(xb)));
            s[2] = __fadd_rn(s[2], __fadd_rn(__fmul_rn(da, da), __fmul_rn(db, db)));
            s[3] = __fadd_rn(s[3], __fadd_rn(__fmul_rn(xa, xa), __fmul_rn(xb, xb)));
            acc[4] = __fma_rn(na, pa, acc[4]); acc[4] = __fma_rn(nb, pb, acc[4]);
            acc[5] = __fma_rn(na, na, acc[5]); acc[5] = __fma_rn(nb, nb, acc[5]);
            acc[6] = __fma_rn(pa, pa, acc[6]); acc[6] = __fma_rn(pb, pb, acc[6]);
        }
        *reinterpret_cast<uint4*>(delta + i * 8) = make_uint4(o[0], o[1], o[2], o[3]);
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = __dadd_rn(acc[j], (double)s[j]);
    }
    __shared__ double red[kTdcThreads / 32][7];
    __shared__ bool is_last;
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
#pragma unroll
    for (int j = 0; j < 7; ++j) {
        double v = warp_sum_d(acc[j]);
        if (l == 0) red[w][j] = v;
    }
    __syncthreads();
    if (threadIdx.x < 7) {
        double v = 0.0;
        for (int ww = 0; ww < kTdcThreads / 32; ++ww) v = __dadd_rn(v, red[ww][threadIdx.x]);
        partials[(size_t)blockIdx.x * 7 + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (is_last) {
        __threadfence();
        sum_partials(partials, gridDim.x, stats_out);
        if (threadIdx.x == 0) *counter = 0u;  // leave the workspace ready for the next call
    }
}

// ---------------------------------------------------------------------------------------------
// NVFP4-compressed delta cache (R16). One thread = 8 consecutive elements
// (one 16-byte vector of each bf16 tensor, one 32-bit word of codes, half of an NVFP4 block):
// every global access is coalesced across the warp; the two halves of a block sit in lanes
// 2j, 2j+1 (one shuffle for the block maximum). Warp-uniform grid-stride loop.
// ---------------------------------------------------------------------------------------------

// two E2M1 codes (one byte, element 2i in the low nibble) -> exact fp32 pair
__device__ __forceinline__ f2 e2m1x2_decode(uint32_t byte) {
    uint32_t h2;
    asm("{ .reg .b8 t; .reg .b16 u; cvt.u16.u32 u, %1; cvt.u8.u16 t, u; cvt.rn.f16x2.e2m1x2 %0, t; }" : "=r"(h2) : "r"(byte));
    return f2make(__half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFFu))),
                  __half2float(__ushort_as_half((unsigned short)(h2 >> 16))));
}

// dq of 8 cached elements (one 32-bit word of codes) under eff = fl(dec(s_b) * g): fl(dec(code) * eff),
// scalar IEEE multiplies (ptxas would contract a packed mul2 feeding an add2 into FFMA2)
__device__ __forceinline__ void cache_dequant8(uint32_t word, float eff, float (&dq)[8]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const f2 v = e2m1x2_decode((word >> (8 * j)) & 0xFFu);
        dq[2 * j] = __fmul_rn(f2lo(v), eff);
        dq[2 * j + 1] = __fmul_rn(f2hi(v), eff);
    }
}

__device__ __forceinline__ float e4m3_eff(const uint8_t* sf, long long blk, float g) {
    return __fmul_rn(e4m3_decode(__ldg(sf + blk)), g);
}

__global__ void __launch_bounds__(kTdcThreads) tdc_skip_nvfp4_kernel(const uint16_t* x_in, const uint8_t* codes,
                                                                     const uint8_t* sf, const float* g_ptr,
                                                                     uint16_t* x_out, long long nvec) {
    const float g = *g_ptr;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
        const uint4 x = ldg_stream(x_in + i * 8);
        const uint32_t cw = __ldg(reinterpret_cast<const uint32_t*>(codes) + i);
        float dq[8];
        cache_dequant8(cw, e4m3_eff(sf, i >> 1, g), dq);
        const uint32_t xw[4] = {x.x, x.y, x.z, x.w};
        uint32_t o[4];
#pragma unroll
        for (int j = 0; j < 4; ++j)
            o[j] = pack_bf16x2(__fadd_rn(bf16lo(xw[j]), dq[2 * j]), __fadd_rn(bf16hi(xw[j]), dq[2 * j + 1]));
        *reinterpret_cast<uint4*>(x_out + i * 8) = make_uint4(o[0], o[1], o[2], o[3]);
    }
}

// max |fl(y - x)|
__global__ void __launch_bounds__(kTdcThreads) tdc_delta_amax_kernel(const uint16_t* x_in, const uint16_t* x_out,
                                                                     long long nvec, float* amax_out) {
    float a = 0.0f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
        const uint4 x = ldg_stream(x_in + i * 8), y = ldg_stream(x_out + i * 8);
        const uint32_t xw[4] = {x.x, x.y, x.z, x.w}, yw[4] = {y.x, y.y, y.z, y.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const f2 d = sub2(bf16x2_to_f2(yw[j]), bf16x2_to_f2(xw[j]));
            a = fmaxf(a, fmaxf(fabsf(f2lo(d)), fabsf(f2hi(d))));
        }
    }
    a = warp_max(a);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(amax_out, a);
}

__global__ void __launch_bounds__(kTdcThreads) tdc_refresh_nvfp4_kernel(
    const uint16_t* __restrict__ x_in, const uint16_t* __restrict__ x_out, uint8_t* codes, uint8_t* sf, float* g_cache,
    const float* g_new_ptr, float* amax_out, long long nvec, double* partials, unsigned int* counter, double* stats_out) {
    const float g_prev = *g_cache, g = *g_new_ptr;
    // fast exact block-scale path (fastmath.cuh) when g and the block maximum are in its guard range
    const bool g_ok = g >= 8.0779356e-28f && g <= 1.2379400e27f;
    const float a_lo = fmaxf(6.3108872e-30f, __fmul_rn(g, 6.3108872e-30f));
    const float a_hi = fminf(FM_HI, __fmul_rn(g, 5.0706024e30f));
    const float rg = g_ok ? recip_refined(g) : 0.0f;
    const f2 g2 = f2make(g, g), ng2 = f2make(-g, -g), rg2 = f2make(rg, rg);
    const f2 n6 = f2make(-6.0f, -6.0f), r6 = f2make(0.16666667163372039795f, 0.16666667163372039795f);
    double acc[7] = {0, 0, 0, 0, 0, 0, 0};
    float amax = 0.0f;
    const int lane = threadIdx.x & 31;
    const long long stride = (long long)gridDim.x * blockDim.x;
    // warp-uniform loop (the block maximum is a lane-pair shuffle)
    for (long long base = (blockIdx.x * (long long)blockDim.x + threadIdx.x) - lane; base < nvec; base += stride) {
        const long long i = base + lane;
        const bool ok = i < nvec;
        uint4 x = make_uint4(0, 0, 0, 0), y = x;
        uint32_t cw = 0;
        float eff_prev = 0.0f;
        if (ok) {
            x = ldg_stream(x_in + i * 8);
            y = ldg_stream(x_out + i * 8);
            cw = *(reinterpret_cast<const uint32_t*>(codes) + i);
            eff_prev = __fmul_rn(e4m3_decode(sf[i >> 1]), g_prev);
        }
        float dq[8];
        cache_dequant8(cw, eff_prev, dq);
        const uint32_t xw[4] = {x.x, x.y, x.z, x.w}, yw[4] = {y.x, y.y, y.z, y.w};
        float d[8];
        // Gamma / L2 sums: FP32 over the 8-element vector, then FP64 (as tdc_refresh_kernel)
        float s4[4] = {0, 0, 0, 0};
        float am = 0.0f;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const float xa = bf16lo(xw[j]), xb = bf16hi(xw[j]);
            const float da = __fsub_rn(bf16lo(yw[j]), xa), db = __fsub_rn(bf16hi(yw[j]), xb);
            d[2 * j] = da;
            d[2 * j + 1] = db;
            am = fmaxf(am, fmaxf(fabsf(da), fabsf(db)));
            const uint32_t nw = pack_bf16x2(da, db);
            const double na = (double)bf16lo(nw), nb = (double)bf16hi(nw);
            const double pa = (double)dq[2 * j], pb = (double)dq[2 * j + 1];
            s4[0] = __fadd_rn(s4[0], __fadd_rn(fabsf(da), fabsf(db)));
            s4[1] = __fadd_rn(s4[1], __fadd_rn(fabsf(xa), fabsf(xb)));
            s4[2] = __fadd_rn(s4[2], __fadd_rn(__fmul_rn(da, da), __fmul_rn(db, db)));
            s4[3] = __fadd_rn(s4[3], __fadd_rn(__fmul_rn(xa, xa), __fmul_rn(xb, xb)));
            // Eq. 9 sums: bf16 x fl32 products are exact in FP64
            acc[4] = __fma_rn(na, pa, acc[4]); acc[4] = __fma_rn(nb, pb, acc[4]);
            acc[5] = __fma_rn(na, na, acc[5]); acc[5] = __fma_rn(nb, nb, acc[5]);
            acc[6] = __fma_rn(pa, pa, acc[6]); acc[6] = __fma_rn(pb, pb, acc[6]);
        }
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[j] = __dadd_rn(acc[j], (double)s4[j]);
        amax = fmaxf(amax, am);
        // re-quantize the cache: NVFP4(d; g_new), the FP32-input quantizer of Eq. 2 (R4); both
        // lanes of a block compute its scale
        const float a_b = fmaxf(am, __shfl_xor_sync(0xffffffffu, am, 1));
        uint32_t sb;
        float r;
        if (g_ok && a_b >= a_lo && a_b <= a_hi) {
            const f2 raw = div2_fast(div2_fast(f2make(a_b, a_b), n6, r6), ng2, rg2);
            sb = e4m3x2(raw) & 0xFFu;
            const f2 e = mul2(e4m3x2_decode(sb), g2);
            const f2 rr = rcp2_fast(e);
            r = f2lo(e) > 0.0f ? f2lo(rr) : 0.0f;
        } else {
            sb = nvfp4_block_scale(a_b, g, r);
        }
        if (ok) {
            const f2 r2 = f2make(r, r);
            *(reinterpret_cast<uint32_t*>(codes) + i) =
                e2m1x8(mul2(f2make(d[0], d[1]), r2), mul2(f2make(d[2], d[3]), r2), mul2(f2make(d[4], d[5]), r2),
                       mul2(f2make(d[6], d[7]), r2));
            if ((i & 1) == 0) sf[i >> 1] = (uint8_t)sb;
        }
    }
    if (amax_out) {
        const float am = warp_max(amax);
        if (lane == 0) atomic_max_nonneg(amax_out, am);
    }
    __shared__ double red[kTdcThreads / 32][7];
    __shared__ bool is_last;
    const int w = threadIdx.x >> 5, l = lane;
#pragma unroll
    for (int j = 0; j < 7; ++j) {
        double v = warp_sum_d(acc[j]);
        if (l == 0) red[w][j] = v;
    }
    __syncthreads();
    if (threadIdx.x < 7) {
        double v = 0.0;
        for (int ww = 0; ww < kTdcThreads / 32; ++ww) v = __dadd_rn(v, red[ww][threadIdx.x]);
        partials[(size_t)blockIdx.x * 7 + threadIdx.x] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) is_last = (atomicAdd(counter, 1u) == gridDim.x - 1);
    __syncthreads();
    if (is_last) {
        __threadfence();
        sum_partials(partials, gridDim.x, stats_out);
        if (threadIdx.x == 0) {
            *g_cache = g;        // every CTA has read the old scale (they all counted in before this one)
            *counter = 0u;       // leave the workspace ready for the next call
        }
    }
}

}  // namespace dmpq

using namespace dmpq;

extern "C" size_t tdc_workspace_bytes(int m, int h) {
    (void)m; (void)h;
    // partials for the largest grid any device can use + the completion counter
    return (size_t)1024 * kTdcCtasPerSm * 7 * sizeof(double) + 256;
}

extern "C" dmpq_status tdc_step(tdc_mode mode, const uint16_t* X_in, uint16_t* X_out, uint16_t* delta_cache, int m, int h,
                                double* stats_out, void* workspace, dmpq_stream_t s) {
    DMPQ_REQUIRE(mode == TDC_SKIP || mode == TDC_REFRESH, DMPQ_EINVAL, "tdc_step: unknown mode %d", (int)mode);
    DMPQ_REQUIRE(m >= 0 && h > 0 && h % 8 == 0, DMPQ_ESHAPE, "tdc_step: need m >= 0, h %% 8 == 0 (m=%d h=%d)", m, h);
    DMPQ_REQUIRE(X_in && X_out && delta_cache && aligned16(X_in) && aligned16(X_out) && aligned16(delta_cache),
                 DMPQ_EALIGN, "tdc_step: tensors must be 16-byte aligned device pointers");
    const long long nvec = (long long)m * h / 8;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    if (mode == TDC_SKIP) {
        if (nvec == 0) return DMPQ_OK;
        DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "tdc_step: needs an sm_100 device");
        tdc_skip_kernel<<<tdc_grid(nvec), kTdcThreads, 0, st>>>(X_in, delta_cache, X_out, nvec);
        return check_launch("tdc_step(SKIP)");
    }
    DMPQ_REQUIRE(X_in != X_out, DMPQ_EINVAL, "tdc_step(REFRESH): X_out must not alias X_in");
    DMPQ_REQUIRE(stats_out && workspace && aligned16(workspace), DMPQ_EINVAL, "tdc_step(REFRESH): stats_out/workspace");
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "tdc_step: needs an sm_100 device");
    const int grid = nvec == 0 ? 1 : tdc_grid(nvec);
    DMPQ_REQUIRE(grid <= 1024 * kTdcCtasPerSm, DMPQ_EUNSUPPORTED, "tdc_step: grid too large for workspace");
    double* partials = reinterpret_cast<double*>(workspace);
    unsigned int* counter = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(workspace) +
                                                            (size_t)1024 * kTdcCtasPerSm * 7 * sizeof(double));
    tdc_refresh_kernel<<<grid, kTdcThreads, 0, st>>>(X_in, X_out, delta_cache, nvec, partials, counter, stats_out);
    return check_launch("tdc_step(REFRESH)");
}

extern "C" dmpq_status tdc_step_nvfp4(tdc_mode mode, const uint16_t* X_in, uint16_t* X_out, const tdc_nvfp4_cache* cache,
                                      const float* g_new, float* amax_out, int m, int h, double* stats_out,
                                      void* workspace, dmpq_stream_t s) {
    DMPQ_REQUIRE(mode == TDC_SKIP || mode == TDC_REFRESH, DMPQ_EINVAL, "tdc_step_nvfp4: unknown mode %d", (int)mode);
    DMPQ_REQUIRE(m >= 0 && h > 0 && h % 64 == 0, DMPQ_ESHAPE, "tdc_step_nvfp4: need m >= 0, h %% 64 == 0 (m=%d h=%d)", m, h);
    DMPQ_REQUIRE(cache && cache->codes && cache->sf && cache->g, DMPQ_EINVAL, "tdc_step_nvfp4: cache buffers");
    DMPQ_REQUIRE(X_in && X_out && aligned16(X_in) && aligned16(X_out) && (reinterpret_cast<uintptr_t>(cache->codes) & 3u) == 0,
                 DMPQ_EALIGN, "tdc_step_nvfp4: X 16-byte, codes 4-byte aligned device pointers");
    const long long nvec = (long long)m * h / 8;
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    if (mode == TDC_SKIP) {
        if (nvec == 0) return DMPQ_OK;
        DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "tdc_step_nvfp4: needs an sm_100 device");
        tdc_skip_nvfp4_kernel<<<tdc_grid(nvec), kTdcThreads, 0, st>>>(X_in, cache->codes, cache->sf, cache->g, X_out,
                                                                      nvec);
        return check_launch("tdc_step_nvfp4(SKIP)");
    }
    DMPQ_REQUIRE(X_in != X_out, DMPQ_EINVAL, "tdc_step_nvfp4(REFRESH): X_out must not alias X_in");
    DMPQ_REQUIRE(g_new && stats_out && workspace && aligned16(workspace), DMPQ_EINVAL,
                 "tdc_step_nvfp4(REFRESH): g_new/stats_out/workspace");
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "tdc_step_nvfp4: needs an sm_100 device");
    const int grid = nvec == 0 ? 1 : tdc_grid(nvec);
    DMPQ_REQUIRE(grid <= 1024 * kTdcCtasPerSm, DMPQ_EUNSUPPORTED, "tdc_step_nvfp4: grid too large for workspace");
    double* partials = reinterpret_cast<double*>(workspace);
    unsigned int* counter = reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(workspace) +
                                                            (size_t)1024 * kTdcCtasPerSm * 7 * sizeof(double));
    tdc_refresh_nvfp4_kernel<<<grid, kTdcThreads, 0, st>>>(X_in, X_out, cache->codes, cache->sf, cache->g, g_new,
                                                           amax_out, nvec, partials, counter, stats_out);
    return check_launch("tdc_step_nvfp4(REFRESH)");
}

extern "C" dmpq_status tdc_delta_amax(const uint16_t* X_in, const uint16_t* X_out, int m, int h, float* amax_out,
                                      dmpq_stream_t s) {
    DMPQ_REQUIRE(m >= 0 && h > 0 && h % 8 == 0, DMPQ_ESHAPE, "tdc_delta_amax: need h %% 8 == 0");
    DMPQ_REQUIRE(X_in && X_out && amax_out && aligned16(X_in) && aligned16(X_out), DMPQ_EALIGN,
                 "tdc_delta_amax: 16-byte aligned device pointers");
    const long long nvec = (long long)m * h / 8;
    if (nvec == 0) return DMPQ_OK;
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "tdc_delta_amax: needs an sm_100 device");
    tdc_delta_amax_kernel<<<tdc_grid(nvec), kTdcThreads, 0, reinterpret_cast<cudaStream_t>(s)>>>(X_in, X_out, nvec,
                                                                                                 amax_out);
    return check_launch("tdc_delta_amax");
}
