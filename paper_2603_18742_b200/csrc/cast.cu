// cast.cu — dmpq_cast_int8: the on-the-fly NVFP4 -> INT8 weight cast of PAPER.md P:184 ("all
// weights are quantized to NVFP4 offline ... for layers routed to INT8, the NVFP4 weights are
// cast to INT8 on-the-fly"; R7, NEXT-4b). Only the NVFP4 form of a layer stays resident;
// right before an INT8-routed GEMM this kernel rebuilds the layer's INT8 codes into a shared
// scratch buffer (sized for the largest layer, so it stays L2-resident for the GEMM that follows):
//   W^ = fl(dec(code) * fl(dec(s_b) * g_w)),   i8 = RNE(fl(W^ * r_w[n])),
// with r_w = fl(127 / max_k |W^|) saved by the pack -- the same operations as the pack's INT8
// half (pack.cu), so the codes are bit-identical to the pre-packed ones.
//
// Layout: one thread per 32 consecutive weights of a row (16 code bytes = two NVFP4 blocks, one
// 16-bit pair of scale bytes in the 128x4 atom layout, two 16-byte INT8 stores); grid-stride,
// coalesced 16-byte loads/stores. HBM-bound: 0.5625 B read + 1 B written per weight.
#include "common.cuh"
#include "quant.cuh"

namespace dmpq {

namespace {

// eight E2M1 codes (one 32-bit word, element i in nibble i) -> four packed fp32 pairs, exact
__device__ __forceinline__ void e2m1x8_decode(uint32_t w, f2* out) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        uint32_t h2;
        const uint16_t byte = (uint16_t)((w >> (8 * j)) & 0xFFu);
        asm("{ .reg .b8 t; cvt.u8.u16 t, %1; cvt.rn.f16x2.e2m1x2 %0, t; }" : "=r"(h2) : "h"(byte));
        out[j] = f2make(__half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFFu))),
                        __half2float(__ushort_as_half((unsigned short)(h2 >> 16))));
    }
}

// four int8 codes of v = (v01.lo, v01.hi, v23.lo, v23.hi), |v| < 2^22, already rounded products:
// fl(v + 1.5 2^23) has ulp 1, so its low byte is the two's complement RNE(v)
__device__ __forceinline__ uint32_t int8x4_rne(f2 v01, f2 v23) {
    const f2 mg = f2make(12582912.0f, 12582912.0f);
    const f2 a = add2(v01, mg), b = add2(v23, mg);
    const uint32_t lo = __byte_perm(__float_as_uint(f2lo(a)), __float_as_uint(f2hi(a)), 0x0040);
    const uint32_t hi = __byte_perm(__float_as_uint(f2lo(b)), __float_as_uint(f2hi(b)), 0x0040);
    return __byte_perm(lo, hi, 0x5410);
}

__global__ void __launch_bounds__(256) cast_int8_kernel(const uint8_t* __restrict__ codes, const uint8_t* __restrict__ sf,
                                                        const float* __restrict__ g_ptr, const float* __restrict__ g_col,
                                                        const float* __restrict__ rcp, int n, int k, int kc4,
                                                        int8_t* __restrict__ out, float zero) {
    const int cpr = k >> 5;   // 32-weight chunks per row
    const long long total = (long long)n * cpr;
    const f2 z2 = f2make(zero, zero);   // +0 addend, opaque to ptxas: the product is not contracted
    const float g_all = g_col ? 0.0f : *g_ptr;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < total; i += (long long)gridDim.x * blockDim.x) {
        const int row = (int)(i / cpr), c = (int)(i - (long long)row * cpr);
        const uint4 q = ldg_stream(codes + (size_t)row * (k >> 1) + (size_t)c * 16);
        const int blk = 2 * c;   // first of the two 16-element scale blocks (even: same atom word)
        const uint32_t s2 = *reinterpret_cast<const uint16_t*>(sf_row_ptr(const_cast<uint8_t*>(sf), kc4, row) +
                                                               (size_t)(blk >> 2) * 512 + (blk & 3));
        const float g = g_col ? g_col[row] : g_all;
        const f2 sd = e4m3x2_decode(s2);
        const f2 eff = mul2(sd, f2make(g, g));     // (fl(dec(s_b) g), fl(dec(s_b+1) g))
        const float r = rcp[row];
        const f2 r2 = f2make(r, r);
        const uint32_t w[4] = {q.x, q.y, q.z, q.w};
        uint32_t o[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {              // word j: elements 8j .. 8j+7 (block j / 2)
            f2 d[4];
            e2m1x8_decode(w[j], d);
            const float e = j < 2 ? f2lo(eff) : f2hi(eff);
            const f2 e2 = f2make(e, e);
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const f2 v0 = fma2(mul2(d[2 * h], e2), r2, z2), v1 = fma2(mul2(d[2 * h + 1], e2), r2, z2);
                o[2 * j + h] = int8x4_rne(v0, v1);
            }
        }
        uint4* dst = reinterpret_cast<uint4*>(out + (size_t)row * k + (size_t)c * 32);
        dst[0] = make_uint4(o[0], o[1], o[2], o[3]);
        dst[1] = make_uint4(o[4], o[5], o[6], o[7]);
    }
}

}  // namespace

}  // namespace dmpq

using namespace dmpq;

extern "C" dmpq_status dmpq_cast_int8(const dmpq_weights* W, int8_t* i8_out, dmpq_stream_t s) {
    DMPQ_REQUIRE(W && i8_out && W->fp4_codes && W->fp4_sf && (W->fp4_g || W->fp4_g_col) && W->i8_rcp, DMPQ_EINVAL,
                 "dmpq_cast_int8: needs the NVFP4 form, g_w and W->i8_rcp (pack with i8_rcp set)");
    DMPQ_REQUIRE(W->n > 0 && W->k > 0 && W->k % 64 == 0 && W->n % 16 == 0, DMPQ_ESHAPE,
                 "dmpq_cast_int8: need n %% 16 == 0, k %% 64 == 0 (n=%d k=%d)", W->n, W->k);
    DMPQ_REQUIRE(aligned16(W->fp4_codes) && aligned16(i8_out), DMPQ_EALIGN, "dmpq_cast_int8: 16-byte alignment");
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_cast_int8: needs an sm_100 device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    const long long chunks = (long long)W->n * (W->k / 32);
    long long grid = (chunks + 255) / 256;
    if (grid > (long long)num_sms() * 8) grid = (long long)num_sms() * 8;
    cast_int8_kernel<<<(int)grid, 256, 0, st>>>(W->fp4_codes, W->fp4_sf, W->fp4_g, W->fp4_g_col, W->i8_rcp, W->n, W->k,
                                                ((W->k / 16) + 3) / 4, i8_out, 0.0f);
    return check_launch("dmpq_cast_int8");
}
