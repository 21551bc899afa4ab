// quant.cuh — shared pieces of the activation quantizers (quant.cu: row-vector kernel for
// rows without the Hadamard option; quant_tma.cu: TMA-staged chunk kernel).
#pragma once

#include "common.cuh"

namespace dmpq {

struct QuantParams {
    const uint16_t* X;
    int m, k, ldx;
    uint32_t flags;
    float ln_eps;
    uint16_t* h_out;
    int ldh;
    int8_t* i8_codes;
    float* i8_scale;
    uint8_t* fp4_codes;
    uint8_t* fp4_sf;
    const float* g;
    float* amax_out;
    float* row_abs_sum;   // PDR statistics (R15): per-row sum |x| of the layer input (pre-rotation)
    float* amax_in;       //                       max |x| of the layer input (pre-rotation)
    int i8_block;   // INT8 scale granularity: 0 per token (R2), 128 per Hadamard block (R17)
    int kc4;     // scale-column atoms per 128-row tile: ceil(k/16/4)
    int m_pad;   // rows rounded up to 128 (scale rows to zero-fill)
};

// bf16 pair (one 32-bit word) -> packed fp32x2 (exact widening)
__device__ __forceinline__ f2 bf16x2_to_f2(uint32_t w) { return f2make(bf16lo(w), bf16hi(w)); }

// Byte address of scale (row, atom column 0) in the 128x4 atom layout (R6).
__device__ __forceinline__ uint8_t* sf_row_ptr(uint8_t* sf, int kc4, int row) {
    return sf + (size_t)(row >> 7) * kc4 * 512 + (row & 31) * 16 + ((row & 127) >> 5) * 4;
}

// NVFP4 block scale of Eq. 2 with the two-level scale (R3/R4), IEEE intrinsics:
// returns the E4M3 code, sets rcp = fl(1/eff)
__device__ __forceinline__ uint32_t nvfp4_block_scale(float a_b, float g, float& rcp) {
    const float raw = __fdiv_rn(__fdiv_rn(a_b, 6.0f), g);
    const uint32_t sb = e4m3_rn_satfinite(raw);
    const float eff = __fmul_rn(e4m3_decode(sb), g);
    rcp = eff > 0.0f ? __frcp_rn(eff) : 0.0f;
    return sb;
}

// Eight E2M1 codes (RN, satfinite, sign kept) of a[0..7] -> one 32-bit word, element i in
// nibble i (element 2j in the low nibble of byte j). ptxas merges the four cvts into one
// register (F2FP ... PACK_AB_MERGE_C), no shifts or ors.
__device__ __forceinline__ uint32_t e2m1x8(f2 a01, f2 a23, f2 a45, f2 a67) {
    uint32_t r;
    asm("{ .reg .b8 b0, b1, b2, b3;\n\t"
        "cvt.rn.satfinite.e2m1x2.f32 b0, %2, %1;\n\t"
        "cvt.rn.satfinite.e2m1x2.f32 b1, %4, %3;\n\t"
        "cvt.rn.satfinite.e2m1x2.f32 b2, %6, %5;\n\t"
        "cvt.rn.satfinite.e2m1x2.f32 b3, %8, %7;\n\t"
        "mov.b32 %0, {b0, b1, b2, b3}; }"
        : "=r"(r)
        : "f"(f2lo(a01)), "f"(f2hi(a01)), "f"(f2lo(a23)), "f"(f2hi(a23)), "f"(f2lo(a45)), "f"(f2hi(a45)),
          "f"(f2lo(a67)), "f"(f2hi(a67)));
    return r;
}

// Two E4M3 codes (RN, satfinite) of non-negative (lo, hi) -> 16 bits, lo in the low byte.
__device__ __forceinline__ uint32_t e4m3x2(f2 v) {
    uint16_t r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(f2hi(v)), "f"(f2lo(v)));
    return r;
}

// Exact decode of two E4M3 codes (low byte -> lo lane).
__device__ __forceinline__ f2 e4m3x2_decode(uint32_t codes16) {
    uint32_t h2;
    const uint16_t c = (uint16_t)codes16;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(c));
    return f2make(__half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFFu))),
                  __half2float(__ushort_as_half((unsigned short)(h2 >> 16))));
}

// four int8 codes RNE(q * rcp) (saturating pack; the clamp never binds). Byte order q0..q3.
__device__ __forceinline__ uint32_t int8x4(f2 q01, f2 q23) {
    uint32_t r;
    asm("{ .reg .s32 i0, i1, i2, i3; .reg .b32 pp;\n\t"
        "cvt.rni.s32.f32 i0, %1; cvt.rni.s32.f32 i1, %2; cvt.rni.s32.f32 i2, %3; cvt.rni.s32.f32 i3, %4;\n\t"
        "cvt.pack.sat.s8.s32.b32 pp, i3, i2, 0; cvt.pack.sat.s8.s32.b32 %0, i1, i0, pp; }"
        : "=r"(r) : "f"(f2lo(q01)), "f"(f2hi(q01)), "f"(f2lo(q23)), "f"(f2hi(q23)));
    return r;
}

// Chunk quantizer (quant_tma.cu): rows staged by TMA, 64 elements per thread.
dmpq_status launch_quant_tma(const QuantParams& p, bool hadamard, cudaStream_t s);
dmpq_status prepare_quant_tma();
// Hadamard quantizer (quant_had.cu): one 128-element block per thread, all FHT stages in registers.
dmpq_status launch_quant_had(const QuantParams& p, cudaStream_t s);
dmpq_status prepare_quant_had();

}  // namespace dmpq
