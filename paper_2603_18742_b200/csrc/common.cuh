// common.cuh — shared host/device plumbing of libdmpq (sm_100a only).
// Not shared with oracle/ (the oracle and the CUDA path share no code).
#pragma once

#include <cuda_runtime.h>
#include <cuda_bf16.h>
#include <stdint.h>
#include <string>

#include "../../include/dmpq.h"

#if defined(__CUDA_ARCH__) && (__CUDA_ARCH__ != 1000)
#error "libdmpq targets sm_100a only (-gencode arch=compute_100a,code=sm_100a)"
#endif

namespace dmpq {

// ---------------------------------------------------------------- host errors
dmpq_status set_error(dmpq_status st, const char* fmt, ...);
dmpq_status check_launch(const char* what);
int num_sms();              // SM count of the current device (cached per device)
bool device_is_sm100();     // current device is compute capability 10.0

#define DMPQ_REQUIRE(cond, status, ...)                 \
    do {                                                \
        if (!(cond)) return ::dmpq::set_error(status, __VA_ARGS__); \
    } while (0)

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

// ---------------------------------------------------------------- device: numerics
// All parity-critical float arithmetic is written with explicit IEEE round-to-
// nearest intrinsics (and the library is built with --fmad=false), so the op
// order matches the definitions in include/dmpq.h and DESIGN.md §3.

__device__ __forceinline__ float bf16lo(uint32_t v) { return __uint_as_float(v << 16); }
__device__ __forceinline__ float bf16hi(uint32_t v) { return __uint_as_float(v & 0xFFFF0000u); }

// fp32 -> bf16 round-to-nearest-even (hardware cvt.rn.bf16x2.f32: first operand -> high half)
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
    uint32_t r;
    asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(r) : "f"(hi), "f"(lo));
    return r;
}

// E4M3 (satfinite, RN) of a non-negative float; returns the code byte.
__device__ __forceinline__ uint32_t e4m3_rn_satfinite(float v) {
    uint16_t r;
    asm("cvt.rn.satfinite.e4m3x2.f32 %0, %1, %2;" : "=h"(r) : "f"(0.0f), "f"(v));
    return r & 0xFFu;
}

// Exact E4M3 -> fp32 (every E4M3 value is an fp16 value).
__device__ __forceinline__ float e4m3_decode(uint32_t code) {
    uint32_t h2;
    uint16_t c = (uint16_t)code;
    asm("cvt.rn.f16x2.e4m3x2 %0, %1;" : "=r"(h2) : "h"(c));
    return __half2float(__ushort_as_half((unsigned short)(h2 & 0xFFFFu)));
}

// Two E2M1 codes (RN, satfinite, sign kept): lo -> bits 0..3, hi -> bits 4..7.
__device__ __forceinline__ uint32_t e2m1x2(float lo, float hi) {
    uint16_t r;
    asm("{ .reg .b8 t; cvt.rn.satfinite.e2m1x2.f32 t, %1, %2; mov.b16 %0, {t, 0}; }" : "=h"(r) : "f"(hi), "f"(lo));
    return r & 0xFFu;
}

// Packed fp32x2 arithmetic (sm_100: FFMA2 / FMUL2 / FADD2), each lane an IEEE
// round-to-nearest operation (never contracted: these are explicit .rn ops).
struct f2 { uint64_t v; };
__device__ __forceinline__ f2 f2make(float lo, float hi) { f2 r; asm("mov.b64 %0, {%1, %2};" : "=l"(r.v) : "f"(lo), "f"(hi)); return r; }
__device__ __forceinline__ float f2lo(f2 a) { return __uint_as_float((uint32_t)a.v); }
__device__ __forceinline__ float f2hi(f2 a) { return __uint_as_float((uint32_t)(a.v >> 32)); }
__device__ __forceinline__ f2 mul2(f2 a, f2 b) { f2 r; asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v)); return r; }
__device__ __forceinline__ f2 add2(f2 a, f2 b) { f2 r; asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v)); return r; }
__device__ __forceinline__ f2 sub2(f2 a, f2 b) { f2 r; asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v)); return r; }
__device__ __forceinline__ f2 fma2(f2 a, f2 b, f2 c) { f2 r; asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v)); return r; }
__device__ __forceinline__ uint32_t pack_bf16x2_f2(f2 a) {
    uint32_t r;
    asm("{ .reg .f32 lo, hi; mov.b64 {lo, hi}, %1; cvt.rn.bf16x2.f32 %0, hi, lo; }" : "=r"(r) : "l"(a.v));
    return r;
}
__device__ __forceinline__ float tanh_approx(float x) { float r; asm("tanh.approx.f32 %0, %1;" : "=f"(r) : "f"(x)); return r; }

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = __dadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// Non-negative float max via integer atomics (order-independent, deterministic).
__device__ __forceinline__ void atomic_max_nonneg(float* addr, float v) {
    atomicMax(reinterpret_cast<int*>(addr), __float_as_int(v));
}

// Streaming 16-byte global accesses.
__device__ __forceinline__ uint4 ldg_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
}

}  // namespace dmpq
