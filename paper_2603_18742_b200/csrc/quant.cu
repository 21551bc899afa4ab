// quant.cu — dmpq_quantize_act: online NVFP4 / per-token INT8 activation
// quantization (Eq. 2; R2-R6), optionally
// with a fused row LayerNorm prologue (block glue), and dmpq_global_scale.
//
// HBM-bound streaming kernel. Each row is held in registers by one warp (k <= 512)
// or one CTA (k > 512): NV 16-byte vectors (8 bf16) per thread, loaded once,
// coalesced (consecutive lanes own consecutive vectors). Reductions: warp
// shuffles + shared memory, fixed order (deterministic). Per 16-element NVFP4
// block the two lanes holding it exchange their maxima with one shuffle; four
// consecutive blocks' E4M3 scales (one 32-bit word of the swizzled scale layout)
// are gathered by shuffles and stored by one lane. Persistent grid over rows.
#include <cstdio>

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
    int kc4;     // scale-column atoms per 128-row tile: ceil(k/16/4)
    int m_pad;   // rows rounded up to 128 (scale rows to zero-fill)
};

template <bool WARP_ROW>
struct RowReduce {
    float* red;  // shared scratch, >= 33 floats
    __device__ __forceinline__ float sum(float v) {
        v = warp_sum(v);
        if constexpr (WARP_ROW) return v;
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
        __syncthreads();
        if (l == 0) red[w] = v;
        __syncthreads();
        float t = (l < nw) ? red[l] : 0.0f;
        return warp_sum(t);
    }
    __device__ __forceinline__ float max(float v) {
        v = warp_max(v);
        if constexpr (WARP_ROW) return v;
        const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
        __syncthreads();
        if (l == 0) red[w] = v;
        __syncthreads();
        float t = (l < nw) ? red[l] : 0.0f;
        return warp_max(t);
    }
};

// bf16 pair (one 32-bit word) -> packed fp32x2 (exact widening)
__device__ __forceinline__ f2 bf16x2_to_f2(uint32_t w) { return f2make(bf16lo(w), bf16hi(w)); }

// |x| max over a vector of 8 bf16, in the bf16 domain (exact): max.bf16x2 on sign-cleared words
__device__ __forceinline__ float vec_absmax(const uint4& v) {
    uint32_t m;
    asm("{ .reg .b32 a, b, c, d, t, u;\n\t"
        "and.b32 a, %1, 0x7fff7fff; and.b32 b, %2, 0x7fff7fff; and.b32 c, %3, 0x7fff7fff; and.b32 d, %4, 0x7fff7fff;\n\t"
        "max.bf16x2 t, a, b; max.bf16x2 u, c, d; max.bf16x2 %0, t, u; }"
        : "=r"(m) : "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w));
    return fmaxf(bf16lo(m), bf16hi(m));
}

// 8 bf16 -> 8 E2M1 codes (4 bytes), x * rcp per element (R4)
__device__ __forceinline__ uint32_t vec_e2m1(const uint4& v, f2 rcp2) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t codes = 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const f2 q = mul2(bf16x2_to_f2(w[j]), rcp2);
        codes |= e2m1x2(f2lo(q), f2hi(q)) << (8 * j);
    }
    return codes;
}

// 8 bf16 -> 8 int8 codes RNE(x * rcp) with saturation (the clamp never binds).
// cvt.pack d, a, b, c: d = {c[15:0], a, b} (bytes 3..0) -> element order i0..i3 in bytes 0..3
__device__ __forceinline__ uint2 vec_int8(const uint4& v, f2 rcp2) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    uint32_t out[2];
#pragma unroll
    for (int h = 0; h < 2; ++h) {
        const f2 q0 = mul2(bf16x2_to_f2(w[2 * h]), rcp2);
        const f2 q1 = mul2(bf16x2_to_f2(w[2 * h + 1]), rcp2);
        uint32_t r;
        asm("{ .reg .s32 i0, i1, i2, i3; .reg .b32 p;\n\t"
            "cvt.rni.s32.f32 i0, %1; cvt.rni.s32.f32 i1, %2; cvt.rni.s32.f32 i2, %3; cvt.rni.s32.f32 i3, %4;\n\t"
            "cvt.pack.sat.s8.s32.b32 p, i3, i2, 0; cvt.pack.sat.s8.s32.b32 %0, i1, i0, p; }"
            : "=r"(r) : "f"(f2lo(q0)), "f"(f2hi(q0)), "f"(f2lo(q1)), "f"(f2hi(q1)));
        out[h] = r;
    }
    return make_uint2(out[0], out[1]);
}

template <int NV>
__device__ __forceinline__ void load_row(uint4 (&v)[NV], const uint16_t* xr, int tid, int tpr, int nvec, bool valid) {
#pragma unroll
    for (int i = 0; i < NV; ++i) {
        const int vi = tid + i * tpr;
        v[i] = (valid && vi < nvec) ? ldg_stream(xr + (size_t)vi * 8) : make_uint4(0, 0, 0, 0);
    }
}

template <int NV, bool WARP_ROW>
__global__ void __launch_bounds__(256) quant_act_kernel(const QuantParams p) {
    __shared__ float red[40];
    RowReduce<WARP_ROW> rr{red};
    const int lane = threadIdx.x & 31;
    const int tpr = WARP_ROW ? 32 : blockDim.x;                 // threads per row
    const int tid = WARP_ROW ? lane : threadIdx.x;
    const int rows_per_cta = WARP_ROW ? (blockDim.x >> 5) : 1;
    const int row_slot = WARP_ROW ? (threadIdx.x >> 5) : 0;
    const int nvec = p.k >> 3;
    const bool want_fp4 = p.fp4_codes != nullptr;
    const bool want_i8 = p.i8_codes != nullptr;
    const float g = want_fp4 ? *p.g : 1.0f;
    const int stride = gridDim.x * rows_per_cta;
    float cta_amax = 0.0f;

    int row = blockIdx.x * rows_per_cta + row_slot;
    uint4 v[NV];
    load_row<NV>(v, p.X + (size_t)row * p.ldx, tid, tpr, nvec, row < p.m);
    // WARP_ROW warps run independent row sequences; CTA rows iterate uniformly
    while (WARP_ROW ? (row < p.m) : (row < p.m)) {
        const int next = row + stride;
        uint4 nv[NV];   // prefetch the next row while this one is processed
        load_row<NV>(nv, p.X + (size_t)next * p.ldx, tid, tpr, nvec, next < p.m);
        if (p.flags & DMPQ_QF_LAYERNORM) {
            // h = bf16((x - mean) * (1/sqrt(var + eps))), var = mean((x - mean)^2)  (glue, R13)
            f2 s2 = f2make(0.0f, 0.0f);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                s2 = add2(s2, add2(bf16x2_to_f2(v[i].x), bf16x2_to_f2(v[i].y)));
                s2 = add2(s2, add2(bf16x2_to_f2(v[i].z), bf16x2_to_f2(v[i].w)));
            }
            const float mean = __fdiv_rn(rr.sum(__fadd_rn(f2lo(s2), f2hi(s2))), (float)p.k);
            const f2 mean2 = f2make(mean, mean);
            f2 q2 = f2make(0.0f, 0.0f);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                if (tid + i * tpr >= nvec) continue;
                const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const f2 d = add2(bf16x2_to_f2(w[j]), f2make(-mean, -mean));
                    q2 = add2(q2, mul2(d, d));
                }
            }
            const float var = __fdiv_rn(rr.sum(__fadd_rn(f2lo(q2), f2hi(q2))), (float)p.k);
            const float rstd = __frcp_rn(__fsqrt_rn(__fadd_rn(var, p.ln_eps)));
            const f2 rstd2 = f2make(rstd, rstd);
            (void)mean2;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int vi = tid + i * tpr;
                uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    w[j] = pack_bf16x2_f2(mul2(add2(bf16x2_to_f2(w[j]), f2make(-mean, -mean)), rstd2));
                v[i] = (vi < nvec) ? make_uint4(w[0], w[1], w[2], w[3]) : make_uint4(0, 0, 0, 0);
                if ((p.flags & DMPQ_QF_WRITE_H) && vi < nvec)
                    *reinterpret_cast<uint4*>(p.h_out + (size_t)row * p.ldh + (size_t)vi * 8) = v[i];
            }
        }
        float vmax[NV];
        float tmax = 0.0f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            vmax[i] = vec_absmax(v[i]);
            tmax = fmaxf(tmax, vmax[i]);
        }
        cta_amax = fmaxf(cta_amax, tmax);

        if (want_fp4) {
            uint8_t* sf_row = p.fp4_sf + (size_t)(row >> 7) * p.kc4 * 512 + (row & 31) * 16 + ((row & 127) >> 5) * 4;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int vi = tid + i * tpr;
                // a_b: max over the 16-element block = this vector and its pair lane
                const float a_b = fmaxf(vmax[i], __shfl_xor_sync(0xffffffffu, vmax[i], 1));
                const float raw = __fdiv_rn(__fdiv_rn(a_b, 6.0f), g);
                const uint32_t sb = e4m3_rn_satfinite(raw);
                const float eff = __fmul_rn(e4m3_decode(sb), g);
                const float rcp = eff > 0.0f ? __frcp_rn(eff) : 0.0f;
                const uint32_t codes = vec_e2m1(v[i], f2make(rcp, rcp));
                // gather the 4 block scales of this 64-element group (lanes 8q, 8q+2, 8q+4, 8q+6)
                const int base = lane & ~7;
                const uint32_t s0 = __shfl_sync(0xffffffffu, sb, base + 0);
                const uint32_t s1 = __shfl_sync(0xffffffffu, sb, base + 2);
                const uint32_t s2 = __shfl_sync(0xffffffffu, sb, base + 4);
                const uint32_t s3 = __shfl_sync(0xffffffffu, sb, base + 6);
                if (vi < nvec) {
                    *reinterpret_cast<uint32_t*>(p.fp4_codes + (size_t)row * (p.k >> 1) + (size_t)vi * 4) = codes;
                    if ((lane & 7) == 0)
                        *reinterpret_cast<uint32_t*>(sf_row + (size_t)(vi >> 3) * 512) = s0 | (s1 << 8) | (s2 << 16) | (s3 << 24);
                }
            }
        }
        if (want_i8) {
            const float a = rr.max(tmax);
            const float rcp = a > 0.0f ? __fdiv_rn(127.0f, a) : 0.0f;
            if (tid == 0) p.i8_scale[row] = a > 0.0f ? __fdiv_rn(a, 127.0f) : 1.0f;
            const f2 rcp2 = f2make(rcp, rcp);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int vi = tid + i * tpr;
                const uint2 c = vec_int8(v[i], rcp2);
                if (vi < nvec) *reinterpret_cast<uint2*>(p.i8_codes + (size_t)row * p.k + (size_t)vi * 8) = c;
            }
        }
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = nv[i];
        row = next;
    }
    // zero the scale rows that pad m up to a multiple of 128 (read by the GEMM's M tail)
    if (want_fp4) {
        const int pad_rows = p.m_pad - p.m;
        const int words_per_row = p.kc4;  // one 32-bit word per (row, atom)
        for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < pad_rows * words_per_row;
             idx += gridDim.x * blockDim.x) {
            const int r = p.m + idx / words_per_row, c4 = idx % words_per_row;
            uint8_t* sf_row = p.fp4_sf + (size_t)(r >> 7) * p.kc4 * 512 + (r & 31) * 16 + ((r & 127) >> 5) * 4;
            *reinterpret_cast<uint32_t*>(sf_row + (size_t)c4 * 512) = 0u;
        }
    }
    if (p.amax_out) {
        float am = warp_max(cta_amax);
        if (lane == 0) atomic_max_nonneg(p.amax_out, am);
    }
}

// ---------------------------------------------------------------------------------------------
// Hadamard-smoothed variant (R14): every 128-element block of the (LN'd) row is rotated
// by the normalized Sylvester FHT before quantization. A block spans 16 consecutive lanes x 8
// elements: stages h = 1, 2, 4 are in-thread, h = 8..64 exchange with lane ^ (h/8); the fixed
// stage order and operand order reproduce the oracle's FP32 butterflies bit for bit.
// ---------------------------------------------------------------------------------------------
__device__ __forceinline__ void fht128_vec(float (&y)[8], int lane) {
#pragma unroll
    for (int h = 1; h < 8; h <<= 1) {
#pragma unroll
        for (int e = 0; e < 8; ++e)
            if ((e & h) == 0) {
                const float a = y[e], b = y[e + h];
                y[e] = __fadd_rn(a, b);
                y[e + h] = __fsub_rn(a, b);
            }
    }
#pragma unroll
    for (int s = 1; s < 16; s <<= 1) {            // element stride h = 8*s
        const bool upper = (lane & s) != 0;         // this lane holds the (i + h) elements
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            const float o = __shfl_xor_sync(0xffffffffu, y[e], s);
            y[e] = upper ? __fsub_rn(o, y[e]) : __fadd_rn(y[e], o);
        }
    }
    const float sc = 0.08838834764831845f;          // fl32(1/sqrt(128))
#pragma unroll
    for (int e = 0; e < 8; ++e) y[e] = __fmul_rn(y[e], sc);
}

template <int NV, bool WARP_ROW>
__global__ void __launch_bounds__(256) quant_act_had_kernel(const QuantParams p) {
    __shared__ float red[40];
    RowReduce<WARP_ROW> rr{red};
    const int lane = threadIdx.x & 31;
    const int tpr = WARP_ROW ? 32 : blockDim.x;
    const int tid = WARP_ROW ? lane : threadIdx.x;
    const int rows_per_cta = WARP_ROW ? (blockDim.x >> 5) : 1;
    const int row_slot = WARP_ROW ? (threadIdx.x >> 5) : 0;
    const int nvec = p.k >> 3;
    const bool want_fp4 = p.fp4_codes != nullptr;
    const bool want_i8 = p.i8_codes != nullptr;
    const float g = want_fp4 ? *p.g : 1.0f;
    const int stride = gridDim.x * rows_per_cta;
    float cta_amax = 0.0f;

    int row = blockIdx.x * rows_per_cta + row_slot;
    uint4 v[NV];
    load_row<NV>(v, p.X + (size_t)row * p.ldx, tid, tpr, nvec, row < p.m);
    while (row < p.m) {
        const int next = row + stride;
        uint4 nv[NV];
        load_row<NV>(nv, p.X + (size_t)next * p.ldx, tid, tpr, nvec, next < p.m);
        if (p.flags & DMPQ_QF_LAYERNORM) {
            f2 s2 = f2make(0.0f, 0.0f);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                s2 = add2(s2, add2(bf16x2_to_f2(v[i].x), bf16x2_to_f2(v[i].y)));
                s2 = add2(s2, add2(bf16x2_to_f2(v[i].z), bf16x2_to_f2(v[i].w)));
            }
            const float mean = __fdiv_rn(rr.sum(__fadd_rn(f2lo(s2), f2hi(s2))), (float)p.k);
            f2 q2 = f2make(0.0f, 0.0f);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                if (tid + i * tpr >= nvec) continue;
                const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const f2 d = add2(bf16x2_to_f2(w[j]), f2make(-mean, -mean));
                    q2 = add2(q2, mul2(d, d));
                }
            }
            const float var = __fdiv_rn(rr.sum(__fadd_rn(f2lo(q2), f2hi(q2))), (float)p.k);
            const f2 rstd2 = f2make(__frcp_rn(__fsqrt_rn(__fadd_rn(var, p.ln_eps))), 0.0f);
            const f2 rs = f2make(f2lo(rstd2), f2lo(rstd2));
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int vi = tid + i * tpr;
                uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                for (int j = 0; j < 4; ++j) w[j] = pack_bf16x2_f2(mul2(add2(bf16x2_to_f2(w[j]), f2make(-mean, -mean)), rs));
                v[i] = (vi < nvec) ? make_uint4(w[0], w[1], w[2], w[3]) : make_uint4(0, 0, 0, 0);
                if ((p.flags & DMPQ_QF_WRITE_H) && vi < nvec)
                    *reinterpret_cast<uint4*>(p.h_out + (size_t)row * p.ldh + (size_t)vi * 8) = v[i];
            }
        }
        float y[NV][8];
        float vmax[NV];
        float tmax = 0.0f;
#pragma unroll
        for (int i = 0; i < NV; ++i) {
            const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
            for (int j = 0; j < 4; ++j) { y[i][2 * j] = bf16lo(w[j]); y[i][2 * j + 1] = bf16hi(w[j]); }
            fht128_vec(y[i], lane);
            float mx = 0.0f;
#pragma unroll
            for (int e = 0; e < 8; ++e) mx = fmaxf(mx, fabsf(y[i][e]));
            vmax[i] = (tid + i * tpr < nvec) ? mx : 0.0f;
            tmax = fmaxf(tmax, vmax[i]);
        }
        cta_amax = fmaxf(cta_amax, tmax);
        if (want_fp4) {
            uint8_t* sf_row = p.fp4_sf + (size_t)(row >> 7) * p.kc4 * 512 + (row & 31) * 16 + ((row & 127) >> 5) * 4;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int vi = tid + i * tpr;
                const float a_b = fmaxf(vmax[i], __shfl_xor_sync(0xffffffffu, vmax[i], 1));
                const float raw = __fdiv_rn(__fdiv_rn(a_b, 6.0f), g);
                const uint32_t sb = e4m3_rn_satfinite(raw);
                const float eff = __fmul_rn(e4m3_decode(sb), g);
                const float rcp = eff > 0.0f ? __frcp_rn(eff) : 0.0f;
                const f2 rcp2 = f2make(rcp, rcp);
                uint32_t codes = 0;
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const f2 q = mul2(f2make(y[i][2 * j], y[i][2 * j + 1]), rcp2);
                    codes |= e2m1x2(f2lo(q), f2hi(q)) << (8 * j);
                }
                const int base = lane & ~7;
                const uint32_t s0 = __shfl_sync(0xffffffffu, sb, base + 0);
                const uint32_t s1 = __shfl_sync(0xffffffffu, sb, base + 2);
                const uint32_t s2 = __shfl_sync(0xffffffffu, sb, base + 4);
                const uint32_t s3 = __shfl_sync(0xffffffffu, sb, base + 6);
                if (vi < nvec) {
                    *reinterpret_cast<uint32_t*>(p.fp4_codes + (size_t)row * (p.k >> 1) + (size_t)vi * 4) = codes;
                    if ((lane & 7) == 0)
                        *reinterpret_cast<uint32_t*>(sf_row + (size_t)(vi >> 3) * 512) = s0 | (s1 << 8) | (s2 << 16) | (s3 << 24);
                }
            }
        }
        if (want_i8) {
            const float a = rr.max(tmax);
            const float rcp = a > 0.0f ? __fdiv_rn(127.0f, a) : 0.0f;
            if (tid == 0) p.i8_scale[row] = a > 0.0f ? __fdiv_rn(a, 127.0f) : 1.0f;
            const f2 rcp2 = f2make(rcp, rcp);
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const int vi = tid + i * tpr;
                uint32_t out[2];
#pragma unroll
                for (int hh = 0; hh < 2; ++hh) {
                    const f2 q0 = mul2(f2make(y[i][4 * hh], y[i][4 * hh + 1]), rcp2);
                    const f2 q1 = mul2(f2make(y[i][4 * hh + 2], y[i][4 * hh + 3]), rcp2);
                    uint32_t r;
                    asm("{ .reg .s32 i0, i1, i2, i3; .reg .b32 pp;\n\t"
                        "cvt.rni.s32.f32 i0, %1; cvt.rni.s32.f32 i1, %2; cvt.rni.s32.f32 i2, %3; cvt.rni.s32.f32 i3, %4;\n\t"
                        "cvt.pack.sat.s8.s32.b32 pp, i3, i2, 0; cvt.pack.sat.s8.s32.b32 %0, i1, i0, pp; }"
                        : "=r"(r) : "f"(f2lo(q0)), "f"(f2hi(q0)), "f"(f2lo(q1)), "f"(f2hi(q1)));
                    out[hh] = r;
                }
                if (vi < nvec) *reinterpret_cast<uint2*>(p.i8_codes + (size_t)row * p.k + (size_t)vi * 8) = make_uint2(out[0], out[1]);
            }
        }
#pragma unroll
        for (int i = 0; i < NV; ++i) v[i] = nv[i];
        row = next;
    }
    if (want_fp4) {
        const int pad_rows = p.m_pad - p.m;
        const int words_per_row = p.kc4;
        for (int idx = blockIdx.x * blockDim.x + threadIdx.x; idx < pad_rows * words_per_row; idx += gridDim.x * blockDim.x) {
            const int r = p.m + idx / words_per_row, c4 = idx % words_per_row;
            uint8_t* sf_row = p.fp4_sf + (size_t)(r >> 7) * p.kc4 * 512 + (r & 31) * 16 + ((r & 127) >> 5) * 4;
            *reinterpret_cast<uint32_t*>(sf_row + (size_t)c4 * 512) = 0u;
        }
    }
    if (p.amax_out) {
        float am = warp_max(cta_amax);
        if (lane == 0) atomic_max_nonneg(p.amax_out, am);
    }
}

__global__ void global_scale_kernel(const float* amax, float div, float* g_out, int count) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        float g = __fdiv_rn(amax[i], div);
        g_out[i] = g < 1.17549435e-38f ? 1.17549435e-38f : g;
    }
}

template <int NV, bool WR>
static void launch_quant(const QuantParams& p, int threads, cudaStream_t s) {
    int rows_per_cta = WR ? threads / 32 : 1;
    int ctas_needed = (p.m + rows_per_cta - 1) / rows_per_cta;
    int grid = num_sms() * (WR ? 8 : (2048 / threads));
    if (grid > ctas_needed) grid = ctas_needed;
    if (grid < 1) grid = 1;
    if (p.flags & DMPQ_QF_HADAMARD) quant_act_had_kernel<NV, WR><<<grid, threads, 0, s>>>(p);
    else quant_act_kernel<NV, WR><<<grid, threads, 0, s>>>(p);
}

}  // namespace dmpq

using namespace dmpq;

extern "C" dmpq_status dmpq_quantize_act(const uint16_t* X, int m, int k, int ldx, const dmpq_quant_opts* opts,
                                         dmpq_act* out_i8, dmpq_act* out_fp4, float* amax_out, dmpq_stream_t s) {
    DMPQ_REQUIRE(out_i8 || out_fp4, DMPQ_EINVAL, "dmpq_quantize_act: both outputs are NULL");
    DMPQ_REQUIRE(m >= 0 && k > 0 && k % 64 == 0 && k <= 16384, DMPQ_ESHAPE,
                 "dmpq_quantize_act: need k %% 64 == 0, 0 < k <= 16384, m >= 0 (m=%d k=%d)", m, k);
    DMPQ_REQUIRE(ldx >= k && ldx % 8 == 0, DMPQ_EALIGN, "dmpq_quantize_act: ldx=%d must be >= k and a multiple of 8", ldx);
    DMPQ_REQUIRE(X && aligned16(X), DMPQ_EALIGN, "dmpq_quantize_act: X must be a 16-byte aligned device pointer");
    if (out_i8) {
        DMPQ_REQUIRE(out_i8->fmt == DMPQ_FMT_INT8 && out_i8->m == m && out_i8->k == k, DMPQ_ESHAPE,
                     "dmpq_quantize_act: INT8 output descriptor mismatch");
        DMPQ_REQUIRE(out_i8->codes && out_i8->row_scale && aligned16(out_i8->codes), DMPQ_EALIGN,
                     "dmpq_quantize_act: INT8 output pointers");
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
    p.fp4_codes = out_fp4 ? reinterpret_cast<uint8_t*>(out_fp4->codes) : nullptr;
    p.fp4_sf = out_fp4 ? out_fp4->sf : nullptr;
    p.g = out_fp4 ? out_fp4->g : nullptr;
    p.amax_out = amax_out;
    p.kc4 = ((k / 16) + 3) / 4;
    p.m_pad = (m + 127) / 128 * 128;
    if (m == 0) return DMPQ_OK;
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_quantize_act: needs an sm_100 device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    const int nvec = k / 8;
    if (nvec <= 64) {  // warp per row
        if (nvec <= 32) launch_quant<1, true>(p, 256, st);
        else launch_quant<2, true>(p, 256, st);
    } else {
        int nv = (nvec + 255) / 256;
        int threads = ((nvec + nv - 1) / nv + 31) / 32 * 32;
        switch (nv) {
            case 1: launch_quant<1, false>(p, threads, st); break;
            case 2: launch_quant<2, false>(p, threads, st); break;
            case 3: launch_quant<3, false>(p, threads, st); break;
            case 4: launch_quant<4, false>(p, threads, st); break;
            case 5: launch_quant<5, false>(p, threads, st); break;
            case 6: launch_quant<6, false>(p, threads, st); break;
            case 7: launch_quant<7, false>(p, threads, st); break;
            default: launch_quant<8, false>(p, threads, st); break;
        }
    }
    return check_launch("dmpq_quantize_act");
}

extern "C" dmpq_status dmpq_global_scale(const float* amax, float div, float* g_out, int count, dmpq_stream_t s) {
    DMPQ_REQUIRE(amax && g_out && count >= 0 && div > 0.0f, DMPQ_EINVAL, "dmpq_global_scale: bad arguments");
    if (count == 0) return DMPQ_OK;
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_global_scale: needs an sm_100 device");
    global_scale_kernel<<<(count + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(s)>>>(amax, div, g_out, count);
    return check_launch("dmpq_global_scale");
}
