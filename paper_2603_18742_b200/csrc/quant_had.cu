// quant_had.cu — the Hadamard quantizer of dmpq_quantize_act (DMPQ_QF_HADAMARD): online
// block Hadamard transform (R14) fused with NVFP4 / per-token
// INT8 activation quantization (Eq. 2; R2-R6), the LayerNorm glue (R13)
// and the PDR input statistics (R15).
//
// Layout. One thread owns one whole 128-element Hadamard block (two 128-byte lines), so all
// seven FHT stages run in registers with no lane exchange: stage h = 1 is formed straight from
// the loaded bf16 word by the mixed-precision FHADD.BF16 / FHFMA.BF16 (plain variant; three
// instructions per pair, measured -3.5 % quantizer time in the CogVideoX-5B step) or, after
// LN / the PDR statistics, one FFMA2 per pair (fl(b * (+1, -1) + a) = (fl(a + b), fl(a - b)),
// the exact product leaves one rounding); stages h = 2..64 are packed FADD2 butterflies between
// register pairs — the oracle's fixed
// butterfly order (R14), so codes are bit-exact. A CTA owns R rows at a time ("row set"),
// tpr threads per row (thread t = block t; tpr = blocks per row rounded up to 8, or to 32
// above 32). Rows arrive by TMA into a 2-4 deep shared-memory ring with full/empty mbarriers.
// The 4-D tensor map {64 elements, block, half, row} (strides 256 B, 128 B, ldx) stages a row
// as [half][block][64 elements], so the eight threads of a quarter-warp read eight
// consecutive 128-byte lines: with the 128-byte swizzle, every 16-byte load is bank-conflict
// free. NVFP4 block reciprocals r = fl(1 / fl(dec(s_b) g)) come from a 256-entry shared
// table built once per CTA with the IEEE intrinsics (g is fixed per launch). INT8 codes
// round with the exact 1.5 * 2^23 magic-number RNE on packed FADD2 (bit-equal to cvt.rni for
// |v| < 2^22; here |v| <= 127.5). Row reductions (LN, INT8 row max, PDR sums) are 8-lane
// segment shuffles + one CTA barrier, summed in fixed order (deterministic).
#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "fastmath.cuh"
#include "quant.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace dmpq {

using namespace sm100;

namespace {

constexpr int HT_MAX = 128;                 // threads per CTA (max)
constexpr int H_MAX_SEG = HT_MAX / 8;       // 8-lane reduction segments per CTA
constexpr int H_MAX_SMEM = 112 * 1024;

__device__ __forceinline__ void hsts_f32(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory"); }
__device__ __forceinline__ float hlds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}
__device__ __forceinline__ uint4 hlds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ float rtab_lookup(uint32_t a) {
    float v;
    asm("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ f2 habs2(f2 a) { f2 r; r.v = a.v & 0x7FFFFFFF7FFFFFFFull; return r; }

#ifndef DMPQ_HAD_S1_MIXED
#define DMPQ_HAD_S1_MIXED 1   // plain variant: FHT stage 1 by the mixed bf16/fp32 add + FMA on load (0: unpack + FFMA2)
#endif
// FHT stage h = 1 (R14) of the bf16 pair w = [b:a], straight from the packed word:
// (fl(a + b), fl(a - b)) by the sm_100 mixed-precision add / FMA (FHADD.BF16 / FHFMA.BF16:
// bf16 operand, fp32 operand and result, one rounding; b * -1 is exact).
__device__ __forceinline__ f2 had_stage1_bf16x2(uint32_t w) {
    float s, d;
    asm("{\n\t.reg .b16 lo, hi, m1;\n\t.reg .f32 a;\n\tmov.b32 {lo, hi}, %2;\n\tmov.b16 m1, 0xBF80;\n\t"
        "shl.b32 a, %2, 16;\n\tadd.rn.f32.bf16 %0, hi, a;\n\tfma.rn.f32.bf16 %1, hi, m1, a;\n\t}"
        : "=f"(s), "=f"(d) : "r"(w));
    return f2make(s, d);
}

__device__ __forceinline__ void tma_load_4d(uint32_t dst, const void* tmap, int x, int y, int z, int w, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, %5}], [%6];"
        ::"r"(dst), "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(w), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void tma_load_3d_h(uint32_t dst, const void* tmap, int x, int y, int z, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(dst), "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}

// Fixed-order row reductions over 8-lane segments (a row = tpr / 8 segments).
struct Seg8 {
    uint32_t red;   // shared address of [8 slots][stride] floats
    int seg0, nseg;
    int stride = H_MAX_SEG;
    __device__ __forceinline__ float sum(float v, int slot) const {
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((threadIdx.x & 7) == 0) hsts_f32(red + 4u * (slot * stride + (threadIdx.x >> 3)), v);
        __syncthreads();
        float t = 0.0f;
        for (int i = 0; i < nseg; ++i) t = __fadd_rn(t, hlds_f32(red + 4u * (slot * stride + seg0 + i)));
        return t;
    }
    __device__ __forceinline__ void sum2(float& a, float& b, int slot) const {
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) {
            a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = __fadd_rn(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if ((threadIdx.x & 7) == 0) {
            hsts_f32(red + 4u * (slot * stride + (threadIdx.x >> 3)), a);
            hsts_f32(red + 4u * ((slot + 1) * stride + (threadIdx.x >> 3)), b);
        }
        __syncthreads();
        float ta = 0.0f, tb = 0.0f;
        for (int i = 0; i < nseg; ++i) {
            ta = __fadd_rn(ta, hlds_f32(red + 4u * (slot * stride + seg0 + i)));
            tb = __fadd_rn(tb, hlds_f32(red + 4u * ((slot + 1) * stride + seg0 + i)));
        }
        a = ta;
        b = tb;
    }
    __device__ __forceinline__ float max(float v, int slot) const {
#pragma unroll
        for (int o = 4; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((threadIdx.x & 7) == 0) hsts_f32(red + 4u * (slot * stride + (threadIdx.x >> 3)), v);
        __syncthreads();
        float t = 0.0f;
        for (int i = 0; i < nseg; ++i) t = fmaxf(t, hlds_f32(red + 4u * (slot * stride + seg0 + i)));
        return t;
    }
};

// three-input maximum (FMNMX3 on sm_100; |x| operands fold into the instruction's modifiers)
__device__ __forceinline__ float hmax3(float a, float b, float c) {
    float r;
    asm("max.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}
// |x| maximum of 16 values (8 packed pairs), exact: 8 FMNMX3
__device__ __forceinline__ float habsmax8p(const f2* y) {
    float m = hmax3(fabsf(f2lo(y[0])), fabsf(f2hi(y[0])), fabsf(f2lo(y[1])));
#pragma unroll
    for (int e = 1; e < 7; ++e) m = hmax3(m, fabsf(f2hi(y[e])), fabsf(f2lo(y[e + 1])));
    return hmax3(m, fabsf(f2hi(y[7])), 0.0f);
}

// four int8 codes RNE(fl(y * r)) of y = (y01.lo, y01.hi, y23.lo, y23.hi), |fl(y r)| < 2^22:
// fl(v + 1.5 2^23) has ulp 1, so its low byte is the two's complement RNE(v) (ties to even,
// like cvt.rni). The product is an FFMA2 with an opaque zero addend z (read from shared
// memory): ptxas contracts a packed mul.rn feeding an add.rn into one FFMA2 (one rounding,
// not RNE(fl(y r))), but never an FFMA into an add.
__device__ __forceinline__ uint32_t int8x4_magic(f2 y01, f2 y23, f2 r2, f2 z2) {
    const f2 mg = f2make(12582912.0f, 12582912.0f);
    const f2 a = add2(fma2(y01, r2, z2), mg), b = add2(fma2(y23, r2, z2), mg);
    const uint32_t lo = __byte_perm(__float_as_uint(f2lo(a)), __float_as_uint(f2hi(a)), 0x0040);
    const uint32_t hi = __byte_perm(__float_as_uint(f2lo(b)), __float_as_uint(f2hi(b)), 0x0040);
    return __byte_perm(lo, hi, 0x5410);
}

#ifndef DMPQ_HAD_LN_MINB
#define DMPQ_HAD_LN_MINB 3   // CTAs per SM the LN variant is register-limited for (experiments)
#endif
// WH: write h (LN variants only). FMT: 1 NVFP4 only, 2 INT8 only, 3 both, 0 from the pointers;
// + 4: the INT8 output is per-block (one scale per thread's 128-block, R17) instead of per-token.
template <bool LN, bool PDR, bool WH, int FMT = 0>
__global__ void __launch_bounds__(HT_MAX, LN ? DMPQ_HAD_LN_MINB : 3) quant_had_kernel(const QuantParams p, const __grid_constant__ CUtensorMap tmX,
                                                              int tpr, int R, int set_stride, int nbuf, int split) {
    extern __shared__ uint8_t hsm_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(hsm_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t rtab = sbase + nbuf * set_stride;   // 256 fp32 block reciprocals
    const uint32_t red = rtab + 1024;
    const uint32_t bar0 = red + 8 * H_MAX_SEG * 4;   // nbuf full + nbuf empty mbarriers

    const int tid = threadIdx.x, lane = tid & 31;
    const int grp = tid / tpr, t = tid - grp * tpr;
    const int nb = p.k >> 7;   // Hadamard blocks per row
    const bool cvalid = t < nb;
    const int nsets = (p.m + R - 1) / R;
    const int iters = (int)blockIdx.x < nsets ? (nsets - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    const uint32_t tx_bytes = (uint32_t)(R * nb * 256);
    const Seg8 sr{red, grp * (tpr >> 3), tpr >> 3};
    const bool want_fp4 = FMT ? (FMT & 1) != 0 : p.fp4_codes != nullptr;
    const bool want_i8 = FMT ? (FMT & 2) != 0 : p.i8_codes != nullptr;
    const bool i8_block = FMT ? (FMT & 4) != 0 : p.i8_block != 0;

    // NVFP4 block-scale constants: raw = fl(fl(a/6)/g) takes the exact fast division when g is
    // in [2^-90, 2^90] and the block maxima in [a_lo, a_hi] (fastmath.cuh), else __fdiv_rn.
    const float g = want_fp4 ? *p.g : 1.0f;
    const bool g_ok = g >= 8.0779356e-28f && g <= 1.2379400e27f;   // [2^-90, 2^90]
    const float a_lo = fmaxf(6.3108872e-30f, __fmul_rn(g, 6.3108872e-30f));   // max(2^-97, g 2^-97)
    const float a_hi = fminf(FM_HI, __fmul_rn(g, 5.0706024e30f));            // min(2^100, g 2^102)
    const float rg = g_ok ? recip_refined(g) : 0.0f;
    const f2 ng2 = f2make(-g, -g), rg2 = f2make(rg, rg);
    const f2 n6 = f2make(-6.0f, -6.0f), r6 = f2make(0.16666667163372039795f, 0.16666667163372039795f);

    {   // r(s) = fl(1 / fl(dec(s) g)), 0 when the effective scale is 0 (R3/R4, Q7); r(0) = +0
        for (int s = tid; s < 256; s += blockDim.x) {
            const float eff = __fmul_rn(e4m3_decode((uint32_t)s), g);
            hsts_f32(rtab + 4u * s, eff > 0.0f ? __frcp_rn(eff) : 0.0f);
        }
    }
    if (tid == 0) {
        prefetch_tmap(&tmX);
        for (int j = 0; j < nbuf; ++j) {
            mbar_init(bar0 + 8 * j, 1);                                 // full: TMA bytes landed
            mbar_init(bar0 + 8 * (nbuf + j), (blockDim.x + 31) >> 5);   // empty: every warp done with it
        }
        fence_barrier_init();
    }
    __syncthreads();
    auto issue = [&](int j, int set) {
        const uint32_t dst = sbase + j * set_stride;
        mbar_arrive_expect_tx(bar0 + 8 * j, tx_bytes);
        if (split) tma_load_4d(dst, &tmX, 0, 0, 0, set * R, bar0 + 8 * j);
        else tma_load_3d_h(dst, &tmX, 0, 0, set * R, bar0 + 8 * j);
    };
    if (tid == 0)
        for (int j = 0; j < nbuf && j < iters; ++j) issue(j, (int)blockIdx.x + j * (int)gridDim.x);

    // this thread's two lines inside a staged row set: [row][half][block] (split) or
    // [row][line] (3-D fallback: lines 2t, 2t + 1)
    // (threads past the row's last block read the row's first lines: never stored, and their
    // maxima and sums are forced to 0)
    const int tt = cvalid ? t : 0;
    const uint32_t line0 = split ? (uint32_t)(grp * 2 * nb + tt) : (uint32_t)(grp * 2 * nb + 2 * tt);
    const uint32_t lstep = split ? (uint32_t)nb : 1u;
    // byte offset of chunk 0 of each line with the swizzle bits folded in: chunk u of the line is
    // at (buf + x) ^ (u << 4) (buf is 1024-byte aligned, so the add leaves bits 4-6 alone)
    const uint32_t x0 = line0 * 128 + ((line0 & 7) << 4), x1 = (line0 + lstep) * 128 + (((line0 + lstep) & 7) << 4);

    const float zr = hlds_f32(rtab);   // +0, opaque to ptxas (int8x4_magic)
    const f2 z2 = f2make(zr, zr);
    float my_amax = 0.0f, my_amax_in = 0.0f;
    int b = 0;
    uint32_t ph = 0;   // parity of the current buffer's use
    for (int it = 0; it < iters; ++it) {
        const int set = (int)blockIdx.x + it * (int)gridDim.x;
        const int row = set * R + grp;
        const bool row_live = row < p.m;
        const bool live = row_live && cvalid;
        const int s0 = (it & 1) * 4;   // reduction slots of this iteration
        mbar_wait(bar0 + 8 * b, ph);
        const uint32_t buf = sbase + b * set_stride;

        constexpr bool S1_ON_LOAD = DMPQ_HAD_S1_MIXED && !LN && !PDR;
        auto unpack = [](uint32_t w) { return S1_ON_LOAD ? had_stage1_bf16x2(w) : bf16x2_to_f2(w); };
        f2 Y[64];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint4 v = hlds128((buf + x0) ^ (u << 4));
            Y[4 * u] = unpack(v.x);
            Y[4 * u + 1] = unpack(v.y);
            Y[4 * u + 2] = unpack(v.z);
            Y[4 * u + 3] = unpack(v.w);
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const uint4 v = hlds128((buf + x1) ^ (u << 4));
            Y[32 + 4 * u] = unpack(v.x);
            Y[32 + 4 * u + 1] = unpack(v.y);
            Y[32 + 4 * u + 2] = unpack(v.z);
            Y[32 + 4 * u + 3] = unpack(v.w);
        }

        if constexpr (LN) {
            // h = bf16(fl(x rstd - fl(mean rstd))) (glue, R13): one pass of packed raw sums
            // S1 = sum x, S2 = sum x^2 (FP32), mean = S1/k, var = max(S2/k - mean^2, 0).
            f2 s1 = f2make(0.0f, 0.0f), s2 = f2make(0.0f, 0.0f);
#pragma unroll
            for (int q = 0; q < 64; ++q) {
                s1 = add2(s1, Y[q]);
                s2 = fma2(Y[q], Y[q], s2);
            }
            float S1 = cvalid ? __fadd_rn(f2lo(s1), f2hi(s1)) : 0.0f, S2 = cvalid ? __fadd_rn(f2lo(s2), f2hi(s2)) : 0.0f;
            sr.sum2(S1, S2, s0 + 0);
            const float mean = __fdiv_rn(S1, (float)p.k);
            const float var = fmaxf(__fsub_rn(__fdiv_rn(S2, (float)p.k), __fmul_rn(mean, mean)), 0.0f);
            const float rstd = __frcp_rn(__fsqrt_rn(__fadd_rn(var, p.ln_eps)));
            const f2 rs = f2make(rstd, rstd), nmr = f2make(-__fmul_rn(mean, rstd), -__fmul_rn(mean, rstd));
            // bf16 rounding in place (cvt.rn.bf16x2.f32 with a zero low half is the fp32 bit
            // pattern of bf16(v)), fused with the PDR statistics of h and FHT stage h = 1 (R14)
            const f2 pm = f2make(1.0f, -1.0f);
            f2 sa = f2make(0.0f, 0.0f);
            float mx = 0.0f;
#pragma unroll
            for (int u = 0; u < 16; ++u) {
                float hv[8];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int q = 4 * u + j;
                    const f2 v = fma2(Y[q], rs, nmr);
                    const float a = __uint_as_float(pack_bf16x2(0.0f, f2lo(v))), bb = __uint_as_float(pack_bf16x2(0.0f, f2hi(v)));
                    hv[2 * j] = a;
                    hv[2 * j + 1] = bb;
                    if constexpr (PDR) {
                        const f2 ab = habs2(f2make(a, bb));
                        sa = add2(sa, ab);
                        mx = fmaxf(mx, fmaxf(f2lo(ab), f2hi(ab)));
                    }
                    Y[q] = fma2(f2make(bb, bb), pm, f2make(a, a));
                }
                if (WH && live) {
                    uint32_t w[4];
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        w[j] = __byte_perm(__float_as_uint(hv[2 * j]), __float_as_uint(hv[2 * j + 1]), 0x7632);
                    *reinterpret_cast<uint4*>(p.h_out + (size_t)row * p.ldh + (size_t)t * 128 + u * 8) =
                        make_uint4(w[0], w[1], w[2], w[3]);
                }
            }
            if constexpr (PDR) {   // PDR outlier statistics of the layer input h (R15), before the rotation
                my_amax_in = fmaxf(my_amax_in, cvalid ? mx : 0.0f);
                const float rsum = sr.sum(cvalid ? __fadd_rn(f2lo(sa), f2hi(sa)) : 0.0f, s0 + 3);
                if (t == 0 && row_live && p.row_abs_sum) p.row_abs_sum[row] = rsum;
            }
        } else {
            if constexpr (PDR) {   // PDR outlier statistics of the layer input (R15), before the rotation
                f2 sa = f2make(0.0f, 0.0f);
                float mx = 0.0f;
#pragma unroll
                for (int q = 0; q < 64; ++q) {
                    const f2 a = habs2(Y[q]);
                    sa = add2(sa, a);
                    mx = fmaxf(mx, fmaxf(f2lo(a), f2hi(a)));
                }
                my_amax_in = fmaxf(my_amax_in, cvalid ? mx : 0.0f);
                const float rsum = sr.sum(cvalid ? __fadd_rn(f2lo(sa), f2hi(sa)) : 0.0f, s0 + 3);
                if (t == 0 && row_live && p.row_abs_sum) p.row_abs_sum[row] = rsum;
            }
            if constexpr (!S1_ON_LOAD) {   // FHT stage h = 1 inside each pair (R14)
                const f2 pm = f2make(1.0f, -1.0f);
#pragma unroll
                for (int q = 0; q < 64; ++q) {
                    const float a = f2lo(Y[q]), bb = f2hi(Y[q]);
                    Y[q] = fma2(f2make(bb, bb), pm, f2make(a, a));
                }
            }
        }

        // FHT stages h = 2..64 between register pairs (R14)
        {
#pragma unroll
            for (int hp = 1; hp < 64; hp <<= 1) {
#pragma unroll
                for (int q = 0; q < 64; ++q) {
                    if (q & hp) continue;
                    const f2 a = Y[q], bb = Y[q + hp];
                    Y[q] = add2(a, bb);
                    Y[q + hp] = sub2(a, bb);
                }
            }
        }

        // the row set is in registers: release buffer b and (thread 0, once every warp has
        // released it) refill it with row set it + nbuf, so nbuf row sets stay in flight.
        // The proxy fence orders this thread's generic-proxy shared loads before the TMA
        // (async-proxy) refill that the release allows: the compiler hoists the arrive above
        // the transform (it is pure register work), and without the fence the arrive does not
        // wait for loads still in flight — a schedule with the arrive five instructions after
        // the last load lost whole 128-blocks to the refill (~3 in 10^4 blocks, dense-row test).
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar0 + 8 * (nbuf + b));
        if (tid == 0 && it + nbuf < iters) {
            mbar_wait(bar0 + 8 * (nbuf + b), ph);
            issue(b, set + nbuf * (int)gridDim.x);
        }

        // per-16-block |y| maxima and this thread's maximum
        float a[8];
#pragma unroll
        for (int bb = 0; bb < 8; ++bb) a[bb] = habsmax8p(&Y[8 * bb]);
        const float tmax = cvalid ? hmax3(hmax3(a[0], a[1], a[2]), hmax3(a[3], a[4], a[5]), fmaxf(a[6], a[7])) : 0.0f;
        my_amax = fmaxf(my_amax, tmax);

        if (want_fp4 && live) {
            const float lo = fminf(fminf(fminf(a[0], a[1]), fminf(a[2], a[3])), fminf(fminf(a[4], a[5]), fminf(a[6], a[7])));
            uint32_t s[4];   // E4M3 codes of blocks (2j, 2j + 1) in bytes 0, 1
            if (g_ok && lo >= a_lo && tmax <= a_hi) {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    s[j] = e4m3x2(div2_fast(div2_fast(f2make(a[2 * j], a[2 * j + 1]), n6, r6), ng2, rg2));
            } else {
#pragma unroll
                for (int j = 0; j < 4; ++j)
                    s[j] = e4m3_rn_satfinite(__fdiv_rn(__fdiv_rn(a[2 * j], 6.0f), g)) |
                           (e4m3_rn_satfinite(__fdiv_rn(__fdiv_rn(a[2 * j + 1], 6.0f), g)) << 8);
            }
            uint4* cp = reinterpret_cast<uint4*>(p.fp4_codes + (size_t)row * (p.k >> 1) + (size_t)t * 64);
#pragma unroll
            for (int j = 0; j < 4; ++j) {   // blocks 2j, 2j + 1 -> 32 codes -> one 16-byte store
                uint32_t c[4];
#pragma unroll
                for (int e = 0; e < 2; ++e) {
                    const float r = rtab_lookup(rtab + 4u * ((s[j] >> (8 * e)) & 0xFFu));
                    const f2 r2 = f2make(r, r);
                    const f2* y = &Y[16 * j + 8 * e];
                    c[2 * e] = e2m1x8(mul2(y[0], r2), mul2(y[1], r2), mul2(y[2], r2), mul2(y[3], r2));
                    c[2 * e + 1] = e2m1x8(mul2(y[4], r2), mul2(y[5], r2), mul2(y[6], r2), mul2(y[7], r2));
                }
                cp[j] = make_uint4(c[0], c[1], c[2], c[3]);
            }
            uint8_t* sp = sf_row_ptr(p.fp4_sf, p.kc4, row) + (size_t)t * 1024;
            *reinterpret_cast<uint32_t*>(sp) = s[0] | (s[1] << 16);
            *reinterpret_cast<uint32_t*>(sp + 512) = s[2] | (s[3] << 16);
        }
        if (want_i8) {
            // per token: the row maximum over the CTA's segment reduction; per block (R17): this
            // thread's own 128-block maximum, no reduction
            const float am = i8_block ? tmax : sr.max(tmax, s0 + 2);
            const float rcp = am > 0.0f ? __fdiv_rn(127.0f, am) : 0.0f;
            if (i8_block) {
                if (live) p.i8_scale[(size_t)row * nb + t] = am > 0.0f ? __fdiv_rn(am, 127.0f) : 1.0f;
            } else if (t == 0 && row_live) {
                p.i8_scale[row] = am > 0.0f ? __fdiv_rn(am, 127.0f) : 1.0f;
            }
            if (live) {
                const f2 r2 = f2make(rcp, rcp);
                uint4* op = reinterpret_cast<uint4*>(p.i8_codes + (size_t)row * p.k + (size_t)t * 128);
#pragma unroll
                for (int j = 0; j < 8; ++j)   // 16 elements -> one 16-byte store
                    op[j] = make_uint4(int8x4_magic(Y[8 * j], Y[8 * j + 1], r2, z2), int8x4_magic(Y[8 * j + 2], Y[8 * j + 3], r2, z2),
                                       int8x4_magic(Y[8 * j + 4], Y[8 * j + 5], r2, z2), int8x4_magic(Y[8 * j + 6], Y[8 * j + 7], r2, z2));
            }
        }
        if (++b == nbuf) {
            b = 0;
            ph ^= 1u;
        }
    }
    // zero the scale rows that pad m up to a multiple of 128 (read by the GEMM's M tail)
    if (want_fp4) {
        const int pad_rows = p.m_pad - p.m;
        for (int idx = blockIdx.x * blockDim.x + tid; idx < pad_rows * p.kc4; idx += gridDim.x * blockDim.x) {
            const int r = p.m + idx / p.kc4, c4 = idx % p.kc4;
            *reinterpret_cast<uint32_t*>(sf_row_ptr(p.fp4_sf, p.kc4, r) + (size_t)c4 * 512) = 0u;
        }
    }
    // tensor maxima: warp -> CTA in shared memory, one atomic per CTA (order-independent)
    if (p.amax_out || p.amax_in) {
        const float am = warp_max(my_amax), ai = warp_max(my_amax_in);
        const int nw = (int)(blockDim.x + 31) >> 5;
        __syncthreads();   // every row reduction of the loop has read its slots
        if (lane == 0) {
            hsts_f32(red + 4u * (tid >> 5), am);
            hsts_f32(red + 4u * (H_MAX_SEG + (tid >> 5)), ai);
        }
        __syncthreads();
        if (tid == 0) {
            float m0 = 0.0f, m1 = 0.0f;
            for (int w = 0; w < nw; ++w) {
                m0 = fmaxf(m0, hlds_f32(red + 4u * w));
                m1 = fmaxf(m1, hlds_f32(red + 4u * (H_MAX_SEG + w)));
            }
            if (p.amax_out) atomic_max_nonneg(p.amax_out, m0);
            if (p.amax_in) atomic_max_nonneg(p.amax_in, m1);
        }
    }
}

// 4-D view of X: {64 elements, nb blocks (256 B), 2 halves (128 B), m rows}, box {64, nb, 2, R}:
// a row lands in shared memory as [half][block][64 elements]. 128-byte swizzle.
bool make_tmap_had_split(CUtensorMap* tm, const void* base, int m, int nb, int ldx, int R) {
    auto enc = tmap_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[4] = {64, (cuuint64_t)nb, 2, (cuuint64_t)m};
    cuuint64_t strides[3] = {256, 128, (cuuint64_t)ldx * 2};
    cuuint32_t box[4] = {64, (cuuint32_t)nb, 2, (cuuint32_t)R};
    cuuint32_t estr[4] = {1, 1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 3-D fallback {64 elements, 2 nb lines, m rows}, box {64, 2 nb, R}.
bool make_tmap_had_lines(CUtensorMap* tm, const void* base, int m, int nb, int ldx, int R) {
    auto enc = tmap_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {64, (cuuint64_t)(2 * nb), (cuuint64_t)m};
    cuuint64_t strides[2] = {128, (cuuint64_t)ldx * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)(2 * nb), (cuuint32_t)R};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int had_ctas_per_sm(int threads, int smem) {
    static std::mutex mu;
    static int cache_threads[8] = {0}, cache_smem[8] = {0}, cache_n[8] = {0};
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < 8; ++i)
        if (cache_threads[i] == threads && cache_smem[i] == smem) return cache_n[i];
    int n = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, quant_had_kernel<false, false, false>, threads, smem) != cudaSuccess || n < 1) {
        cudaGetLastError();
        n = 1;
    }
    for (int i = 0; i < 8; ++i)
        if (cache_threads[i] == 0) { cache_threads[i] = threads; cache_smem[i] = smem; cache_n[i] = n; break; }
    return n;
}

}  // namespace

dmpq_status prepare_quant_had() {
    const void* kernels[] = {(const void*)quant_had_kernel<false, false, false, 1>, (const void*)quant_had_kernel<false, false, false, 2>,
                             (const void*)quant_had_kernel<false, false, false, 3>, (const void*)quant_had_kernel<true, false, false, 1>,
                             (const void*)quant_had_kernel<true, false, false, 2>,  (const void*)quant_had_kernel<true, false, false, 3>,
                             (const void*)quant_had_kernel<true, false, true>,      (const void*)quant_had_kernel<false, true, false>,
                             (const void*)quant_had_kernel<true, true, false>,      (const void*)quant_had_kernel<true, true, true>,
                             (const void*)quant_had_kernel<false, false, false>,    (const void*)quant_had_kernel<true, false, false>,
                             (const void*)quant_had_kernel<false, false, false, 6>, (const void*)quant_had_kernel<false, false, false, 7>,
                             (const void*)quant_had_kernel<true, false, false, 6>,  (const void*)quant_had_kernel<true, false, false, 7>};
    bool ok = true;
    for (const void* k : kernels)
        ok = ok && cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, H_MAX_SMEM) == cudaSuccess;
    if (!ok)
        return check_launch("dmpq_quantize_act(smem attribute)");
    return DMPQ_OK;
}

dmpq_status launch_quant_had(const QuantParams& p, cudaStream_t s) {
    static std::once_flag once;
    static dmpq_status prep = DMPQ_OK;
    std::call_once(once, [] { prep = prepare_quant_had(); });
    if (prep != DMPQ_OK) return prep;
    const int nb = p.k / 128;
    int tpr = (nb + 7) / 8 * 8;
    if (tpr > 32) tpr = (tpr + 31) / 32 * 32;
    int R = 1;
    while ((R * tpr) % 32) ++R;
    while (R * tpr < 96) R *= 2;
    const int threads = R * tpr;
    const int set_bytes = R * nb * 256;
    const int set_stride = (set_bytes + 1023) / 1024 * 1024;
    int nbuf = 2;
    while (nbuf < 4 && nbuf * set_stride < 32 * 1024) ++nbuf;
    const int smem = nbuf * set_stride + 1024 + 8 * H_MAX_SEG * 4 + 16 * nbuf + 1024;
    if (threads > HT_MAX || smem > H_MAX_SMEM)
        return set_error(DMPQ_ESHAPE, "dmpq_quantize_act: k=%d exceeds the Hadamard quantizer's limits", p.k);
    CUtensorMap tm;
    int split = 1;
    if (!make_tmap_had_split(&tm, p.X, p.m, nb, p.ldx, R)) {
        split = 0;
        if (!make_tmap_had_lines(&tm, p.X, p.m, nb, p.ldx, R))
            return set_error(DMPQ_ECUDA, "dmpq_quantize_act: cuTensorMapEncodeTiled failed");
    }
    const int nsets = (p.m + R - 1) / R;
    const int grid = std::max(1, std::min(nsets, had_ctas_per_sm(threads, smem) * num_sms()));
    const bool ln = (p.flags & DMPQ_QF_LAYERNORM) != 0, pdr = p.row_abs_sum != nullptr || p.amax_in != nullptr;
    const bool wh = ln && (p.flags & DMPQ_QF_WRITE_H) != 0;
#define DMPQ_HAD_LAUNCH(a, b, c) quant_had_kernel<a, b, c><<<grid, threads, smem, s>>>(p, tm, tpr, R, set_stride, nbuf, split)
    if (ln && pdr) { if (wh) DMPQ_HAD_LAUNCH(true, true, true); else DMPQ_HAD_LAUNCH(true, true, false); }
    else if (pdr) DMPQ_HAD_LAUNCH(false, true, false);
    else if (ln && wh) DMPQ_HAD_LAUNCH(true, false, true);
    else {   // the common cases: formats fixed at compile time
        const int fmt = (p.fp4_codes ? 1 : 0) | (p.i8_codes ? 2 : 0);
#define DMPQ_HAD_LAUNCH_F(a, f) quant_had_kernel<a, false, false, f><<<grid, threads, smem, s>>>(p, tm, tpr, R, set_stride, nbuf, split)
        const int f = fmt | (p.i8_codes && p.i8_block ? 4 : 0);
        if (ln) {
            if (f == 1) DMPQ_HAD_LAUNCH_F(true, 1); else if (f == 2) DMPQ_HAD_LAUNCH_F(true, 2);
            else if (f == 3) DMPQ_HAD_LAUNCH_F(true, 3); else if (f == 6) DMPQ_HAD_LAUNCH_F(true, 6);
            else if (f == 7) DMPQ_HAD_LAUNCH_F(true, 7); else DMPQ_HAD_LAUNCH(true, false, false);
        } else {
            if (f == 1) DMPQ_HAD_LAUNCH_F(false, 1); else if (f == 2) DMPQ_HAD_LAUNCH_F(false, 2);
            else if (f == 3) DMPQ_HAD_LAUNCH_F(false, 3); else if (f == 6) DMPQ_HAD_LAUNCH_F(false, 6);
            else if (f == 7) DMPQ_HAD_LAUNCH_F(false, 7); else DMPQ_HAD_LAUNCH(false, false, false);
        }
#undef DMPQ_HAD_LAUNCH_F
    }
#undef DMPQ_HAD_LAUNCH
    return check_launch("dmpq_quantize_act");
}

}  // namespace dmpq
