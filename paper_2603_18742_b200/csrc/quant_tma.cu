// quant_tma.cu — the chunk quantizer of dmpq_quantize_act: online NVFP4 / per-token INT8
// activation quantization (Eq. 2; R2-R6), optionally
// with the online block Hadamard transform (R14), the LayerNorm glue (R13) and the
// PDR input statistics (R15).
//
// Layout. A CTA owns R rows at a time ("row set"); each row is handled by a group of `tpr`
// threads (nch = k/64 chunks rounded up to 16), thread t owning chunk t = 64 consecutive
// elements = one 128-byte line = four NVFP4 blocks = one 32-bit word of the scale-atom
// layout. Rows arrive by TMA (3-D box {64, nch, R}, 128-byte swizzle) into a double-buffered
// shared-memory ring (2-4 row sets deep), so the next row sets stream in while this one is processed, with no
// registers or load instructions spent on prefetching; each thread then reads its own line
// with conflict-free 16-byte loads (the swizzle spreads 8 consecutive lines over all banks).
// Hadamard: FHT stages h = 1..32 run in registers on packed fp32 pairs; stage h = 64 pairs
// chunk t with chunk t^1 (the neighbouring lane) through the two threads' own smem lines;
// no normalization (the packed weights carry the exact 2^-7, R14).
// Row reductions (LN mean/var, INT8 row max, PDR sums) are fixed-order: 16-lane segment
// shuffles, then the row's segments summed in order after one CTA barrier (deterministic).
#include <algorithm>
#include <mutex>

#include "fastmath.cuh"
#include "quant.cuh"
#include "sm100.cuh"
#include "tmap.cuh"

namespace dmpq {

using namespace sm100;

namespace {

constexpr int MAX_THREADS = 512;
constexpr int MAX_SEG = MAX_THREADS / 16;
constexpr int MAX_SMEM = 112 * 1024;

__device__ __forceinline__ void sts_f32(uint32_t a, float v) { asm volatile("st.shared.f32 [%0], %1;" ::"r"(a), "f"(v) : "memory"); }
__device__ __forceinline__ float lds_f32(uint32_t a) {
    float v;
    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(a) : "memory");
    return v;
}

struct SegReduce {
    uint32_t red;   // shared address of [8 slots][MAX_SEG] floats
    int seg0, nseg;
    __device__ __forceinline__ float sum(float v, int slot) const {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((threadIdx.x & 15) == 0) sts_f32(red + 4u * (slot * MAX_SEG + (threadIdx.x >> 4)), v);
        __syncthreads();
        float t = 0.0f;
        for (int i = 0; i < nseg; ++i) t = __fadd_rn(t, lds_f32(red + 4u * (slot * MAX_SEG + seg0 + i)));
        return t;
    }
    // two sums in one barrier (slots `slot` and `slot + 1`)
    __device__ __forceinline__ void sum2(float& a, float& b, int slot) const {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {
            a = __fadd_rn(a, __shfl_xor_sync(0xffffffffu, a, o));
            b = __fadd_rn(b, __shfl_xor_sync(0xffffffffu, b, o));
        }
        if ((threadIdx.x & 15) == 0) {
            sts_f32(red + 4u * (slot * MAX_SEG + (threadIdx.x >> 4)), a);
            sts_f32(red + 4u * ((slot + 1) * MAX_SEG + (threadIdx.x >> 4)), b);
        }
        __syncthreads();
        float ta = 0.0f, tb = 0.0f;
        for (int i = 0; i < nseg; ++i) {
            ta = __fadd_rn(ta, lds_f32(red + 4u * (slot * MAX_SEG + seg0 + i)));
            tb = __fadd_rn(tb, lds_f32(red + 4u * ((slot + 1) * MAX_SEG + seg0 + i)));
        }
        a = ta;
        b = tb;
    }
    __device__ __forceinline__ float max(float v, int slot) const {
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
        if ((threadIdx.x & 15) == 0) sts_f32(red + 4u * (slot * MAX_SEG + (threadIdx.x >> 4)), v);
        __syncthreads();
        float t = 0.0f;
        for (int i = 0; i < nseg; ++i) t = fmaxf(t, lds_f32(red + 4u * (slot * MAX_SEG + seg0 + i)));
        return t;
    }
};

__device__ __forceinline__ void tma_load_3d(uint32_t dst, const void* tmap, int x, int y, int z, uint32_t bar) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];"
        ::"r"(dst), "l"(tmap), "r"(x), "r"(y), "r"(z), "r"(bar)
        : "memory");
}

__device__ __forceinline__ uint32_t lds32(uint32_t a) {
    uint32_t v;
    asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
    return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t a) {
    uint4 v;
    asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ void sts_f2x2(uint32_t a, f2 x, f2 y) {
    asm volatile("st.shared.v2.b64 [%0], {%1, %2};" ::"r"(a), "l"(x.v), "l"(y.v) : "memory");
}
__device__ __forceinline__ void lds_f2x2(uint32_t a, f2& x, f2& y) {
    asm volatile("ld.shared.v2.b64 {%0, %1}, [%2];" : "=l"(x.v), "=l"(y.v) : "r"(a));
}
__device__ __forceinline__ f2 abs2(f2 a) { f2 r; r.v = a.v & 0x7FFFFFFF7FFFFFFFull; return r; }

// |x| maximum of 16 values (8 packed pairs), exact
__device__ __forceinline__ float absmax8p(const f2* y) {
    float m = 0.0f;
#pragma unroll
    for (int e = 0; e < 8; ++e) m = fmaxf(m, fmaxf(fabsf(f2lo(y[e])), fabsf(f2hi(y[e]))));
    return m;
}

// FHT stages h = 1 (within each pair), h = 2..32 (between pairs p and p + h/2): one FP32
// add/sub per butterfly in the oracle's order (R14).
__device__ __forceinline__ void fht_stages_1_32(f2 (&Y)[32]) {
#pragma unroll
    for (int p = 0; p < 32; ++p) {
        const float a = f2lo(Y[p]), b = f2hi(Y[p]);
        Y[p] = f2make(__fadd_rn(a, b), __fsub_rn(a, b));
    }
#pragma unroll
    for (int hp = 1; hp < 32; hp <<= 1) {
#pragma unroll
        for (int p = 0; p < 32; ++p) {
            if (p & hp) continue;
            const f2 a = Y[p], b = Y[p + hp];
            Y[p] = add2(a, b);
            Y[p + hp] = sub2(a, b);
        }
    }
}

template <bool HAD>
__global__ void __launch_bounds__(MAX_THREADS) quant_tma_kernel(const QuantParams p, const __grid_constant__ CUtensorMap tmX,
                                                                  int tpr, int R, int set_stride, int nbuf) {
    extern __shared__ uint8_t qsm_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(qsm_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t red = sbase + nbuf * set_stride;
    const uint32_t bar0 = red + 8 * MAX_SEG * 4;   // nbuf mbarriers

    const int tid = threadIdx.x, lane = tid & 31;
    const int grp = tid / tpr, t = tid - grp * tpr;
    const int nch = p.k >> 6;
    const bool cvalid = t < nch;
    const int nsets = (p.m + R - 1) / R;
    const int iters = (int)blockIdx.x < nsets ? (nsets - (int)blockIdx.x + (int)gridDim.x - 1) / (int)gridDim.x : 0;
    const uint32_t tx_bytes = (uint32_t)(R * nch * 128);
    const SegReduce sr{red, grp * (tpr >> 4), tpr >> 4};
    const bool want_fp4 = p.fp4_codes != nullptr, want_i8 = p.i8_codes != nullptr;
    const bool ln = (p.flags & DMPQ_QF_LAYERNORM) != 0, write_h = (p.flags & DMPQ_QF_WRITE_H) != 0;
    const bool pdr = p.row_abs_sum != nullptr || p.amax_in != nullptr;

    // NVFP4 block-scale constants; the fast exact path needs g in [2^-90, 2^90] and the
    // block maxima in [a_lo, a_hi] (then a/6, a/(6g) and s*g stay in [2^-100, 2^100], the
    // range fastmath_check verifies exhaustively); other blocks use the IEEE intrinsics.
    const float g = want_fp4 ? *p.g : 1.0f;
    const bool g_ok = g >= 8.0779356e-28f && g <= 1.2379400e27f;   // [2^-90, 2^90]
    const float a_lo = fmaxf(6.3108872e-30f, __fmul_rn(g, 6.3108872e-30f));   // max(2^-97, g 2^-97)
    const float a_hi = fminf(FM_HI, __fmul_rn(g, 5.0706024e30f));            // min(2^100, g 2^102)
    const float rg = g_ok ? recip_refined(g) : 0.0f;
    const f2 g2 = f2make(g, g), ng2 = f2make(-g, -g), rg2 = f2make(rg, rg);
    const f2 n6 = f2make(-6.0f, -6.0f), r6 = f2make(0.16666667163372039795f, 0.16666667163372039795f);

    if (tid == 0) {
        prefetch_tmap(&tmX);
        for (int j = 0; j < nbuf; ++j) {
            mbar_init(bar0 + 8 * j, 1);                                 // full: TMA bytes landed
            mbar_init(bar0 + 8 * (nbuf + j), (blockDim.x + 31) >> 5);   // empty: every warp done with it
        }
        fence_barrier_init();
    }
    __syncthreads();
    if (tid == 0) {
        for (int j = 0; j < nbuf && j < iters; ++j) {
            mbar_arrive_expect_tx(bar0 + 8 * j, tx_bytes);
            tma_load_3d(sbase + j * set_stride, &tmX, 0, 0, ((int)blockIdx.x + j * (int)gridDim.x) * R, bar0 + 8 * j);
        }
    }
    float my_amax = 0.0f, my_amax_in = 0.0f;

    for (int it = 0; it < iters; ++it) {
        const int b = it % nbuf;
        const int set = (int)blockIdx.x + it * (int)gridDim.x;
        const int row = set * R + grp;
        const bool row_live = row < p.m;
        const bool live = row_live && cvalid;
        const int s0 = (it & 1) * 4;   // reduction slots of this iteration
        // refill the buffer of the previous iteration once every warp has released it (only
        // thread 0 waits; the other warps run ahead), keeping nbuf - 1 row sets in flight
        if (tid == 0 && it >= 1 && it - 1 + nbuf < iters) {
            const int pb = (it - 1) % nbuf;
            mbar_wait(bar0 + 8 * (nbuf + pb), ((it - 1) / nbuf) & 1);
            mbar_arrive_expect_tx(bar0 + 8 * pb, tx_bytes);
            tma_load_3d(sbase + pb * set_stride, &tmX, 0, 0, (set - (int)gridDim.x + nbuf * (int)gridDim.x) * R,
                        bar0 + 8 * pb);
        }
        mbar_wait(bar0 + 8 * b, (it / nbuf) & 1);
        const uint32_t L = (uint32_t)(grp * nch + t);
        const uint32_t line = sbase + b * set_stride + L * 128, sw = L & 7;

        f2 Y[32];
        if (cvalid) {
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const uint4 v = lds128(line + ((u ^ sw) << 4));
                Y[4 * u] = bf16x2_to_f2(v.x);
                Y[4 * u + 1] = bf16x2_to_f2(v.y);
                Y[4 * u + 2] = bf16x2_to_f2(v.z);
                Y[4 * u + 3] = bf16x2_to_f2(v.w);
            }
        } else {
#pragma unroll
            for (int q = 0; q < 32; ++q) Y[q] = f2make(0.0f, 0.0f);
        }

        if (ln) {
            // h = bf16((x - mean) * (1/sqrt(var + eps))), var = mean((x - mean)^2)  (glue, R13).
            // One pass and one reduction: sums of d = x - c and d^2 around the row's first
            // element c (read straight from the staged row), mean = c + S1/k,
            // var = S2/k - (S1/k)^2 (shifted data keeps the cancellation small).
            const uint32_t L0 = (uint32_t)(grp * nch);
            const float c = bf16lo(lds32(sbase + b * set_stride + L0 * 128 + ((0u ^ (L0 & 7)) << 4)));
            const f2 nc = f2make(-c, -c);
            f2 s1 = f2make(0.0f, 0.0f), s2 = f2make(0.0f, 0.0f);
            if (cvalid) {
#pragma unroll
                for (int q = 0; q < 32; ++q) {
                    const f2 d = add2(Y[q], nc);
                    s1 = add2(s1, d);
                    s2 = fma2(d, d, s2);
                }
            }
            float S1 = __fadd_rn(f2lo(s1), f2hi(s1)), S2 = __fadd_rn(f2lo(s2), f2hi(s2));
            sr.sum2(S1, S2, s0 + 0);
            const float md = __fdiv_rn(S1, (float)p.k);
            const float mean = __fadd_rn(c, md);
            const f2 nm = f2make(-mean, -mean);
            const float var = fmaxf(__fsub_rn(__fdiv_rn(S2, (float)p.k), __fmul_rn(md, md)), 0.0f);
            const float rstd = __frcp_rn(__fsqrt_rn(__fadd_rn(var, p.ln_eps)));
            const f2 rs = f2make(rstd, rstd);
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                uint32_t w[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    w[j] = cvalid ? pack_bf16x2_f2(mul2(add2(Y[4 * u + j], nm), rs)) : 0u;
                    Y[4 * u + j] = bf16x2_to_f2(w[j]);
                }
                if (write_h && live)
                    *reinterpret_cast<uint4*>(p.h_out + (size_t)row * p.ldh + (size_t)t * 64 + u * 8) =
                        make_uint4(w[0], w[1], w[2], w[3]);
            }
        }
        if (pdr) {   // PDR outlier statistics of the layer input (R15), before any rotation
            f2 sa = f2make(0.0f, 0.0f);
            float mx = 0.0f;
#pragma unroll
            for (int q = 0; q < 32; ++q) {
                const f2 a = abs2(Y[q]);
                sa = add2(sa, a);
                mx = fmaxf(mx, fmaxf(f2lo(a), f2hi(a)));
            }
            my_amax_in = fmaxf(my_amax_in, mx);
            const float rsum = sr.sum(__fadd_rn(f2lo(sa), f2hi(sa)), s0 + 3);
            if (t == 0 && row_live && p.row_abs_sum) p.row_abs_sum[row] = rsum;
        }

        if constexpr (HAD) {
            fht_stages_1_32(Y);
            // h = 64: lower lane keeps a + b, upper lane gets a - b = fma(-1, b, a) (exact
            // product, one rounding), exchanged through the two threads' own smem lines in
            // four 64-byte quarters. No normalization: the weights carry 2^-7 (R14).
            const uint32_t pl = sbase + b * set_stride + (L ^ 1u) * 128, psw = (L ^ 1u) & 7;
            const f2 sg = (t & 1) ? f2make(-1.0f, -1.0f) : f2make(1.0f, 1.0f);
#pragma unroll
            for (int h = 0; h < 4; ++h) {   // four 64-byte quarters (keeps the partner values to 16 registers)
                if (cvalid) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) sts_f2x2(line + ((u ^ sw) << 4), Y[8 * h + 2 * u], Y[8 * h + 2 * u + 1]);
                }
                __syncwarp();
                f2 O[8];
                if (cvalid) {
#pragma unroll
                    for (int u = 0; u < 4; ++u) lds_f2x2(pl + ((u ^ psw) << 4), O[2 * u], O[2 * u + 1]);
                } else {
#pragma unroll
                    for (int u = 0; u < 8; ++u) O[u] = f2make(0.0f, 0.0f);
                }
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 8; ++i) Y[8 * h + i] = fma2(sg, Y[8 * h + i], O[i]);
            }
        }

        // per-16-block |y| maxima and this thread's maximum
        float a[4];
#pragma unroll
        for (int bb = 0; bb < 4; ++bb) a[bb] = absmax8p(&Y[8 * bb]);
        const float tmax = fmaxf(fmaxf(a[0], a[1]), fmaxf(a[2], a[3]));
        my_amax = fmaxf(my_amax, tmax);

        if (want_fp4 && live) {
            const float lo = fminf(fminf(a[0], a[1]), fminf(a[2], a[3]));
            uint32_t sfw;
            float r[4];
            if (g_ok && lo >= a_lo && tmax <= a_hi) {
                // raw = fl(fl(a/6)/g), s = E4M3(raw), eff = fl(s g), r = fl(1/eff): exact, 2 blocks per op
                const f2 A01 = f2make(a[0], a[1]), A23 = f2make(a[2], a[3]);
                const f2 raw01 = div2_fast(div2_fast(A01, n6, r6), ng2, rg2);
                const f2 raw23 = div2_fast(div2_fast(A23, n6, r6), ng2, rg2);
                const uint32_t s01 = e4m3x2(raw01), s23 = e4m3x2(raw23);
                const f2 e01 = mul2(e4m3x2_decode(s01), g2), e23 = mul2(e4m3x2_decode(s23), g2);
                const f2 r01 = rcp2_fast(e01), r23 = rcp2_fast(e23);
                r[0] = f2lo(e01) > 0.0f ? f2lo(r01) : 0.0f;
                r[1] = f2hi(e01) > 0.0f ? f2hi(r01) : 0.0f;
                r[2] = f2lo(e23) > 0.0f ? f2lo(r23) : 0.0f;
                r[3] = f2hi(e23) > 0.0f ? f2hi(r23) : 0.0f;
                sfw = s01 | (s23 << 16);
            } else {
                sfw = 0;
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) sfw |= nvfp4_block_scale(a[bb], g, r[bb]) << (8 * bb);
            }
            uint32_t c[8];
#pragma unroll
            for (int bb = 0; bb < 4; ++bb) {
                const f2 r2 = f2make(r[bb], r[bb]);
                const f2* y = &Y[8 * bb];
                c[2 * bb] = e2m1x8(mul2(y[0], r2), mul2(y[1], r2), mul2(y[2], r2), mul2(y[3], r2));
                c[2 * bb + 1] = e2m1x8(mul2(y[4], r2), mul2(y[5], r2), mul2(y[6], r2), mul2(y[7], r2));
            }
            uint4* cp = reinterpret_cast<uint4*>(p.fp4_codes + (size_t)row * (p.k >> 1) + (size_t)t * 32);
            cp[0] = make_uint4(c[0], c[1], c[2], c[3]);
            cp[1] = make_uint4(c[4], c[5], c[6], c[7]);
            *reinterpret_cast<uint32_t*>(sf_row_ptr(p.fp4_sf, p.kc4, row) + (size_t)t * 512) = sfw;
        }
        if (want_i8) {
            const float am = sr.max(tmax, s0 + 2);
            const float rcp = am > 0.0f ? __fdiv_rn(127.0f, am) : 0.0f;
            if (t == 0 && row_live) p.i8_scale[row] = am > 0.0f ? __fdiv_rn(am, 127.0f) : 1.0f;
            if (live) {
                const f2 r2 = f2make(rcp, rcp);
                uint4* op = reinterpret_cast<uint4*>(p.i8_codes + (size_t)row * p.k + (size_t)t * 64);
#pragma unroll
                for (int j = 0; j < 4; ++j)   // 16 elements -> one 16-byte store
                    op[j] = make_uint4(int8x4(mul2(Y[8 * j], r2), mul2(Y[8 * j + 1], r2)),
                                       int8x4(mul2(Y[8 * j + 2], r2), mul2(Y[8 * j + 3], r2)),
                                       int8x4(mul2(Y[8 * j + 4], r2), mul2(Y[8 * j + 5], r2)),
                                       int8x4(mul2(Y[8 * j + 6], r2), mul2(Y[8 * j + 7], r2)));
            }
        }
        // release buffer b: this warp's reads and exchange writes are done (the generic-proxy
        // writes are ordered before the TMA refill by the proxy fence + mbarrier release/acquire)
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(bar0 + 8 * (nbuf + b));
    }
    // zero the scale rows that pad m up to a multiple of 128 (read by the GEMM's M tail)
    if (want_fp4) {
        const int pad_rows = p.m_pad - p.m;
        for (int idx = blockIdx.x * blockDim.x + tid; idx < pad_rows * p.kc4; idx += gridDim.x * blockDim.x) {
            const int r = p.m + idx / p.kc4, c4 = idx % p.kc4;
            *reinterpret_cast<uint32_t*>(sf_row_ptr(p.fp4_sf, p.kc4, r) + (size_t)c4 * 512) = 0u;
        }
    }
    if (p.amax_out) {
        const float am = warp_max(my_amax);
        if (lane == 0) atomic_max_nonneg(p.amax_out, am);
    }
    if (p.amax_in) {
        const float am = warp_max(my_amax_in);
        if (lane == 0) atomic_max_nonneg(p.amax_in, am);
    }
}

// 3-D view of X: {64 elements, nch lines, m rows}, box {64, nch, R}, 128-byte swizzle.
bool make_tmap_x(CUtensorMap* tm, const void* base, int m, int nch, int ldx, int R) {
    auto enc = tmap_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {64, (cuuint64_t)nch, (cuuint64_t)m};
    cuuint64_t strides[2] = {128, (cuuint64_t)ldx * 2};
    cuuint32_t box[3] = {64, (cuuint32_t)nch, (cuuint32_t)R};
    cuuint32_t estr[3] = {1, 1, 1};
    return enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims, strides, box, estr,
               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <bool HAD>
int ctas_per_sm(int threads, int smem) {
    static std::mutex mu;
    static int cache_threads[8] = {0}, cache_smem[8] = {0}, cache_n[8] = {0};
    std::lock_guard<std::mutex> lk(mu);
    for (int i = 0; i < 8; ++i)
        if (cache_threads[i] == threads && cache_smem[i] == smem) return cache_n[i];
    int n = 1;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, quant_tma_kernel<HAD>, threads, smem) != cudaSuccess || n < 1) {
        cudaGetLastError();
        n = 1;
    }
    for (int i = 0; i < 8; ++i)
        if (cache_threads[i] == 0) { cache_threads[i] = threads; cache_smem[i] = smem; cache_n[i] = n; break; }
    return n;
}

template <bool HAD>
dmpq_status set_attrs() {
    if (cudaFuncSetAttribute(quant_tma_kernel<HAD>, cudaFuncAttributeMaxDynamicSharedMemorySize, MAX_SMEM) != cudaSuccess)
        return check_launch("dmpq_quantize_act(smem attribute)");
    return DMPQ_OK;
}

}  // namespace

dmpq_status prepare_quant_tma() {
    dmpq_status rc = set_attrs<false>();
    if (rc == DMPQ_OK) rc = set_attrs<true>();
    return rc;
}

dmpq_status launch_quant_tma(const QuantParams& p, bool hadamard, cudaStream_t s) {
    static std::once_flag once;
    static dmpq_status prep = DMPQ_OK;
    std::call_once(once, [] { prep = prepare_quant_tma(); });
    if (prep != DMPQ_OK) return prep;
    const int nch = p.k / 64;
    const int tpr = (nch + 15) / 16 * 16;
    int R = 1;
    while ((R * tpr) % 32) ++R;
    while (R * tpr < 128) R *= 2;
    const int threads = R * tpr;
    const int set_bytes = R * nch * 128;
    const int set_stride = (set_bytes + 1023) / 1024 * 1024;
    // ring depth: enough row sets in flight to cover HBM latency (about 48 KB or more per CTA)
    int nbuf = 2;
    while (nbuf < 4 && (nbuf + 1) * set_stride <= 96 * 1024 && nbuf * set_stride < 72 * 1024) ++nbuf;
    const int smem = nbuf * set_stride + 8 * MAX_SEG * 4 + 16 * nbuf + 1024;
    if (threads > MAX_THREADS || smem > MAX_SMEM)
        return set_error(DMPQ_ESHAPE, "dmpq_quantize_act: k=%d exceeds the chunk quantizer's limits", p.k);
    CUtensorMap tm;
    if (!make_tmap_x(&tm, p.X, p.m, nch, p.ldx, R))
        return set_error(DMPQ_ECUDA, "dmpq_quantize_act: cuTensorMapEncodeTiled failed");
    const int nsets = (p.m + R - 1) / R;
    const int per_sm = hadamard ? ctas_per_sm<true>(threads, smem) : ctas_per_sm<false>(threads, smem);
    const int grid = std::max(1, std::min(nsets, per_sm * num_sms()));
    if (hadamard) quant_tma_kernel<true><<<grid, threads, smem, s>>>(p, tm, tpr, R, set_stride, nbuf);
    else quant_tma_kernel<false><<<grid, threads, smem, s>>>(p, tm, tpr, R, set_stride, nbuf);
    return check_launch("dmpq_quantize_act");
}

}  // namespace dmpq
