// quant.cu — dmpq_quantize_act: online NVFP4 / per-token INT8 activation
// quantization (Eq. 2; R2-R6), optionally
// with a fused row LayerNorm prologue (block glue), and dmpq_global_scale.
//
// HBM-bound streaming kernel: each row is held in registers by a group of threads
// (64-element chunks per thread, one 128-byte line each), the next row prefetched
// while the current one is processed; fixed-order reductions (deterministic);
// persistent grid over rows.
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
    float* row_abs_sum;   // PDR statistics (R15): per-row sum |x| of the layer input (pre-rotation)
    float* amax_in;       //                       max |x| of the layer input (pre-rotation)
    int kc4;     // scale-column atoms per 128-row tile: ceil(k/16/4)
    int m_pad;   // rows rounded up to 128 (scale rows to zero-fill)
};

// ---------------------------------------------------------------------------------------------
// Hadamard path (R14). Layout: a row is quantised by a group of `tpr` threads (a multiple of 32); each thread owns
// chunks of 64 consecutive elements (8 x 16-byte loads, one full 128-byte line), chunk
// c = tid + i*tpr. A chunk holds four whole NVFP4 blocks and exactly one 32-bit word of the
// scale-atom layout (c == atom column), so block maxima and the scale store need no lane
// exchange; with the Hadamard option, FHT stages h = 1..32 are in-thread and h = 64 pairs
// lanes (tid ^ 1). Group reductions: warp shuffles, then smem + a named barrier per group.
// ---------------------------------------------------------------------------------------------
struct GroupReduce {
    float* red;      // [8 areas][8 groups][8 warps]
    int tpr, group, warp_in_group, lane;
    __device__ __forceinline__ float sum(float v, int area) {
        v = warp_sum(v);
        if (tpr == 32) return v;
        float* r = red + (area * 8 + group) * 8;
        if (lane == 0) r[warp_in_group] = v;
        named_barrier(1 + group, tpr);
        float t = 0.0f;
        for (int w = 0; w < (tpr >> 5); ++w) t = __fadd_rn(t, r[w]);
        return t;
    }
    __device__ __forceinline__ float max(float v, int area) {
        v = warp_max(v);
        if (tpr == 32) return v;
        float* r = red + (area * 8 + group) * 8;
        if (lane == 0) r[warp_in_group] = v;
        named_barrier(1 + group, tpr);
        float t = 0.0f;
        for (int w = 0; w < (tpr >> 5); ++w) t = fmaxf(t, r[w]);
        return t;
    }
    __device__ __forceinline__ static void named_barrier(int id, int n) {
        asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
    }
};

// bf16 pair (one 32-bit word) -> packed fp32x2 (exact widening)
__device__ __forceinline__ f2 bf16x2_to_f2(uint32_t w) { return f2make(bf16lo(w), bf16hi(w)); }

// |x| max over 8 packed bf16 words (16 elements), in the bf16 domain (exact)
__device__ __forceinline__ float absmax16(const uint32_t* w) {
    uint32_t m;
    asm("{ .reg .b32 a0, a1, a2, a3, a4, a5, a6, a7, t0, t1, t2, t3, u0, u1;\n\t"
        "and.b32 a0, %1, 0x7fff7fff; and.b32 a1, %2, 0x7fff7fff; and.b32 a2, %3, 0x7fff7fff; and.b32 a3, %4, 0x7fff7fff;\n\t"
        "and.b32 a4, %5, 0x7fff7fff; and.b32 a5, %6, 0x7fff7fff; and.b32 a6, %7, 0x7fff7fff; and.b32 a7, %8, 0x7fff7fff;\n\t"
        "max.bf16x2 t0, a0, a1; max.bf16x2 t1, a2, a3; max.bf16x2 t2, a4, a5; max.bf16x2 t3, a6, a7;\n\t"
        "max.bf16x2 u0, t0, t1; max.bf16x2 u1, t2, t3; max.bf16x2 %0, u0, u1; }"
        : "=r"(m) : "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]));
    return fmaxf(bf16lo(m), bf16hi(m));
}

// NVFP4 block scale of Eq. 2 with the two-level scale (R3/R4): returns the E4M3 code, sets rcp = fl(1/eff)
__device__ __forceinline__ uint32_t nvfp4_block_scale(float a_b, float g, float& rcp) {
    const float raw = __fdiv_rn(__fdiv_rn(a_b, 6.0f), g);
    const uint32_t sb = e4m3_rn_satfinite(raw);
    const float eff = __fmul_rn(e4m3_decode(sb), g);
    rcp = eff > 0.0f ? __frcp_rn(eff) : 0.0f;
    return sb;
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

// FHT over the 128-element block held by this thread (64 elements as 32 packed pairs
// Y[p] = (y[2p], y[2p+1])) and its partner lane (tid ^ 1): stage h = 1 within each pair
// (scalar add/sub), stages h = 2..32 between pairs p and p + h/2 (packed FADD2, no register
// moves), h = 64 across the lane pair (two shuffles + one exact FFMA2 per pair), then
// * fl32(1/sqrt(128)). Every butterfly is one FP32 add/sub in the oracle's order (R14).
__device__ __forceinline__ void fht128_chunk(f2 (&Y)[32], bool upper) {
#pragma unroll
    for (int p = 0; p < 32; ++p) {
        const float a = f2lo(Y[p]), b = f2hi(Y[p]);
        Y[p] = f2make(__fadd_rn(a, b), __fsub_rn(a, b));
    }
#pragma unroll
    for (int hp = 1; hp < 32; hp <<= 1) {            // pair stride hp = h/2, h = 2..32
#pragma unroll
        for (int p = 0; p < 32; ++p) {
            if (p & hp) continue;
            const f2 a = Y[p], b = Y[p + hp];
            Y[p] = add2(a, b);
            Y[p + hp] = sub2(a, b);
        }
    }
    // h = 64: lower lane keeps a + b, upper lane gets a - b = fma(-1, b, a) (exact product, one rounding)
    const f2 sg = upper ? f2make(-1.0f, -1.0f) : f2make(1.0f, 1.0f);
    const f2 sc = f2make(0.08838834764831845f, 0.08838834764831845f);   // fl32(1/sqrt(128))
#pragma unroll
    for (int p = 0; p < 32; ++p) {
        const float o0 = __shfl_xor_sync(0xffffffffu, f2lo(Y[p]), 1), o1 = __shfl_xor_sync(0xffffffffu, f2hi(Y[p]), 1);
        Y[p] = mul2(fma2(sg, Y[p], f2make(o0, o1)), sc);
    }
}

template <int NC>
__device__ __forceinline__ void load_chunks(uint4 (&v)[NC][8], const uint16_t* xr, int tid, int tpr, int nch, bool valid) {
#pragma unroll
    for (int i = 0; i < NC; ++i) {
        const int c = tid + i * tpr;
        const bool ok = valid && c < nch;
#pragma unroll
        for (int j = 0; j < 8; ++j)
            v[i][j] = ok ? *reinterpret_cast<const uint4*>(xr + (size_t)c * 64 + j * 8) : make_uint4(0, 0, 0, 0);
    }
}

// Coalesced row load for the chunk layout: the group's threads read 16-byte vectors
// consecutively (lane-contiguous), park them in shared memory (one 16-byte pad per
// 128-byte chunk keeps the later chunk reads at the 4-wavefront minimum), and each
// thread then picks up its own 64-element chunk.
template <int VPT>
__device__ __forceinline__ void load_row_coalesced(uint4 (&pv)[VPT], const uint16_t* xr, int tid, int tpr, int nvec, bool valid) {
#pragma unroll
    for (int j = 0; j < VPT; ++j) {
        const int vi = tid + j * tpr;
        pv[j] = (valid && vi < nvec) ? ldg_stream(xr + (size_t)vi * 8) : make_uint4(0, 0, 0, 0);
    }
}

template <int NC, bool HAD, bool SMEM>
__global__ void __launch_bounds__(256) quant_act_chunk_kernel(const QuantParams p, int tpr) {
    __shared__ float red[8 * 8 * 8];
    const int lane = threadIdx.x & 31;
    const int group = threadIdx.x / tpr, tid = threadIdx.x % tpr;
    const int groups = blockDim.x / tpr;
    GroupReduce gr{red, tpr, group, tid >> 5, lane};
    const int nch = p.k >> 6;
    const bool want_fp4 = p.fp4_codes != nullptr;
    const bool want_i8 = p.i8_codes != nullptr;
    const float g = want_fp4 ? *p.g : 1.0f;
    const int stride = gridDim.x * groups;
    float my_amax = 0.0f, my_amax_in = 0.0f;
    int parity = 0;

    // Every group of the CTA runs the same number of iterations (rows past m are computed on
    // zeros and not stored), so the shuffles and named barriers below are provably convergent
    // (no WARPSYNC/collective fallback code around the FHT's lane exchange).
    const int first = blockIdx.x * groups;
    const int iters = first < p.m ? (p.m - first + stride - 1) / stride : 0;
    int row = first + group;
    // SMEM: coalesced loads transposed through shared memory (long rows); otherwise each thread
    // reads its own 128-byte chunk directly (fewer registers; better for short rows).
    constexpr int VPT = SMEM ? 8 * NC : 1;
    const int nvec = p.k >> 3;
    extern __shared__ uint4 qsm[];                  // [groups][nch][9] (8 vectors + 1 pad per chunk)
    uint4* gbuf = qsm + (size_t)group * nch * 9;
    uint4 pv[VPT];
    uint4 dv[SMEM ? 1 : NC][SMEM ? 1 : 8];
    if constexpr (SMEM) load_row_coalesced<VPT>(pv, p.X + (size_t)row * p.ldx, tid, tpr, nvec, row < p.m);
    else load_chunks<NC>(dv, p.X + (size_t)row * p.ldx, tid, tpr, nch, row < p.m);
    for (int it = 0; it < iters; ++it) {
        const bool live = row < p.m;
        const int next = row + stride;
        uint4 v[NC][8];
        if constexpr (SMEM) {
            // transpose through smem: lane-contiguous vectors -> per-thread 64-element chunks
            GroupReduce::named_barrier(1 + group, tpr);     // previous row's chunk reads are done
#pragma unroll
            for (int j = 0; j < VPT; ++j) {
                const int vi = tid + j * tpr;
                if (vi < nvec) gbuf[(vi >> 3) * 9 + (vi & 7)] = pv[j];
            }
            GroupReduce::named_barrier(1 + group, tpr);
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const int c = tid + i * tpr;
#pragma unroll
                for (int j = 0; j < 8; ++j) v[i][j] = (c < nch) ? gbuf[c * 9 + j] : make_uint4(0, 0, 0, 0);
            }
            // prefetch the next row while this one is processed
            load_row_coalesced<VPT>(pv, p.X + (size_t)next * p.ldx, tid, tpr, nvec, next < p.m);
        } else {
#pragma unroll
            for (int i = 0; i < NC; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) v[i][j] = dv[i][j];
            load_chunks<NC>(dv, p.X + (size_t)next * p.ldx, tid, tpr, nch, next < p.m);
        }
        const int a0 = parity * 4;
        if (p.flags & DMPQ_QF_LAYERNORM) {
            // h = bf16((x - mean) * (1/sqrt(var + eps))), var = mean((x - mean)^2)  (glue, R13)
            f2 s2 = f2make(0.0f, 0.0f);
#pragma unroll
            for (int i = 0; i < NC; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    s2 = add2(s2, add2(bf16x2_to_f2(v[i][j].x), bf16x2_to_f2(v[i][j].y)));
                    s2 = add2(s2, add2(bf16x2_to_f2(v[i][j].z), bf16x2_to_f2(v[i][j].w)));
                }
            const float mean = __fdiv_rn(gr.sum(__fadd_rn(f2lo(s2), f2hi(s2)), a0 + 0), (float)p.k);
            const f2 nm = f2make(-mean, -mean);
            f2 q2 = f2make(0.0f, 0.0f);
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                if (tid + i * tpr >= nch) continue;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t w[4] = {v[i][j].x, v[i][j].y, v[i][j].z, v[i][j].w};
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const f2 d = add2(bf16x2_to_f2(w[t]), nm);
                        q2 = add2(q2, mul2(d, d));
                    }
                }
            }
            const float var = __fdiv_rn(gr.sum(__fadd_rn(f2lo(q2), f2hi(q2)), a0 + 1), (float)p.k);
            const float rstd = __frcp_rn(__fsqrt_rn(__fadd_rn(var, p.ln_eps)));
            const f2 rs = f2make(rstd, rstd);
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const int c = tid + i * tpr;
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    uint32_t w[4] = {v[i][j].x, v[i][j].y, v[i][j].z, v[i][j].w};
#pragma unroll
                    for (int t = 0; t < 4; ++t) w[t] = pack_bf16x2_f2(mul2(add2(bf16x2_to_f2(w[t]), nm), rs));
                    v[i][j] = (c < nch) ? make_uint4(w[0], w[1], w[2], w[3]) : make_uint4(0, 0, 0, 0);
                    if ((p.flags & DMPQ_QF_WRITE_H) && c < nch && live)
                        *reinterpret_cast<uint4*>(p.h_out + (size_t)row * p.ldh + (size_t)c * 64 + j * 8) = v[i][j];
                }
            }
        }
        if (p.row_abs_sum || p.amax_in) {   // PDR outlier statistics of the layer input (R15)
            float sa = 0.0f, mx = 0.0f;
#pragma unroll
            for (int i = 0; i < NC; ++i)
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t w[4] = {v[i][j].x, v[i][j].y, v[i][j].z, v[i][j].w};
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const float lo = fabsf(bf16lo(w[t])), hi = fabsf(bf16hi(w[t]));
                        sa = __fadd_rn(__fadd_rn(sa, lo), hi);
                        mx = fmaxf(mx, fmaxf(lo, hi));
                    }
                }
            my_amax_in = fmaxf(my_amax_in, mx);
            const float rs = gr.sum(sa, a0 + 3);
            if (tid == 0 && p.row_abs_sum && live) p.row_abs_sum[row] = rs;
        }
        // per-16-block |x| maxima (4 per chunk) and this thread's row maximum
        float bmax[NC][4];
        float tmax = 0.0f;
        f2 Y[HAD ? NC : 1][HAD ? 32 : 1];
#pragma unroll
        for (int i = 0; i < NC; ++i) {
            const bool ok = tid + i * tpr < nch;
            if constexpr (HAD) {
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const uint32_t w[4] = {v[i][j].x, v[i][j].y, v[i][j].z, v[i][j].w};
#pragma unroll
                    for (int t = 0; t < 4; ++t) Y[i][4 * j + t] = bf16x2_to_f2(w[t]);
                }
                fht128_chunk(Y[i], (tid & 1) != 0);
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    float mx = 0.0f;
#pragma unroll
                    for (int e = 0; e < 8; ++e) mx = fmaxf(mx, fmaxf(fabsf(f2lo(Y[i][8 * b + e])), fabsf(f2hi(Y[i][8 * b + e]))));
                    bmax[i][b] = ok ? mx : 0.0f;
                }
            } else {
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    const uint32_t w[8] = {v[i][2 * b].x, v[i][2 * b].y, v[i][2 * b].z, v[i][2 * b].w,
                                           v[i][2 * b + 1].x, v[i][2 * b + 1].y, v[i][2 * b + 1].z, v[i][2 * b + 1].w};
                    bmax[i][b] = absmax16(w);
                }
            }
            tmax = fmaxf(tmax, fmaxf(fmaxf(bmax[i][0], bmax[i][1]), fmaxf(bmax[i][2], bmax[i][3])));
        }
        my_amax = fmaxf(my_amax, tmax);

        if (want_fp4 && live) {
            uint8_t* sf_row = p.fp4_sf + (size_t)(row >> 7) * p.kc4 * 512 + (row & 31) * 16 + ((row & 127) >> 5) * 4;
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const int c = tid + i * tpr;
                if (c >= nch) continue;
                uint32_t sfw = 0;
                uint32_t codes[8];
#pragma unroll
                for (int b = 0; b < 4; ++b) {
                    float rcp;
                    sfw |= nvfp4_block_scale(bmax[i][b], g, rcp) << (8 * b);
                    const f2 r2 = f2make(rcp, rcp);
#pragma unroll
                    for (int t = 0; t < 2; ++t) {   // 8 elements -> one 32-bit word of codes
                        uint32_t cw = 0;
#pragma unroll
                        for (int u = 0; u < 4; ++u) {
                            const int e = 16 * b + 8 * t + 2 * u;
                            f2 q;
                            if constexpr (HAD) q = mul2(Y[i][e >> 1], r2);
                            else {
                                const uint4& vv = v[i][e >> 3];
                                const uint32_t ww = ((e & 7) == 0) ? vv.x : ((e & 7) == 2) ? vv.y : ((e & 7) == 4) ? vv.z : vv.w;
                                q = mul2(bf16x2_to_f2(ww), r2);
                            }
                            cw |= e2m1x2(f2lo(q), f2hi(q)) << (8 * u);
                        }
                        codes[2 * b + t] = cw;
                    }
                }
                uint4* cp = reinterpret_cast<uint4*>(p.fp4_codes + (size_t)row * (p.k >> 1) + (size_t)c * 32);
                cp[0] = make_uint4(codes[0], codes[1], codes[2], codes[3]);
                cp[1] = make_uint4(codes[4], codes[5], codes[6], codes[7]);
                *reinterpret_cast<uint32_t*>(sf_row + (size_t)c * 512) = sfw;
            }
        }
        if (want_i8) {
            const float a = gr.max(tmax, a0 + 2);
            const float rcp = a > 0.0f ? __fdiv_rn(127.0f, a) : 0.0f;
            if (tid == 0 && live) p.i8_scale[row] = a > 0.0f ? __fdiv_rn(a, 127.0f) : 1.0f;
            const f2 r2 = f2make(rcp, rcp);
#pragma unroll
            for (int i = 0; i < NC; ++i) {
                const int c = tid + i * tpr;
                if (c >= nch || !live) continue;
                uint4* op = reinterpret_cast<uint4*>(p.i8_codes + (size_t)row * p.k + (size_t)c * 64);
#pragma unroll
                for (int j = 0; j < 4; ++j) {   // 16 elements -> one 16-byte store
                    uint32_t o[4];
#pragma unroll
                    for (int t = 0; t < 4; ++t) {
                        const int e = 16 * j + 4 * t;
                        f2 q0, q1;
                        if constexpr (HAD) {
                            q0 = mul2(Y[i][e >> 1], r2);
                            q1 = mul2(Y[i][(e >> 1) + 1], r2);
                        } else {
                            const uint4& vv = v[i][e >> 3];
                            const uint32_t w0 = ((e & 7) == 0) ? vv.x : vv.z, w1 = ((e & 7) == 0) ? vv.y : vv.w;
                            q0 = mul2(bf16x2_to_f2(w0), r2);
                            q1 = mul2(bf16x2_to_f2(w1), r2);
                        }
                        o[t] = int8x4(q0, q1);
                    }
                    op[j] = make_uint4(o[0], o[1], o[2], o[3]);
                }
            }
        }
        row = next;
        parity ^= 1;
    }
    // zero the scale rows that pad m up to a multiple of 128 (read by the GEMM's M tail)
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
        const float am = warp_max(my_amax);
        if (lane == 0) atomic_max_nonneg(p.amax_out, am);
    }
    if (p.amax_in) {
        const float am = warp_max(my_amax_in);
        if (lane == 0) atomic_max_nonneg(p.amax_in, am);
    }
}


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
        if (p.row_abs_sum) {   // PDR outlier statistics of the layer input (R15)
            float sa = 0.0f;
#pragma unroll
            for (int i = 0; i < NV; ++i) {
                const uint32_t w[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                for (int t = 0; t < 4; ++t) sa = __fadd_rn(__fadd_rn(sa, fabsf(bf16lo(w[t]))), fabsf(bf16hi(w[t])));
            }
            const float rs = rr.sum(sa);
            if (tid == 0) p.row_abs_sum[row] = rs;
        }

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
    if (p.amax_out || p.amax_in) {
        float am = warp_max(cta_amax);
        if (lane == 0 && p.amax_out) atomic_max_nonneg(p.amax_out, am);
        if (lane == 0 && p.amax_in) atomic_max_nonneg(p.amax_in, am);   // unrotated: the same values
    }
}

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

__global__ void global_scale_kernel(const float* amax, float div, float* g_out, int count) {
    int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < count) {
        float g = __fdiv_rn(amax[i], div);
        g_out[i] = g < 1.17549435e-38f ? 1.17549435e-38f : g;
    }
}

template <int NC, bool SMEM>
static void launch_quant_had(const QuantParams& p, int tpr, cudaStream_t s) {
    const int groups = (256 % tpr == 0) ? 256 / tpr : 1;
    const int threads = groups * tpr;
    int ctas_needed = (p.m + groups - 1) / groups;
    int grid = num_sms() * (2048 / threads);
    if (grid > ctas_needed) grid = ctas_needed;
    if (grid < 1) grid = 1;
    const int smem = SMEM ? groups * (p.k / 64) * 9 * 16 : 0;
    quant_act_chunk_kernel<NC, true, SMEM><<<grid, threads, smem, s>>>(p, tpr);
}

template <int NV, bool WR>
static void launch_quant(const QuantParams& p, int threads, cudaStream_t s) {
    int rows_per_cta = WR ? threads / 32 : 1;
    int ctas_needed = (p.m + rows_per_cta - 1) / rows_per_cta;
    int grid = num_sms() * (WR ? 8 : (2048 / threads));
    if (grid > ctas_needed) grid = ctas_needed;
    if (grid < 1) grid = 1;
    quant_act_kernel<NV, WR><<<grid, threads, 0, s>>>(p);
}

}  // namespace dmpq

using namespace dmpq;

extern "C" dmpq_status dmpq_quantize_act(const uint16_t* X, int m, int k, int ldx, const dmpq_quant_opts* opts,
                                         dmpq_act* out_i8, dmpq_act* out_fp4, float* amax_out, dmpq_stream_t s) {
    DMPQ_REQUIRE(out_i8 || out_fp4 ||
                     (opts && ((opts->flags & DMPQ_QF_WRITE_H) || opts->row_abs_sum || opts->amax_in)),
                 DMPQ_EINVAL, "dmpq_quantize_act: nothing to produce (no output, h_out or statistics)");
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
    p.row_abs_sum = opts ? opts->row_abs_sum : nullptr;
    p.amax_in = opts ? opts->amax_in : nullptr;
    p.kc4 = ((k / 16) + 3) / 4;
    p.m_pad = (m + 127) / 128 * 128;
    if (m == 0) return DMPQ_OK;
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_quantize_act: needs an sm_100 device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    if (p.flags & DMPQ_QF_HADAMARD) {
        // chunk layout: 64 elements per thread, FHT stages 1..32 in-thread
        const int nch = k / 64;
        const int tpr = (nch + 31) / 32 * 32;
        if (k > 4096) launch_quant_had<1, true>(p, tpr, st);   // long rows: coalesced + smem transpose
        else launch_quant_had<1, false>(p, tpr, st);
        return check_launch("dmpq_quantize_act");
    }
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

extern "C" dmpq_status dmpq_outlier_reduce(const float* row_sums, int m, int segments, double* out, dmpq_stream_t s) {
    DMPQ_REQUIRE(row_sums && out && m >= 0 && segments >= 0, DMPQ_EINVAL, "dmpq_outlier_reduce: bad arguments");
    if (segments == 0) return DMPQ_OK;
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_outlier_reduce: needs an sm_100 device");
    outlier_reduce_kernel<<<segments, 256, 0, reinterpret_cast<cudaStream_t>(s)>>>(row_sums, m, out);
    return check_launch("dmpq_outlier_reduce");
}

extern "C" dmpq_status dmpq_global_scale(const float* amax, float div, float* g_out, int count, dmpq_stream_t s) {
    DMPQ_REQUIRE(amax && g_out && count >= 0 && div > 0.0f, DMPQ_EINVAL, "dmpq_global_scale: bad arguments");
    if (count == 0) return DMPQ_OK;
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_global_scale: needs an sm_100 device");
    global_scale_kernel<<<(count + 127) / 128, 128, 0, reinterpret_cast<cudaStream_t>(s)>>>(amax, div, g_out, count);
    return check_launch("dmpq_global_scale");
}
