// gemm.cu — dmpq_gemm: the DMPQ linear layer on 5th-generation tensor cores.
//   INT8  : tcgen05.mma.kind::i8, exact int32 accumulation in TMEM, FP32
//           per-token x per-channel dequant epilogue (R8).
//   NVFP4 : tcgen05.mma.kind::mxf4nvf4.block_scale.scale_vec::4X, E4M3 block scales
//           staged smem -> TMEM with tcgen05.cp, FP32 accumulation in TMEM,
//           per-tensor g_a*g_w dequant in the epilogue (R3).
// Both then apply the bias / GELU / gated-residual epilogue and store bf16 (+ fp32).
//
// Persistent, warp-specialised kernel, one CTA per SM (tile 128 x BN):
//   warp 0     TMA producer (A, B tiles, 128-byte swizzle; NVFP4 scale atoms by bulk copy)
//   warp 1     MMA issuer (one thread; tcgen05.mma + tcgen05.commit)
//   warp 2     TMEM allocator
//   warps 4..7 epilogue (TMEM -> registers -> global), warp w%4 owns TMEM lanes 32(w%4)..
// smem pipeline: STAGES x {A 128x128B, B BNx128B[, SFA 2 KB, SFB BN/128 x 2 KB]},
// full/empty mbarriers; TMEM: ACC_STAGES accumulators of BN columns (full/empty
// mbarriers), so the epilogue of tile i overlaps the mainloop of tile i+1.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "sm100.cuh"

namespace dmpq {

using namespace sm100;

struct GemmParams {
    int m, n, k;           // logical sizes (k in elements)
    int kbytes;            // bytes per row of A/B codes
    int num_m_tiles, num_n_tiles, num_kb;
    // INT8 epilogue
    const float* a_scale;  // [m]
    const float* w_scale;  // [n]
    // NVFP4
    const uint8_t* sfa;    // swizzled scale atoms
    const uint8_t* sfb;
    const float* g_a;
    const float* g_w;
    int kc4;               // scale atoms per 128-row tile (= k/64)
    int sfb_row_tiles;     // ceil(n/128)
    // epilogue
    uint32_t flags;
    const float* bias;
    const float* gate;
    const uint16_t* residual;
    int ldr;
    uint16_t* Y;
    int ldy;
    float* Y32;
    int32_t* acc_out;
};

constexpr int BM = 128;
constexpr int BK_BYTES = 128;  // one 128-byte swizzle row per K block (128 int8 / 256 fp4)

template <bool FP4, int BN, int STAGES>
struct SmemLayout {
    static constexpr int A_BYTES = BM * BK_BYTES;
    static constexpr int B_BYTES = BN * BK_BYTES;
    static constexpr int SFA_BYTES = FP4 ? 4 * 512 : 0;
    static constexpr int SFB_BYTES = FP4 ? (BN / 128) * 4 * 512 : 0;
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES + SFA_BYTES + SFB_BYTES;
    static constexpr int BAR_OFFSET = STAGES * STAGE_BYTES;
    static constexpr int TOTAL = BAR_OFFSET + 256 + 1024;  // barriers + holder + alignment slack
};

__device__ __forceinline__ float gelu_tanh(float x) {
    const float k0 = 0.7978845608028654f, k1 = 0.044715f;
    float x3 = __fmul_rn(__fmul_rn(x, x), x);
    float t = tanhf(__fmul_rn(k0, __fadd_rn(x, __fmul_rn(k1, x3))));
    return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.0f, t));
}

template <bool FP4, int BN, int STAGES, int ACC_STAGES>
__global__ void __launch_bounds__(256, 1) dmpq_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                                                           const __grid_constant__ CUtensorMap tmB, const GemmParams p) {
    using L = SmemLayout<FP4, BN, STAGES>;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar_full = sbase + L::BAR_OFFSET;          // STAGES x 8 B
    const uint32_t bar_empty = bar_full + STAGES * 8;
    const uint32_t bar_tfull = bar_empty + STAGES * 8;        // ACC_STAGES x 8 B
    const uint32_t bar_tempty = bar_tfull + ACC_STAGES * 8;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::BAR_OFFSET + 2 * STAGES * 8 + 2 * ACC_STAGES * 8);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    constexpr uint32_t ACC_COLS = ACC_STAGES * BN;
    constexpr uint32_t SF_COLS = FP4 ? (4 * 4 + 4 * (BN / 32)) : 0;
    constexpr uint32_t NEED_COLS = ACC_COLS + SF_COLS;
    constexpr uint32_t TMEM_COLS = NEED_COLS <= 32 ? 32 : NEED_COLS <= 64 ? 64 : NEED_COLS <= 128 ? 128 : NEED_COLS <= 256 ? 256 : 512;
    static_assert(NEED_COLS <= 512, "TMEM budget");

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int a = 0; a < ACC_STAGES; ++a) {
            mbar_init(bar_tfull + 8 * a, 1);
            mbar_init(bar_tempty + 8 * a, 4);  // one arrive per epilogue warp
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(smem_u32(tmem_holder), TMEM_COLS);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int num_tiles = p.num_m_tiles * p.num_n_tiles;

    if (warp == 0) {
        // ===================== TMA producer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
                const int mt = tile % p.num_m_tiles, nt = tile / p.num_m_tiles;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                    const uint32_t sA = sbase + stage * L::STAGE_BYTES;
                    const uint32_t sB = sA + L::A_BYTES;
                    uint32_t bytes = L::A_BYTES + L::B_BYTES;
                    int nsub = 4;
                    if constexpr (FP4) {
                        nsub = min(4, p.kc4 - kb * 4);  // valid 64-element sub-blocks in this K block
                        const int sfb_tiles = min(BN / 128, p.sfb_row_tiles - nt * (BN / 128));
                        bytes += nsub * 512 * (1 + sfb_tiles);
                    }
                    mbar_arrive_expect_tx(bar_full + 8 * stage, bytes);
                    tma_load_2d(sA, &tmA, kb * BK_BYTES, mt * BM, bar_full + 8 * stage);
                    tma_load_2d(sB, &tmB, kb * BK_BYTES, nt * BN, bar_full + 8 * stage);
                    if constexpr (FP4) {
                        const uint32_t sSFA = sB + L::B_BYTES;
                        const uint32_t sSFB = sSFA + L::SFA_BYTES;
                        bulk_load(sSFA, p.sfa + ((size_t)mt * p.kc4 + kb * 4) * 512, nsub * 512, bar_full + 8 * stage);
                        for (int h = 0; h < BN / 128; ++h) {
                            const int rt = nt * (BN / 128) + h;
                            if (rt < p.sfb_row_tiles)
                                bulk_load(sSFB + h * 2048, p.sfb + ((size_t)rt * p.kc4 + kb * 4) * 512, nsub * 512,
                                          bar_full + 8 * stage);
                        }
                    }
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer =====================
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            const uint32_t sfa_t = tmem_base + ACC_COLS;
            const uint32_t sfb_t = sfa_t + 16;
            for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
                const int nt = tile / p.num_m_tiles;
                const int acc = local % ACC_STAGES;
                const uint32_t acc_phase = (local / ACC_STAGES) & 1;
                const int n_here = min(BN, p.n - nt * BN);           // multiple of 16
                uint32_t idesc;
                if constexpr (FP4) {
                    // block-scaled descriptor: A/B E2M1 (1), scale UE4M3, K-major, N>>3 @17, M>>4 @24
                    idesc = (1u << 7) | (1u << 10) | ((uint32_t)(n_here >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
                } else {
                    // S32 accumulate (2 @4), A/B signed int8 (1), K-major
                    idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n_here >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
                }
                mbar_wait(bar_tempty + 8 * acc, acc_phase ^ 1);
                tc_fence_after();
                const uint32_t d_t = tmem_base + acc * BN;
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(bar_full + 8 * stage, phase);
                    tc_fence_after();
                    const uint32_t sA = sbase + stage * L::STAGE_BYTES;
                    const uint32_t sB = sA + L::A_BYTES;
                    int nsub = 4;
                    if constexpr (FP4) {
                        nsub = min(4, p.kc4 - kb * 4);
                        const uint32_t sSFA = sB + L::B_BYTES;
                        const uint32_t sSFB = sSFA + L::SFA_BYTES;
                        for (int j = 0; j < nsub; ++j) {
                            tc_cp_32x128b_warpx4(sfa_t + j * 4, sdesc_rows16(sSFA + j * 512));
                            for (int h = 0; h < BN / 128; ++h)
                                tc_cp_32x128b_warpx4(sfb_t + j * (BN / 32) + h * 4, sdesc_rows16(sSFB + h * 2048 + j * 512));
                        }
                    }
                    const uint64_t adesc = sdesc_k_sw128(sA), bdesc = sdesc_k_sw128(sB);
                    for (int j = 0; j < nsub; ++j) {
                        const uint32_t accum = (kb | j) ? 1u : 0u;
                        // advance 32 bytes along K inside the swizzle row (start address is in 16-B units)
                        if constexpr (FP4)
                            mma_fp4(d_t, adesc + 2 * j, bdesc + 2 * j, idesc, sfa_t + j * 4, sfb_t + j * (BN / 32), accum);
                        else
                            mma_i8(d_t, adesc + 2 * j, bdesc + 2 * j, idesc, accum);
                    }
                    tc_commit(bar_empty + 8 * stage);  // smem slot free once these MMAs retire
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                tc_commit(bar_tfull + 8 * acc);        // accumulator ready for the epilogue
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue =====================
        const int q = warp & 3;                          // TMEM lane quarter
        int local = 0;
        float gg = 0.0f;
        if constexpr (FP4) gg = __fmul_rn(*p.g_a, *p.g_w);
        for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x, ++local) {
            const int mt = tile % p.num_m_tiles, nt = tile / p.num_m_tiles;
            const int acc = local % ACC_STAGES;
            const uint32_t acc_phase = (local / ACC_STAGES) & 1;
            mbar_wait(bar_tfull + 8 * acc, acc_phase);
            tc_fence_after();
            const int row = mt * BM + q * 32 + lane;
            const bool row_ok = row < p.m;
            float sa = 0.0f;
            if constexpr (!FP4) sa = row_ok ? p.a_scale[row] : 0.0f;
            const int n_here = min(BN, p.n - nt * BN);
            for (int c = 0; c < BN / 32; ++c) {
                if (c * 32 >= n_here) break;             // uniform across the CTA
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, r);
                tmem_ld_wait();
                if (c * 32 + 32 >= n_here) {
                    // last chunk of this accumulator: hand TMEM back to the MMA warp
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(bar_tempty + 8 * acc);
                }
                if (!row_ok) continue;
                const int col0 = nt * BN + c * 32;
                float y[32];
#pragma unroll
                for (int j = 0; j < 32; ++j) {
                    float v;
                    if constexpr (FP4) {
                        v = __fmul_rn(__uint_as_float(r[j]), gg);
                    } else {
                        v = __fmul_rn(__fmul_rn(__int2float_rn((int)r[j]), sa), __ldg(p.w_scale + col0 + j));
                    }
                    if (p.flags & DMPQ_EP_BIAS) v = __fadd_rn(v, __ldg(p.bias + col0 + j));
                    if (p.flags & DMPQ_EP_GELU_TANH) v = gelu_tanh(v);
                    y[j] = v;
                }
                if (p.flags & DMPQ_EP_RESIDUAL) {
                    const uint4* rp = reinterpret_cast<const uint4*>(p.residual + (size_t)row * p.ldr + col0);
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4) {
                        const uint4 rv = rp[v4];
                        const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const int e = v4 * 8 + j * 2;
                            y[e] = __fadd_rn(bf16lo(w[j]), __fmul_rn(__ldg(p.gate + col0 + e), y[e]));
                            y[e + 1] = __fadd_rn(bf16hi(w[j]), __fmul_rn(__ldg(p.gate + col0 + e + 1), y[e + 1]));
                        }
                    }
                }
                if (p.Y) {
                    uint4* yp = reinterpret_cast<uint4*>(p.Y + (size_t)row * p.ldy + col0);
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4)
                        yp[v4] = make_uint4(pack_bf16x2(y[v4 * 8 + 0], y[v4 * 8 + 1]), pack_bf16x2(y[v4 * 8 + 2], y[v4 * 8 + 3]),
                                            pack_bf16x2(y[v4 * 8 + 4], y[v4 * 8 + 5]), pack_bf16x2(y[v4 * 8 + 6], y[v4 * 8 + 7]));
                }
                if (p.Y32) {
                    float4* yp = reinterpret_cast<float4*>(p.Y32 + (size_t)row * p.n + col0);
#pragma unroll
                    for (int v4 = 0; v4 < 8; ++v4) yp[v4] = make_float4(y[4 * v4], y[4 * v4 + 1], y[4 * v4 + 2], y[4 * v4 + 3]);
                }
                if constexpr (!FP4) {
                    if (p.acc_out) {
                        int4* ap = reinterpret_cast<int4*>(p.acc_out + (size_t)row * p.n + col0);
#pragma unroll
                        for (int v4 = 0; v4 < 8; ++v4)
                            ap[v4] = make_int4((int)r[4 * v4], (int)r[4 * v4 + 1], (int)r[4 * v4 + 2], (int)r[4 * v4 + 3]);
                    }
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 2) tmem_dealloc(tmem_base, TMEM_COLS);
}

// ------------------------------------------------------------------ host side

static PFN_cuTensorMapEncodeTiled_v12000 get_encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        void* ptr = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &ptr, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(ptr);
    });
    return fn;
}

// 2-D uint8 tensor map over a [rows x row_bytes] row-major matrix, box 128 B x box_rows, 128-B swizzle.
static bool make_tmap(CUtensorMap* tm, const void* base, int rows, int row_bytes, int box_rows) {
    auto enc = get_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)row_bytes, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)row_bytes};
    cuuint32_t box[2] = {(cuuint32_t)BK_BYTES, (cuuint32_t)box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <bool FP4, int BN, int STAGES, int ACC_STAGES>
static dmpq_status launch_gemm(const GemmParams& p, const void* a_codes, const void* w_codes, cudaStream_t s) {
    using L = SmemLayout<FP4, BN, STAGES>;
    CUtensorMap tmA, tmB;
    if (!make_tmap(&tmA, a_codes, p.m, p.kbytes, BM) || !make_tmap(&tmB, w_codes, p.n, p.kbytes, BN))
        return set_error(DMPQ_ECUDA, "dmpq_gemm: cuTensorMapEncodeTiled failed");
    auto kern = dmpq_gemm_kernel<FP4, BN, STAGES, ACC_STAGES>;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL) != cudaSuccess)
            return check_launch("dmpq_gemm(smem attribute)");
        attr_set = true;
    }
    int tiles = p.num_m_tiles * p.num_n_tiles;
    int grid = tiles < num_sms() ? tiles : num_sms();
    kern<<<grid, 256, L::TOTAL, s>>>(tmA, tmB, p);
    return check_launch("dmpq_gemm");
}

}  // namespace dmpq

using namespace dmpq;

extern "C" dmpq_status dmpq_gemm(const dmpq_act* A, const dmpq_weights* W, const dmpq_epilogue* ep, uint16_t* Y, int ldy,
                                 float* Y32, int32_t* acc_or_null, dmpq_stream_t s) {
    DMPQ_REQUIRE(A && W, DMPQ_EINVAL, "dmpq_gemm: NULL operand");
    DMPQ_REQUIRE(A->fmt == DMPQ_FMT_INT8 || A->fmt == DMPQ_FMT_NVFP4, DMPQ_EINVAL, "dmpq_gemm: unknown format");
    const bool fp4 = A->fmt == DMPQ_FMT_NVFP4;
    const int m = A->m, n = W->n, k = A->k;
    DMPQ_REQUIRE(k == W->k && k > 0 && k % 64 == 0 && n > 0 && n % 32 == 0 && m >= 0, DMPQ_ESHAPE,
                 "dmpq_gemm: need A.k == W.k, k %% 64 == 0, n %% 32 == 0 (m=%d n=%d k=%d Wk=%d)", m, n, k, W->k);
    DMPQ_REQUIRE(Y || Y32 || acc_or_null, DMPQ_EINVAL, "dmpq_gemm: no output");
    DMPQ_REQUIRE(!Y || (aligned16(Y) && ldy >= n && ldy % 8 == 0), DMPQ_EALIGN, "dmpq_gemm: Y / ldy alignment");
    DMPQ_REQUIRE(!Y32 || aligned16(Y32), DMPQ_EALIGN, "dmpq_gemm: Y32 alignment");
    DMPQ_REQUIRE(!acc_or_null || !fp4, DMPQ_EINVAL, "dmpq_gemm: raw accumulators are INT8-only");
    DMPQ_REQUIRE(!acc_or_null || aligned16(acc_or_null), DMPQ_EALIGN, "dmpq_gemm: acc alignment");
    GemmParams p{};
    p.m = m; p.n = n; p.k = k;
    p.flags = ep ? ep->flags : 0u;
    if (p.flags & DMPQ_EP_BIAS) {
        DMPQ_REQUIRE(W->bias != nullptr, DMPQ_EINVAL, "dmpq_gemm: DMPQ_EP_BIAS without W->bias");
        p.bias = W->bias;
    }
    if (p.flags & DMPQ_EP_RESIDUAL) {
        DMPQ_REQUIRE(ep->gate && ep->residual && aligned16(ep->residual) && ep->ldr >= n && ep->ldr % 8 == 0, DMPQ_EALIGN,
                     "dmpq_gemm: residual/gate");
        p.gate = ep->gate; p.residual = ep->residual; p.ldr = ep->ldr;
    }
    p.Y = Y; p.ldy = ldy; p.Y32 = Y32; p.acc_out = acc_or_null;
    if (m == 0) return DMPQ_OK;
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_gemm: needs an sm_100 device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    if (fp4) {
        DMPQ_REQUIRE(A->codes && A->sf && A->g && W->fp4_codes && W->fp4_sf && W->fp4_g && aligned16(A->codes) &&
                         aligned16(A->sf) && aligned16(W->fp4_codes) && aligned16(W->fp4_sf),
                     DMPQ_EALIGN, "dmpq_gemm: NVFP4 operand pointers");
        p.kbytes = k / 2;
        p.sfa = A->sf; p.sfb = W->fp4_sf; p.g_a = A->g; p.g_w = W->fp4_g;
        p.kc4 = k / 64;
        p.sfb_row_tiles = (n + 127) / 128;
        p.num_m_tiles = (m + BM - 1) / BM;
        p.num_kb = (p.kbytes + BK_BYTES - 1) / BK_BYTES;
        const char* v = getenv("DMPQ_FP4_VARIANT");
        if (v && v[0] == '1') {
            p.num_n_tiles = (n + 127) / 128;
            return launch_gemm<true, 128, 6, 2>(p, A->codes, W->fp4_codes, st);
        }
        constexpr int BN = 256;
        p.num_n_tiles = (n + BN - 1) / BN;
        return launch_gemm<true, BN, 4, 1>(p, A->codes, W->fp4_codes, st);
    } else {
        DMPQ_REQUIRE(A->codes && A->row_scale && W->i8_codes && W->i8_scale && aligned16(A->codes) && aligned16(W->i8_codes),
                     DMPQ_EALIGN, "dmpq_gemm: INT8 operand pointers");
        p.kbytes = k;
        p.a_scale = A->row_scale; p.w_scale = W->i8_scale;
        p.num_m_tiles = (m + BM - 1) / BM;
        p.num_kb = (p.kbytes + BK_BYTES - 1) / BK_BYTES;
        constexpr int BN = 256;
        p.num_n_tiles = (n + BN - 1) / BN;
        return launch_gemm<false, BN, 4, 2>(p, A->codes, W->i8_codes, st);
    }
}
