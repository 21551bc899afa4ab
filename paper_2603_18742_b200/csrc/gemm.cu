// gemm.cu — dmpq_gemm: the DMPQ linear layer on 5th-generation tensor cores.
//   INT8  : tcgen05.mma.kind::i8, exact int32 accumulation in TMEM, FP32
//           per-token x per-channel dequant epilogue, bit-exact (R8).
//   BF16  : tcgen05.mma.kind::f16 (BF16 x BF16 -> FP32), the full-precision fallback of
//           the Purified Cache Refresh outlier gate (R15).
//   NVFP4 : tcgen05.mma.kind::mxf4nvf4.block_scale.scale_vec::4X, E4M3 block scales
//           staged smem -> TMEM with tcgen05.cp, FP32 accumulation in TMEM,
//           per-tensor g_a*g_w dequant fused with the bias as one FMA (R3).
// Both then apply the bias / GELU / gated-residual epilogue and store bf16 (+ fp32).
//
// Persistent, warp-specialised, CTA-pair kernel (one CTA per SM, cluster of 2):
//   warp 0     TMA producer (A, B-half, NVFP4 scale atoms; 128-byte swizzle)
//   warp 1     MMA issuer (leader CTA, one thread; tcgen05.mma.cta_group::2 + commit)
//   warp 2     TMEM allocator (cta_group::2)
//   warps 4..7 epilogue (TMEM -> registers -> smem -> TMA store), warp w%4 owns TMEM lanes 32(w%4)..
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstdlib>
#include <cstring>
#include <mutex>

#include "common.cuh"
#include "tmap.cuh"
#include "quant.cuh"
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
    const float* g_w_col;  // [n] per-column g_w (layers packed side by side) or NULL
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
    // fused TDC refresh (DMPQ_EP_TDC_REFRESH)
    const uint16_t* tdc_x_in;
    uint16_t* tdc_delta;
    double* tdc_stats;
    double* tdc_partials;      // [gridDim.x * EPI_WARPS][7]
    unsigned int* tdc_counter;
    // device-predicated launch (R18): run only when *run_if == run_if_value
    const int* run_if;
    int run_if_value;
    // producer-fused NVFP4 quantization of bf16(Y) (DMPQ_EP_QUANT_NVFP4)
    uint8_t* q_codes;
    uint8_t* q_sf;
    const float* q_g;
    float* q_amax;
    int q_kc4, q_m_pad;
};

constexpr int BM = 128;
constexpr int BK_BYTES = 128;  // one 128-byte swizzle row per K block (128 int8 / 256 fp4)


// ============================================================================
// 2-CTA kernel (the production path): a CTA pair (cluster of 2) computes a
// 256 x BN tile with tcgen05.mma.cta_group::2 (M = 256). Each CTA loads its own
// 128 A rows and half of the BN B rows (the MMA reads B from both CTAs' smem), so
// per-SM L2->smem traffic per FLOP drops by 1.5x vs a 1-CTA 128 x BN tile. NVFP4
// scale atoms arrive by 3-D TMA (OOB -> zero), SFA per CTA, SFB in both (each CTA loads one
// row tile and multicasts it to the pair).
// TMEM: two BN-column accumulators per CTA (epilogue of tile i overlaps the
// mainloop of tile i+1). Epilogue: TMEM -> registers -> swizzled smem staging (128-B rows shared by
// the two warps of a lane quarter, DMPQ_EPI_PAIR)
// -> TMA store; per-column vectors (bias, w_scale, gate) staged in smem per tile.
// ============================================================================
#ifndef DMPQ_EPI_WARPS
#define DMPQ_EPI_WARPS 8
#endif
constexpr int EPI_WARPS = DMPQ_EPI_WARPS;   // epilogue warps per CTA (2 per TMEM lane quarter, column-interleaved)
#ifndef DMPQ_GEMM_PREFETCH
#define DMPQ_GEMM_PREFETCH 0   // 1: L2 prefetch of the next tile's A / B rows at each tile start (measured 25-30 % slower);
                               // 2: the next tile's A, one K block per K block (~8 % slower). A partitioned prefetch (each
                               // pair its 1/num_n_tiles share of the next A panel, fetched once from DRAM) was no faster
                               // at K = 3072 and 1-5 % slower at K = 12288 (round 2): DRAM latency is not the tile-start limiter
#endif
#ifndef DMPQ_MAX_STAGING
#define DMPQ_MAX_STAGING 3     // output/residual staging buffers per epilogue warp (at most)
#endif
#ifndef DMPQ_EPI_PAIR
#define DMPQ_EPI_PAIR 1        // 1: the two epilogue warps of a TMEM lane quarter share 32 x 64-column staging buffers (128-B rows, one TMA store / residual load per chunk pair)
#endif
#ifndef DMPQ_SFB_MC
#define DMPQ_SFB_MC 1          // NVFP4: the two CTAs of a pair each load one SFB row tile and multicast it to both (SFB L2 reads halved)
#endif
#ifndef DMPQ_GEMM_RASTER
#define DMPQ_GEMM_RASTER 0     // 0: pair c takes tiles c, c + P, ... (n-fastest); 1: a contiguous run of tiles per pair
#endif
// the tiles of CTA pair `cid` of `ncl`: for (t = t0; t < t1; t += step)
__device__ __forceinline__ void tile_span(int cid, int ncl, int num_tiles, int& t0, int& t1, int& step) {
    if (DMPQ_GEMM_RASTER) {
        t0 = (int)(((long long)cid * num_tiles) / ncl);
        t1 = (int)(((long long)(cid + 1) * num_tiles) / ncl);
        step = 1;
    } else {
        t0 = cid; t1 = num_tiles; step = ncl;
    }
}

template <int KIND, int BN, int STAGES>   // KIND: 0 INT8, 1 NVFP4, 2 BF16
struct PairLayout {
    static constexpr bool FP4 = KIND == 1;
    static constexpr int A_BYTES = BM * BK_BYTES;                 // 16 KB
    static constexpr int B_BYTES = (BN / 2) * BK_BYTES;           // this CTA's half of B
    static constexpr int SFA_BYTES = FP4 ? 4 * 512 : 0;
    static constexpr int SFB_BYTES = FP4 ? 2 * 4 * 512 : 0;       // 2 row-tiles of atoms (256 B rows)
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES + SFA_BYTES + SFB_BYTES;
    static constexpr int PAIR_TX = 2 * STAGE_BYTES;               // bytes both CTAs land per stage
    static constexpr int STAGING_OFFSET = STAGES * STAGE_BYTES;   // per epilogue warp: STAGING_BUFS x (32 rows x 64 B)
    static constexpr int VEC_BYTES = 2 * 3 * BN * 4;              // [acc parity][bias|wscale|gate][BN]
    static constexpr int SMEM_LIMIT = 232448;                     // 227 KB opt-in per CTA
    // double-buffered output staging when it fits next to the stage ring, else single-buffered
    // output / residual staging buffers per epilogue warp: 3 when they fit next to the stage ring
    // (NVFP4 BN = 192: a warp's three chunks of a tile all get their residual requested before the
    // accumulator is ready), else 2, else 1
    static constexpr int STAGING_BUFS =
        (DMPQ_MAX_STAGING >= 3 && STAGING_OFFSET + EPI_WARPS * 3 * 2048 + VEC_BYTES + 512 + 1024 <= SMEM_LIMIT) ? 3
        : (STAGING_OFFSET + EPI_WARPS * 2 * 2048 + VEC_BYTES + 512 + 1024 <= SMEM_LIMIT) ? 2 : 1;
    static constexpr int STAGING_BYTES = EPI_WARPS * STAGING_BUFS * 2048;
    // DMPQ_EPI_PAIR: the two warps of a lane quarter share 128-B-row staging buffers (needs >= 2 of them)
    static constexpr bool PAIRED = DMPQ_EPI_PAIR != 0 && EPI_WARPS == 8 && STAGING_BUFS >= 2;
    static constexpr int VEC_OFFSET = STAGING_OFFSET + STAGING_BYTES;
    static constexpr int BAR_OFFSET = VEC_OFFSET + VEC_BYTES;
    static constexpr int TOTAL = BAR_OFFSET + 512 + 1024;   // mbarriers, TMEM holder, residual barriers
    static_assert(STAGE_BYTES % 1024 == 0, "stage buffers must stay 1024-B aligned");
    static_assert(TOTAL <= SMEM_LIMIT, "shared memory budget");
};

// CL = 2: one CTA pair per cluster. CL = 4 (experiment, DMPQ_GEMM_CLUSTER=4): two pairs per cluster
// work on vertically adjacent 256-row tiles of the same N tile; each CTA loads a quarter of the
// pair's B tile and TMA-multicasts it to the same-rank CTA of the other pair, and two CTAs load the
// NVFP4 SFB atoms for all four (B and SFB L2 reads halved / quartered); a stage is refilled only
// once both pairs' MMAs have released it.
template <int KIND, int BN, int STAGES, bool TDC = false, bool QNT = false, int CL = 2>   // TDC: fused refresh; QNT: fused NVFP4 quantizer
__global__ void __cluster_dims__(CL, 1, 1) __launch_bounds__(128 + 32 * EPI_WARPS, 1)
    dmpq_gemm_pair_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                          const __grid_constant__ CUtensorMap tmSFA, const __grid_constant__ CUtensorMap tmSFB,
                          const __grid_constant__ CUtensorMap tmY, const __grid_constant__ CUtensorMap tmR,
                          const GemmParams p) {
    using L = PairLayout<KIND, BN, STAGES>;
    constexpr bool FP4 = KIND == 1;
    constexpr bool I8 = KIND == 0;
    // device-predicated launch: every CTA of the grid reads the same flag, so whole clusters exit
    // together before any barrier, TMEM allocation or TMA is touched
    if (p.run_if && *p.run_if != p.run_if_value) return;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar_full = sbase + L::BAR_OFFSET;
    const uint32_t bar_empty = bar_full + STAGES * 8;
    const uint32_t bar_tfull = bar_empty + STAGES * 8;
    const uint32_t bar_tempty = bar_tfull + 2 * 8;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::BAR_OFFSET + 2 * STAGES * 8 + 4 * 8);
    const uint32_t bar_res = bar_full + 2 * STAGES * 8 + 4 * 8 + 16;   // [EPI_WARPS][3] residual-chunk TMA loads

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    static_assert(CL == 2 || CL == 4, "cluster of one or two CTA pairs");
    const uint32_t crank = cluster_ctarank();
    const uint32_t rank = crank & 1;            // rank inside the CTA pair
    const int pp = (int)(crank >> 1);           // pair index inside the cluster (CL = 4)
    constexpr uint16_t EMPTY_MASK = CL == 4 ? 0xF : 0x3;
    const uint16_t pair_mask = (uint16_t)(0x3u << (2 * pp));
    // accumulator buffers in TMEM: two (the epilogue of tile i overlaps the mainloop of tile
    // i + 1) unless BN = 256 NVFP4, where 2 x 256 columns leave no room for the scale factors:
    // one buffer, and the mainloop of tile i + 1 waits for the epilogue of tile i
    constexpr int NACC = (FP4 && BN == 256) ? 1 : 2;
    constexpr uint32_t ACC_COLS = NACC * BN;
    constexpr uint32_t SF_COLS = FP4 ? (4 * 4 + 4 * 8) : 0;
    static_assert(ACC_COLS + SF_COLS <= 512, "TMEM budget");
    constexpr uint32_t TMEM_COLS = 512;

    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        if constexpr (FP4) { prefetch_tmap(&tmSFA); prefetch_tmap(&tmSFB); }
        if (p.Y) prefetch_tmap(&tmY);
        if (p.Y && (p.flags & DMPQ_EP_RESIDUAL)) prefetch_tmap(&tmR);
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, CL / 2);   // every pair that reads the stage releases it
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(bar_tfull + 8 * a, 1);
            mbar_init(bar_tempty + 8 * a, 2 * EPI_WARPS);  // every epilogue warp of both CTAs
        }
        for (int i = 0; i < 3 * EPI_WARPS; ++i) mbar_init(bar_res + 8 * i, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_pair(smem_u32(tmem_holder), TMEM_COLS);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    // cluster tiles: CL = 2 one 256-row pair tile, CL = 4 a 512-row group (pair pp takes its half)
    const int num_mg = CL == 4 ? (p.num_m_tiles + 1) >> 1 : p.num_m_tiles;
    const int num_tiles = num_mg * p.num_n_tiles;
    auto tile_mt = [&](int tile) { return CL == 4 ? (tile / p.num_n_tiles) * 2 + pp : tile / p.num_n_tiles; };
    const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
    int ts0, ts1, tstep;
    tile_span(cid, ncl, num_tiles, ts0, ts1, tstep);

    if (warp == 0) {
        // ===================== TMA producer (both CTAs; whole warp, one elected issuer) =====================
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = ts0; tile < ts1; tile += tstep) {
            const int mt = tile_mt(tile), nt = tile % p.num_n_tiles;   // n-fastest: A tile reused across N while L2-resident
            const int m0 = mt * 256 + (int)rank * BM;
            const int nb0 = nt * BN + (int)rank * (BN / 2);
            // next tile's A rows, one K block per K block of this tile (mode 2)
            const bool pf2 = DMPQ_GEMM_PREFETCH == 2 && tile + tstep < ts1;
            const int pf_m = pf2 ? ((tile + tstep) / p.num_n_tiles) * 256 + (int)rank * BM : 0;
            if (DMPQ_GEMM_PREFETCH == 1 && tile + tstep < ts1) {
                // the next tile's A and B rows -> L2 a whole tile ahead: at short K the stage ring
                // (~1 us deep) cannot hide a DRAM miss at every tile start (ncu: the MMA warp waited
                // on the full barrier ~35 % of its time at K = 3072)
                const int mt2 = (tile + tstep) / p.num_n_tiles, nt2 = (tile + tstep) % p.num_n_tiles;
                const int m2 = mt2 * 256 + (int)rank * BM, n2 = nt2 * BN + (int)rank * (BN / 2);
                if (elect_one()) {
                    for (int kb = 0; kb < p.num_kb; ++kb) {
                        tma_prefetch_2d(&tmA, kb * BK_BYTES, m2);
                        tma_prefetch_2d(&tmB, kb * BK_BYTES, n2);
                    }
                }
                __syncwarp();
            }
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                if (elect_one()) {
                    const uint32_t full_l = leader_addr(bar_full + 8 * stage);
                    if (rank == 0) mbar_arrive_expect_tx(bar_full + 8 * stage, L::PAIR_TX);
                    const uint32_t sA = sbase + stage * L::STAGE_BYTES;
                    const uint32_t sB = sA + L::A_BYTES;
                    tma_load_2d_pair(sA, &tmA, kb * BK_BYTES, m0, full_l);
                    if constexpr (CL == 4) {   // quarter pp of this CTA's B half -> both pairs' same-rank CTAs
                        tma_load_2d_pair_mc(sB + pp * (BN / 4) * BK_BYTES, &tmB, kb * BK_BYTES, nb0 + pp * (BN / 4), full_l,
                                            (uint16_t)((1u << rank) | (1u << (rank + 2))));
                    } else {
                        tma_load_2d_pair(sB, &tmB, kb * BK_BYTES, nb0, full_l);
                    }
                    if (pf2 && pf_m != m0) tma_prefetch_2d(&tmA, kb * BK_BYTES, pf_m);
                    if constexpr (FP4) {
                        const uint32_t sSFA = sB + L::B_BYTES;
                        const uint32_t sSFB = sSFA + L::SFA_BYTES;
                        tma_load_3d_pair(sSFA, &tmSFA, 0, kb * 4, mt * 2 + (int)rank, full_l);
                        if constexpr (CL == 4) {   // CTAs 0 / 1 load SFB row tile 0 / 1 for all four
                            if (crank < 2)
                                tma_load_3d_pair_mc(sSFB + crank * 2048, &tmSFB, 0, kb * 4, ((nt * BN) >> 7) + (int)crank, full_l, 0xF);
                        } else if constexpr (DMPQ_SFB_MC != 0) {   // CTA r loads SFB row tile r for both CTAs of the pair
                            tma_load_3d_pair_mc(sSFB + rank * 2048, &tmSFB, 0, kb * 4, ((nt * BN) >> 7) + (int)rank, full_l, 0x3);
                        } else {
                            tma_load_3d_pair(sSFB, &tmSFB, 0, kb * 4, (nt * BN) >> 7, full_l);
                        }
                    }
                }
                __syncwarp();
                if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA; whole warp, one elected issuer) =====================
        if (rank == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            const uint32_t sfa_t = tmem_base + ACC_COLS;
            const uint32_t sfb_t = sfa_t + 16;
            uint32_t idesc;
            if constexpr (FP4) idesc = (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
            else if constexpr (I8) idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
            else idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);  // F32 acc, BF16 x BF16
            for (int tile = ts0; tile < ts1; tile += tstep, ++local) {
                const int nt = tile % p.num_n_tiles;
                const int acc = local & 1;
                const uint32_t acc_phase = (local >> 1) & 1;
                // SFB rows start at the 128-row atom below n0; BN=192 odd tiles start 64 rows (2 columns) in
                const uint32_t sfb_shift = (uint32_t)(((nt * BN) & 127) >> 5);
                mbar_wait(bar_tempty + 8 * acc, acc_phase ^ 1);
                if constexpr (NACC == 1) {   // single buffer: the previous tile's epilogue must be done too
                    if (local >= 1) mbar_wait(bar_tempty + 8 * ((local - 1) & 1), ((local - 1) >> 1) & 1);
                }
                tc_fence_after();
                const uint32_t d_t = tmem_base + (NACC == 2 ? acc * BN : 0);
                for (int kb = 0; kb < p.num_kb; ++kb) {
                    mbar_wait(bar_full + 8 * stage, phase);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t sA = sbase + stage * L::STAGE_BYTES;
                        const uint32_t sB = sA + L::A_BYTES;
                        if constexpr (FP4) {
                            const uint32_t sSFA = sB + L::B_BYTES;
                            const uint32_t sSFB = sSFA + L::SFA_BYTES;
                            const uint64_t da = sdesc_rows16(sSFA), db = sdesc_rows16(sSFB);
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                tc_cp_pair_32x128b_warpx4(sfa_t + j * 4, da + (uint64_t)(j * 32));
                                tc_cp_pair_32x128b_warpx4(sfb_t + j * 8, db + (uint64_t)(j * 32));
                                tc_cp_pair_32x128b_warpx4(sfb_t + j * 8 + 4, db + (uint64_t)(128 + j * 32));
                            }
                        }
                        const uint64_t adesc = sdesc_k_sw128(sA), bdesc = sdesc_k_sw128(sB);
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t accum = (kb | j) ? 1u : 0u;
                            if constexpr (FP4)
                                mma_fp4_pair(d_t, adesc + 2 * j, bdesc + 2 * j, idesc, sfa_t + j * 4, sfb_t + j * 8 + sfb_shift, accum);
                            else if constexpr (I8)
                                mma_i8_pair(d_t, adesc + 2 * j, bdesc + 2 * j, idesc, accum);
                            else
                                mma_f16_pair(d_t, adesc + 2 * j, bdesc + 2 * j, idesc, accum);
                        }
                        tc_commit_pair_mc(bar_empty + 8 * stage, EMPTY_MASK);
                    }
                    __syncwarp();
                    if (++stage == STAGES) { stage = 0; phase ^= 1; }
                }
                if (elect_one()) tc_commit_pair_mc(bar_tfull + 8 * acc, pair_mask);
                __syncwarp();
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue (both CTAs, 4 warps each) =====================
        // Instruction-lean: the epilogue issues ~1.5 (NVFP4) / ~3.5 (INT8) instructions per
        // output element and is the critical path for short-K layers, so
        // the math is packed fp32x2 (FFMA2/FMUL2/FADD2) and per-column vectors come from smem
        // as 128-bit broadcast loads.
        const int q = warp & 3;                 // TMEM lane quarter this warp may access
        const int ew = warp - 4;                 // epilogue warp index
        const int chalf = ew >> 2;               // column phase: chunks chalf, chalf + CSTEP, ...
        constexpr int CSTEP = EPI_WARPS / 4;
        const int etid = threadIdx.x - 128;
        int local = 0;
        uint32_t chunk_ctr = 0;
        float gg = 0.0f, ga = 0.0f;
        const bool gcol = FP4 && p.g_w_col != nullptr;
        if constexpr (FP4) {
            ga = *p.g_a;
            if (!gcol) gg = __fmul_rn(ga, *p.g_w);
        }
        else if constexpr (!I8) gg = 1.0f;   // BF16: y = fma(acc, 1, bias) = fl(acc + bias)
        const f2 gg2 = f2make(gg, gg);
        // staging: per warp NSB x (32 rows x 64 B, 64-B swizzle), or (DMPQ_EPI_PAIR) per lane quarter
        // NSB x (32 rows x 128 B, 128-B swizzle), warp chalf owning bytes [64 chalf, 64 chalf + 64) of a row
        constexpr bool PAIRST = L::PAIRED;
        constexpr uint32_t SBUF = PAIRST ? 4096 : 2048;
        const uint32_t staging = PAIRST ? sbase + L::STAGING_OFFSET + q * (L::STAGING_BUFS * 4096)
                                        : sbase + L::STAGING_OFFSET + ew * (L::STAGING_BUFS * 2048);
        const int sb_id = PAIRST ? q : ew;        // residual barrier group
        const bool issuer = !PAIRST || chalf == 0; // the warp that issues the pair's TMA loads / stores
        const uint32_t vec_s = sbase + L::VEC_OFFSET;
        const bool has_bias = (p.flags & DMPQ_EP_BIAS) != 0;
        const bool has_gelu = (p.flags & DMPQ_EP_GELU_TANH) != 0;
        const bool has_res = (p.flags & DMPQ_EP_RESIDUAL) != 0;
        // gated residual with a bf16 output: the residual chunk arrives by TMA into the chunk's
        // output staging buffer (coalesced; the lane-per-row global loads cost 30-50 us per GEMM)
        const bool tma_res = has_res && p.Y != nullptr;
        // the fused-refresh code only exists in the TDC instantiation (it costs the plain epilogue
        // ~10 registers and spills in the INT8 kernel)
        const bool has_tdc = TDC && (p.flags & DMPQ_EP_TDC_REFRESH) != 0;
        // fused TDC refresh statistics of this warp's rows / chunks over all its tiles (fixed order)
        double tacc[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
        const float qg = QNT ? *p.q_g : 1.0f;   // the consumer's NVFP4 global scale (R3)
        float qamax = 0.0f;
        for (int tile = ts0; tile < ts1; tile += tstep, ++local) {
            const int mt = tile_mt(tile), nt = tile % p.num_n_tiles;   // n-fastest: A tile reused across N while L2-resident
            const int acc = local & 1;
            const uint32_t acc_phase = (local >> 1) & 1;
            const int n0 = nt * BN;
            // per-column epilogue vectors of this tile -> smem (double-buffered by tile parity)
            const uint32_t vb = vec_s + acc * 3 * BN * 4;
            for (int i = etid; i < BN; i += 32 * EPI_WARPS) {
                const int col = n0 + i;
                const bool ok = col < p.n;
                const float bv = (ok && has_bias) ? p.bias[col] : -0.0f;   // fma(x, s, -0) == fl(x * s) exactly
                // INT8: s_w[n]; NVFP4 with per-column g_w: fl(g_a g_w[n]) (same product as gg)
                const float wv = (I8 && ok) ? p.w_scale[col] : ((FP4 && ok && gcol) ? __fmul_rn(ga, p.g_w_col[col]) : 0.0f);
                const float gv = (ok && has_res) ? p.gate[col] : 0.0f;
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(vb + i * 4), "f"(bv) : "memory");
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(vb + (BN + i) * 4), "f"(wv) : "memory");
                asm volatile("st.shared.f32 [%0], %1;" ::"r"(vb + (2 * BN + i) * 4), "f"(gv) : "memory");
            }
            named_bar_sync(1, 32 * EPI_WARPS);
            const int rowbase = mt * 256 + (int)rank * BM + q * 32;
            const int row = rowbase + lane;
            const bool row_ok = row < p.m;
            if (((has_res && !tma_res) || has_tdc) && row_ok && chalf == 0) {
                // this tile's row segments of the epilogue's global inputs -> L2 while the
                // mainloop still runs (one bulk prefetch per row and tensor)
                const uint32_t seg = (uint32_t)min(BN, p.n - n0) * 2;
                if (has_res && !tma_res) bulk_prefetch_l2(p.residual + (size_t)row * p.ldr + n0, seg);
                if (has_tdc) {
                    bulk_prefetch_l2(p.tdc_x_in + (size_t)row * p.n + n0, seg);
                    bulk_prefetch_l2(p.tdc_delta + (size_t)row * p.n + n0, seg);
                }
            }
            float sa = 0.0f;
            if constexpr (I8) sa = row_ok ? p.a_scale[row] : 0.0f;
            const f2 sa2 = f2make(sa, sa);
            const int n_here = min(BN, p.n - n0);
            const int nch_here = (n_here + 31) >> 5;
            const int my_last = nch_here > chalf ? chalf + ((nch_here - 1 - chalf) / CSTEP) * CSTEP : -1;
            const int nmine = my_last < 0 ? 0 : (my_last - chalf) / CSTEP + 1;   // this warp's chunks of the tile
            // staging iterations of the tile: one per chunk of this warp, or (paired) one per chunk pair
            const int niter = PAIRST ? (nch_here + 1) >> 1 : nmine;
            constexpr int NSB = L::STAGING_BUFS;
            // residual chunk j of this warp -> staging buffer (chunk_ctr + j) % NSB, by TMA; the first
            // NSB chunks are requested now, while the mainloop of this tile still runs
            const uint32_t ctr0 = chunk_ctr;   // this tile's first chunk counter
            auto res_load = [&](int j) {
                const uint32_t cj = ctr0 + (uint32_t)j;
                mbar_arrive_expect_tx(bar_res + 8 * (sb_id * 3 + (int)(cj % NSB)), SBUF);
                tma_load_2d(staging + (cj % NSB) * SBUF, &tmR, PAIRST ? n0 + j * 64 : n0 + (chalf + j * CSTEP) * 32, rowbase,
                            bar_res + 8 * (sb_id * 3 + (int)(cj % NSB)));
            };
            if (tma_res && niter > 0 && issuer) {
                if (lane == 0) {
                    bulk_wait_read0();   // every earlier store of this warp has read its staging buffer
                    for (int j = 0; j < NSB && j < niter; ++j) res_load(j);
                }
                __syncwarp();
            }
            mbar_wait(bar_tfull + 8 * acc, acc_phase);
            tc_fence_after();
            if (my_last < 0) {   // no chunk for this warp in a narrow tile: release TMEM right away
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_cluster(leader_addr(bar_tempty + 8 * acc));
            }
            for (int jc = 0; jc < niter; ++jc) {   // jc: staging iteration of the tile
                const int c = chalf + jc * CSTEP;      // this warp's chunk (paired: none past the tile's last)
                const uint32_t buf = staging + (chunk_ctr % NSB) * SBUF;
                const uint32_t rbar = bar_res + 8 * (sb_id * 3 + (int)(chunk_ctr % NSB));
                const uint32_t rphase = (chunk_ctr / NSB) & 1;
                // this lane's 16-byte piece v4 (0..3) of its row in the staging buffer
                auto sptr = [&](int v4) -> uint32_t {
                    return PAIRST ? buf + lane * 128 + (((uint32_t)(chalf * 4 + v4) ^ (lane & 7)) << 4)      // 128B swizzle
                                  : buf + lane * 64 + (((uint32_t)v4 ^ ((lane >> 1) & 3)) << 4);             // 64B swizzle
                };
                if (c < nch_here) {
                // gated-residual chunk (TMA-staged: requested ahead, see res_load; else loaded
                // here, before the TMEM read so the two latencies overlap)
                uint4 rv4[4];
                if (!tma_res && has_res && row_ok) {
                    const uint4* rp = reinterpret_cast<const uint4*>(p.residual + (size_t)row * p.ldr + n0 + c * 32);
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4) rv4[v4] = __ldg(rp + v4);
                }
                uint32_t r[32];
                tmem_ld_32x32b_x32(tmem_base + ((uint32_t)(q * 32) << 16) + (NACC == 2 ? acc * BN : 0) + c * 32, r);
                tmem_ld_wait();
                if (c == my_last) {   // this warp's last TMEM read of the accumulator
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_cluster(leader_addr(bar_tempty + 8 * acc));
                }
                const int col0 = n0 + c * 32;
                f2 y[16];
#pragma unroll
                for (int v4 = 0; v4 < 8; ++v4) {
                    float b0, b1, b2, b3;
                    asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                 : "=f"(b0), "=f"(b1), "=f"(b2), "=f"(b3) : "r"(vb + (c * 32 + v4 * 4) * 4));
                    const f2 bb0 = f2make(b0, b1), bb1 = f2make(b2, b3);
                    if constexpr (!I8) {
                        const f2 a0 = f2make(__uint_as_float(r[4 * v4]), __uint_as_float(r[4 * v4 + 1]));
                        const f2 a1 = f2make(__uint_as_float(r[4 * v4 + 2]), __uint_as_float(r[4 * v4 + 3]));
                        f2 g0 = gg2, g1 = gg2;
                        if (gcol) {   // per-column fl(g_a g_w[n]) staged with the tile's vectors
                            float w0, w1, w2, w3;
                            asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                         : "=f"(w0), "=f"(w1), "=f"(w2), "=f"(w3) : "r"(vb + (BN + c * 32 + v4 * 4) * 4));
                            g0 = f2make(w0, w1);
                            g1 = f2make(w2, w3);
                        }
                        // y = fma(acc, g_a*g_w, bias): one rounding (FP32 tolerance path, R3)
                        y[2 * v4] = fma2(a0, g0, bb0);
                        y[2 * v4 + 1] = fma2(a1, g1, bb1);
                    } else {
                        float w0, w1, w2, w3;
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(w0), "=f"(w1), "=f"(w2), "=f"(w3) : "r"(vb + (BN + c * 32 + v4 * 4) * 4));
                        const f2 a0 = f2make(__int2float_rn((int)r[4 * v4]), __int2float_rn((int)r[4 * v4 + 1]));
                        const f2 a1 = f2make(__int2float_rn((int)r[4 * v4 + 2]), __int2float_rn((int)r[4 * v4 + 3]));
                        // y = fma(fl(float(acc) * s_a), s_w, bias)  (R8; bias -0.0 when absent)
                        y[2 * v4] = fma2(mul2(a0, sa2), f2make(w0, w1), bb0);
                        y[2 * v4 + 1] = fma2(mul2(a1, sa2), f2make(w2, w3), bb1);
                    }
                }
                if (has_gelu) {   // GELU-tanh glue (R13), packed: 0.5x(1 + tanh(k0 (x + k1 x^3)))
                    const f2 k1 = f2make(0.044715f, 0.044715f), k0 = f2make(0.7978845608028654f, 0.7978845608028654f);
                    const f2 hf = f2make(0.5f, 0.5f);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const f2 x = y[j];
                        const f2 x3 = mul2(mul2(x, x), x);
                        const f2 u = mul2(k0, fma2(k1, x3, x));
                        const f2 t = f2make(tanh_approx(f2lo(u)), tanh_approx(f2hi(u)));
                        const f2 h = mul2(hf, x);
                        y[j] = fma2(h, t, h);
                    }
                }
                if (tma_res) {   // this lane's row of the staged chunk (64-byte swizzle, as the store)
                    mbar_wait(rbar, rphase);
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4) {
                        const uint32_t a = sptr(v4);
                        asm volatile("ld.shared.v4.b32 {%0, %1, %2, %3}, [%4];"
                                     : "=r"(rv4[v4].x), "=r"(rv4[v4].y), "=r"(rv4[v4].z), "=r"(rv4[v4].w) : "r"(a) : "memory");
                    }
                }
                if (has_res && row_ok) {
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4) {
                        const uint4 rv = rv4[v4];
                        const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
                        float g0, g1, g2, g3, g4, g5, g6, g7;
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(g0), "=f"(g1), "=f"(g2), "=f"(g3) : "r"(vb + (2 * BN + c * 32 + v4 * 8) * 4));
                        asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
                                     : "=f"(g4), "=f"(g5), "=f"(g6), "=f"(g7) : "r"(vb + (2 * BN + c * 32 + v4 * 8 + 4) * 4));
                        const f2 gp[4] = {f2make(g0, g1), f2make(g2, g3), f2make(g4, g5), f2make(g6, g7)};
#pragma unroll
                        for (int j = 0; j < 4; ++j)   // y = fma(gate, y, res)
                            y[v4 * 4 + j] = fma2(gp[j], y[v4 * 4 + j], f2make(bf16lo(w[j]), bf16hi(w[j])));
                    }
                }
                uint32_t yb[16];   // the stored bf16 output (X_out for the fused TDC refresh)
#pragma unroll
                for (int j = 0; j < 16; ++j) yb[j] = pack_bf16x2_f2(y[j]);
                if constexpr (QNT) {
                    // producer-fused NVFP4 quantization of v = bf16(y) (Eq. 2, R3/R4, IEEE block-scale
                    // arithmetic = dmpq_quantize_act's): two 16-element blocks per 32-column chunk
                    if (row < p.q_m_pad) {
                        uint32_t sc = 0;
                        if (row_ok) {
                            uint32_t cw[4];
#pragma unroll
                            for (int h = 0; h < 2; ++h) {
                                float a = 0.0f;
#pragma unroll
                                for (int j = 0; j < 8; ++j)
                                    a = fmaxf(a, fmaxf(fabsf(bf16lo(yb[8 * h + j])), fabsf(bf16hi(yb[8 * h + j]))));
                                const uint32_t sb = e4m3_rn_satfinite(__fdiv_rn(__fdiv_rn(a, 6.0f), qg));
                                const float eff = __fmul_rn(e4m3_decode(sb), qg);
                                const float rq = eff > 0.0f ? __frcp_rn(eff) : 0.0f;
                                const f2 r2 = f2make(rq, rq);
                                f2 v[8];
#pragma unroll
                                for (int j = 0; j < 8; ++j) v[j] = mul2(f2make(bf16lo(yb[8 * h + j]), bf16hi(yb[8 * h + j])), r2);
                                cw[2 * h] = e2m1x8(v[0], v[1], v[2], v[3]);
                                cw[2 * h + 1] = e2m1x8(v[4], v[5], v[6], v[7]);
                                sc |= sb << (8 * h);
                                qamax = fmaxf(qamax, a);
                            }
                            *reinterpret_cast<uint4*>(p.q_codes + (size_t)row * (p.n >> 1) + (col0 >> 1)) =
                                make_uint4(cw[0], cw[1], cw[2], cw[3]);
                        }
                        *reinterpret_cast<uint16_t*>(sf_row_ptr(p.q_sf, p.q_kc4, row) + (size_t)(col0 >> 6) * 512 +
                                                     ((col0 >> 4) & 3)) = (uint16_t)sc;
                    }
                }
                if (p.Y) {
                    if (!tma_res && !PAIRST) {
                        if (lane == 0) {   // the store issued from this buffer (2 chunks ago / last chunk) has read it
                            if constexpr (L::STAGING_BUFS == 3) bulk_wait_read2();
                            else if constexpr (L::STAGING_BUFS == 2) bulk_wait_read1();
                            else bulk_wait_read0();
                        }
                        __syncwarp();
                    }
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4)
                        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(sptr(v4)), "r"(yb[4 * v4]),
                                     "r"(yb[4 * v4 + 1]), "r"(yb[4 * v4 + 2]), "r"(yb[4 * v4 + 3])
                                     : "memory");
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (!PAIRST && lane == 0) {
                        tma_store_2d(&tmY, buf, col0, rowbase);
                        bulk_commit();
                        if (tma_res && jc + NSB < nmine) {   // this buffer's next residual chunk, once the store has read it
                            bulk_wait_read0();
                            res_load(jc + NSB);
                        }
                    }
                }
                if (has_tdc && row_ok) {
                    // TDC refresh (Eq. 8) with tdc_step's arithmetic: d = fl(X_out - X_in),
                    // Delta_new = bf16(d); Gamma / L2 sums FP32 per 8-element vector then FP64,
                    // cosine sums exact bf16 products in FP64 (R12)
                    const size_t off = (size_t)row * p.n + col0;
                    const uint4* xp = reinterpret_cast<const uint4*>(p.tdc_x_in + off);
                    uint4* dp = reinterpret_cast<uint4*>(p.tdc_delta + off);
#pragma unroll
                    for (int v = 0; v < 4; ++v) {
                        const uint4 xv = __ldg(xp + v), pv = dp[v];
                        const uint32_t xw[4] = {xv.x, xv.y, xv.z, xv.w}, pw[4] = {pv.x, pv.y, pv.z, pv.w};
                        float sv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
                        uint32_t o[4];
#pragma unroll
                        for (int j = 0; j < 4; ++j) {
                            const uint32_t yw = yb[4 * v + j];
                            const float xa = bf16lo(xw[j]), xb = bf16hi(xw[j]);
                            const float da = __fsub_rn(bf16lo(yw), xa), db = __fsub_rn(bf16hi(yw), xb);
                            o[j] = pack_bf16x2(da, db);
                            const double na = (double)bf16lo(o[j]), nb = (double)bf16hi(o[j]);
                            const double pa = (double)bf16lo(pw[j]), pb = (double)bf16hi(pw[j]);
                            sv[0] = __fadd_rn(sv[0], __fadd_rn(fabsf(da), fabsf(db)));
                            sv[1] = __fadd_rn(sv[1], __fadd_rn(fabsf(xa), fabsf(xb)));
                            sv[2] = __fadd_rn(sv[2], __fadd_rn(__fmul_rn(da, da), __fmul_rn(db, db)));
                            sv[3] = __fadd_rn(sv[3], __fadd_rn(__fmul_rn(xa, xa), __fmul_rn(xb, xb)));
                            tacc[4] = __fma_rn(na, pa, tacc[4]); tacc[4] = __fma_rn(nb, pb, tacc[4]);
                            tacc[5] = __fma_rn(na, na, tacc[5]); tacc[5] = __fma_rn(nb, nb, tacc[5]);
                            tacc[6] = __fma_rn(pa, pa, tacc[6]); tacc[6] = __fma_rn(pb, pb, tacc[6]);
                        }
                        dp[v] = make_uint4(o[0], o[1], o[2], o[3]);
#pragma unroll
                        for (int j = 0; j < 4; ++j) tacc[j] = __dadd_rn(tacc[j], (double)sv[j]);
                    }
                }
                if (row_ok) {
                    if (p.Y32) {
                        float4* yp = reinterpret_cast<float4*>(p.Y32 + (size_t)row * p.n + col0);
#pragma unroll
                        for (int v4 = 0; v4 < 8; ++v4)
                            yp[v4] = make_float4(f2lo(y[2 * v4]), f2hi(y[2 * v4]), f2lo(y[2 * v4 + 1]), f2hi(y[2 * v4 + 1]));
                    }
                    if constexpr (I8) {
                        if (p.acc_out) {
                            int4* ap = reinterpret_cast<int4*>(p.acc_out + (size_t)row * p.n + col0);
#pragma unroll
                            for (int v4 = 0; v4 < 8; ++v4)
                                ap[v4] = make_int4((int)r[4 * v4], (int)r[4 * v4 + 1], (int)r[4 * v4 + 2], (int)r[4 * v4 + 3]);
                        }
                    }
                }
                }   // c < nch_here
                if (p.Y) {
                    if constexpr (PAIRST) {
                        // both halves written: one TMA store of the 32 x 64 box. Without a TMA-staged
                        // residual the issuer first lets the store NSB - 1 iterations back finish reading
                        // its buffer, so this barrier also frees the next iteration's buffer.
                        if (!tma_res && issuer && lane == 0) {
                            if constexpr (L::STAGING_BUFS == 3) bulk_wait_read1();
                            else bulk_wait_read0();
                        }
                        named_bar_sync(2 + q, 64);
                        if (issuer && lane == 0) {
                            tma_store_2d(&tmY, buf, n0 + jc * 64, rowbase);
                            bulk_commit();
                            if (tma_res && jc + NSB < niter) {   // this buffer's next residual chunk pair
                                bulk_wait_read0();
                                res_load(jc + NSB);
                            }
                        }
                        __syncwarp();
                    }
                    ++chunk_ctr;
                }
            }
        }
        if (has_tdc) {
            // per-warp partial (fixed butterfly), then the last warp of the grid sums the
            // partials in slot order: deterministic for a given grid
#pragma unroll
            for (int j = 0; j < 7; ++j) tacc[j] = warp_sum_d(tacc[j]);
            const int nslots = (int)gridDim.x * EPI_WARPS;
            const int slot = (int)blockIdx.x * EPI_WARPS + ew;
            unsigned int last = 0;
            if (lane == 0) {
#pragma unroll
                for (int j = 0; j < 7; ++j) p.tdc_partials[(size_t)slot * 7 + j] = tacc[j];
                __threadfence();
                last = (atomicAdd(p.tdc_counter, 1u) == (unsigned)nslots - 1u) ? 1u : 0u;
            }
            last = __shfl_sync(0xffffffffu, last, 0);
            if (last) {
                __threadfence();
                double v[7] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
                for (int i = lane; i < nslots; i += 32)
#pragma unroll
                    for (int j = 0; j < 7; ++j) v[j] = __dadd_rn(v[j], __ldcg(p.tdc_partials + (size_t)i * 7 + j));
#pragma unroll
                for (int j = 0; j < 7; ++j) v[j] = warp_sum_d(v[j]);
                if (lane == 0) {
#pragma unroll
                    for (int j = 0; j < 7; ++j) p.tdc_stats[j] = v[j];
                    *p.tdc_counter = 0u;   // ready for the next call
                }
            }
        }
        if constexpr (QNT) {
            qamax = warp_max(qamax);
            if (lane == 0) atomic_max_nonneg(p.q_amax, qamax);
        }
        if (lane == 0) bulk_wait_all();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 2) tmem_dealloc_pair(tmem_base, TMEM_COLS);
}

// ============================================================================
// Per-block INT8 GEMM ("per-block symmetric INT8"; R17, NEXT-1): A carries one
// scale per 128-element K block of each row, so K blocks cannot share one integer accumulator.
// The kind::i8 MMAs of one 128-K block accumulate exactly into a TMEM partial (two partials
// ping-pong), and the epilogue warps promote every partial into FP32 registers,
//   t += float(P_b) * s_a[row][b]    (float(P_b) exact: |P_b| <= 128 * 127 * 128 < 2^24),
// then y = fma(t, s_w[n], bias[n]) (+ GELU / gated-residual glue). One promotion (a conversion
// and an FMA) per output element per 128-K block costs about as many issue slots as the MMA
// takes cycles, so this kernel is epilogue-bound by construction.
// CTA pair, 256 x 192 tiles, 12 epilogue warps (3 per TMEM lane quarter, 64 columns each).
// ============================================================================
constexpr int I8B_BN = 192;
constexpr int I8B_EPI_WARPS = 12;
constexpr int I8B_STAGES = 5;

struct I8BLayout {
    static constexpr int A_BYTES = BM * BK_BYTES;                   // 16 KB
    static constexpr int B_BYTES = (I8B_BN / 2) * BK_BYTES;         // 12 KB
    static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
    static constexpr int PAIR_TX = 2 * STAGE_BYTES;
    static constexpr int BAR_OFFSET = I8B_STAGES * STAGE_BYTES;
    static constexpr int TOTAL = BAR_OFFSET + 256 + 1024;
    static_assert(STAGE_BYTES % 1024 == 0, "stage alignment");
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128 + 32 * I8B_EPI_WARPS, 1)
    dmpq_gemm_i8b_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                         const GemmParams p) {
    using L = I8BLayout;
    constexpr int BN = I8B_BN;
    if (p.run_if && *p.run_if != p.run_if_value) return;
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    const uint32_t sbase = smem_u32(smem);
    const uint32_t bar_full = sbase + L::BAR_OFFSET;
    const uint32_t bar_empty = bar_full + I8B_STAGES * 8;
    const uint32_t bar_pfull = bar_empty + I8B_STAGES * 8;
    const uint32_t bar_pempty = bar_pfull + 2 * 8;
    uint32_t* tmem_holder = reinterpret_cast<uint32_t*>(smem + L::BAR_OFFSET + 2 * I8B_STAGES * 8 + 4 * 8);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_ctarank();
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tmA);
        prefetch_tmap(&tmB);
        for (int s = 0; s < I8B_STAGES; ++s) {
            mbar_init(bar_full + 8 * s, 1);
            mbar_init(bar_empty + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            mbar_init(bar_pfull + 8 * a, 1);
            mbar_init(bar_pempty + 8 * a, 2 * I8B_EPI_WARPS);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc_pair(smem_u32(tmem_holder), 512);
    tc_fence_before();
    cluster_sync();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_holder;
    const int num_tiles = p.num_m_tiles * p.num_n_tiles;
    const int cid = (int)cluster_id_x(), ncl = (int)nclusters_x();
    int ts0, ts1, tstep;
    tile_span(cid, ncl, num_tiles, ts0, ts1, tstep);

    if (warp == 0) {
        // ===== TMA producer (as the INT8 pair kernel)
        int stage = 0;
        uint32_t phase = 0;
        for (int tile = ts0; tile < ts1; tile += tstep) {
            const int mt = tile / p.num_n_tiles, nt = tile % p.num_n_tiles;
            const int m0 = mt * 256 + (int)rank * BM;
            const int nb0 = nt * BN + (int)rank * (BN / 2);
            for (int kb = 0; kb < p.num_kb; ++kb) {
                mbar_wait(bar_empty + 8 * stage, phase ^ 1);
                if (elect_one()) {
                    const uint32_t full_l = leader_addr(bar_full + 8 * stage);
                    if (rank == 0) mbar_arrive_expect_tx(bar_full + 8 * stage, L::PAIR_TX);
                    const uint32_t sA = sbase + stage * L::STAGE_BYTES;
                    tma_load_2d_pair(sA, &tmA, kb * BK_BYTES, m0, full_l);
                    tma_load_2d_pair(sA + L::A_BYTES, &tmB, kb * BK_BYTES, nb0, full_l);
                }
                __syncwarp();
                if (++stage == I8B_STAGES) { stage = 0; phase ^= 1; }
            }
        }
    } else if (warp == 1) {
        // ===== MMA issuer (leader CTA): one TMEM partial per 128-K block, two partials ping-pong
        if (rank == 0) {
            int stage = 0;
            uint32_t phase = 0, g = 0;
            const uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
            for (int tile = ts0; tile < ts1; tile += tstep) {
                for (int kb = 0; kb < p.num_kb; ++kb, ++g) {
                    const uint32_t pb = g & 1u, pph = (g >> 1) & 1u;
                    mbar_wait(bar_pempty + 8 * pb, pph ^ 1);     // the epilogue has read this partial's last use
                    tc_fence_after();
                    mbar_wait(bar_full + 8 * stage, phase);
                    tc_fence_after();
                    if (elect_one()) {
                        const uint32_t sA = sbase + stage * L::STAGE_BYTES;
                        const uint64_t adesc = sdesc_k_sw128(sA), bdesc = sdesc_k_sw128(sA + L::A_BYTES);
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            mma_i8_pair(tmem_base + pb * BN, adesc + 2 * j, bdesc + 2 * j, idesc, j ? 1u : 0u);
                        tc_commit_pair_mc(bar_empty + 8 * stage, 0x3);
                        tc_commit_pair_mc(bar_pfull + 8 * pb, 0x3);
                    }
                    __syncwarp();
                    if (++stage == I8B_STAGES) { stage = 0; phase ^= 1; }
                }
            }
        }
    } else if (warp >= 4) {
        // ===== epilogue: promotion of every K-block partial, then the output of the tile
        const int q = warp & 3, ew = warp - 4, csub = ew >> 2;   // lane quarter, 64-column slice
        const bool has_bias = (p.flags & DMPQ_EP_BIAS) != 0, has_gelu = (p.flags & DMPQ_EP_GELU_TANH) != 0;
        const bool has_res = (p.flags & DMPQ_EP_RESIDUAL) != 0;
        uint32_t g = 0;
        for (int tile = ts0; tile < ts1; tile += tstep) {
            const int mt = tile / p.num_n_tiles, nt = tile % p.num_n_tiles;
            const int row = mt * 256 + (int)rank * BM + q * 32 + lane;
            const bool row_ok = row < p.m;
            const float* sa_row = p.a_scale + (size_t)(row_ok ? row : 0) * p.num_kb;
            f2 acc[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) acc[i] = f2make(0.0f, 0.0f);
            float s_next = row_ok ? __ldg(sa_row) : 0.0f;
            for (int kb = 0; kb < p.num_kb; ++kb, ++g) {
                const uint32_t pb = g & 1u, pph = (g >> 1) & 1u;
                const float s = s_next;
                if (kb + 1 < p.num_kb && row_ok) s_next = __ldg(sa_row + kb + 1);
                const f2 s2 = f2make(s, s);
                mbar_wait(bar_pfull + 8 * pb, pph);
                tc_fence_after();
                const uint32_t taddr = tmem_base + ((uint32_t)(q * 32) << 16) + pb * BN + csub * 64;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    // (measured: four pipelined 16-column loads with an integer-add / subtract
                    // conversion instead of I2F were 18 % slower -- the promotion is issue-bound)
                    uint32_t r[32];
                    tmem_ld_32x32b_x32(taddr + h * 32, r);
                    tmem_ld_wait();
                    if (h == 1) {   // both halves in registers: release the partial to the MMA
                        tc_fence_before();
                        __syncwarp();
                        if (lane == 0) mbar_arrive_cluster(leader_addr(bar_pempty + 8 * pb));
                    }
#pragma unroll
                    for (int i = 0; i < 16; ++i) {
                        const f2 a = f2make(__int2float_rn((int)r[2 * i]), __int2float_rn((int)r[2 * i + 1]));
                        acc[16 * h + i] = fma2(a, s2, acc[16 * h + i]);
                    }
                }
            }
            // output: y = fma(t, s_w[n], bias[n]), glue, bf16 / fp32 stores (lane = row)
#pragma unroll
            for (int c = 0; c < 2; ++c) {
                const int col0 = nt * BN + csub * 64 + c * 32;
                if (col0 >= p.n || !row_ok) continue;
                f2 y[16];
#pragma unroll
                for (int v4 = 0; v4 < 8; ++v4) {
                    const float4 w4 = __ldg(reinterpret_cast<const float4*>(p.w_scale + col0) + v4);
                    const float4 b4 = has_bias ? __ldg(reinterpret_cast<const float4*>(p.bias + col0) + v4)
                                               : make_float4(-0.0f, -0.0f, -0.0f, -0.0f);
                    y[2 * v4] = fma2(acc[16 * c + 2 * v4], f2make(w4.x, w4.y), f2make(b4.x, b4.y));
                    y[2 * v4 + 1] = fma2(acc[16 * c + 2 * v4 + 1], f2make(w4.z, w4.w), f2make(b4.z, b4.w));
                }
                if (has_gelu) {
                    const f2 k1 = f2make(0.044715f, 0.044715f), k0 = f2make(0.7978845608028654f, 0.7978845608028654f);
                    const f2 hf = f2make(0.5f, 0.5f);
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        const f2 x = y[j];
                        const f2 u = mul2(k0, fma2(k1, mul2(mul2(x, x), x), x));
                        const f2 t = f2make(tanh_approx(f2lo(u)), tanh_approx(f2hi(u)));
                        const f2 hh = mul2(hf, x);
                        y[j] = fma2(hh, t, hh);
                    }
                }
                if (has_res) {
                    const uint4* rp = reinterpret_cast<const uint4*>(p.residual + (size_t)row * p.ldr + col0);
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4) {
                        const uint4 rv = __ldg(rp + v4);
                        const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
                        const float4 ga = __ldg(reinterpret_cast<const float4*>(p.gate + col0) + 2 * v4);
                        const float4 gb = __ldg(reinterpret_cast<const float4*>(p.gate + col0) + 2 * v4 + 1);
                        const f2 gp[4] = {f2make(ga.x, ga.y), f2make(ga.z, ga.w), f2make(gb.x, gb.y), f2make(gb.z, gb.w)};
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            y[v4 * 4 + j] = fma2(gp[j], y[v4 * 4 + j], f2make(bf16lo(w[j]), bf16hi(w[j])));
                    }
                }
                if (p.Y) {
                    uint4* yp = reinterpret_cast<uint4*>(p.Y + (size_t)row * p.ldy + col0);
#pragma unroll
                    for (int v4 = 0; v4 < 4; ++v4)
                        yp[v4] = make_uint4(pack_bf16x2_f2(y[4 * v4]), pack_bf16x2_f2(y[4 * v4 + 1]),
                                            pack_bf16x2_f2(y[4 * v4 + 2]), pack_bf16x2_f2(y[4 * v4 + 3]));
                }
                if (p.Y32) {
                    float4* yp = reinterpret_cast<float4*>(p.Y32 + (size_t)row * p.n + col0);
#pragma unroll
                    for (int v4 = 0; v4 < 8; ++v4)
                        yp[v4] = make_float4(f2lo(y[2 * v4]), f2hi(y[2 * v4]), f2lo(y[2 * v4 + 1]), f2hi(y[2 * v4 + 1]));
                }
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();
    if (warp == 2) tmem_dealloc_pair(tmem_base, 512);
}

// ------------------------------------------------------------------ host side


// 2-D uint8 tensor map over a [rows x row_bytes] row-major matrix, box 128 B x box_rows, 128-B swizzle.
static bool make_tmap(CUtensorMap* tm, const void* base, int rows, int row_bytes, int box_rows) {
    auto enc = tmap_encode_fn();
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

// 3-D view of a swizzled scale buffer: [row_tiles][kc4 atoms][128 x u32 (512 B)], box {128, 4, box_tiles}.
static bool make_tmap_sf(CUtensorMap* tm, const void* base, int row_tiles, int kc4, int box_tiles) {
    auto enc = tmap_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[3] = {128, (cuuint64_t)kc4, (cuuint64_t)row_tiles};
    cuuint64_t strides[2] = {512, (cuuint64_t)kc4 * 512};
    cuuint32_t box[3] = {128, 4, (cuuint32_t)box_tiles};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_UINT32, 3, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

// bf16 output [rows x cols] (row stride ld elements), box 32 x 32 with 64-B swizzle, or (wide, paired
// epilogue staging) 32 rows x 64 columns with 128-B swizzle (epilogue TMA store / residual load).
static bool make_tmap_y(CUtensorMap* tm, const void* base, int rows, int cols, int ld, bool wide) {
    auto enc = tmap_encode_fn();
    if (!enc) return false;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
    cuuint32_t box[2] = {wide ? 64u : 32u, 32};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = enc(tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, estr,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, wide ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    return r == CUDA_SUCCESS;
}

template <int KIND, int BN, int STAGES, bool TDC = false, bool QNT = false, int CL = 2>
static dmpq_status set_pair_attrs() {
    using L = PairLayout<KIND, BN, STAGES>;
    if (cudaFuncSetAttribute(dmpq_gemm_pair_kernel<KIND, BN, STAGES, TDC, QNT, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             L::TOTAL) != cudaSuccess)
        return check_launch("dmpq_gemm(smem attribute)");
    return DMPQ_OK;
}

template <int KIND, int BN, int STAGES, bool TDC = false, bool QNT = false, int CL = 2>
static dmpq_status launch_gemm_pair(GemmParams p, const void* a_codes, const void* w_codes, cudaStream_t s) {
    using L = PairLayout<KIND, BN, STAGES>;
    constexpr bool FP4 = KIND == 1;
    CUtensorMap tmA, tmB, tmSFA, tmSFB, tmY, tmR;
    std::memset(&tmSFA, 0, sizeof(tmSFA));
    std::memset(&tmSFB, 0, sizeof(tmSFB));
    std::memset(&tmY, 0, sizeof(tmY));
    std::memset(&tmR, 0, sizeof(tmR));
    if (!make_tmap(&tmA, a_codes, p.m, p.kbytes, BM) || !make_tmap(&tmB, w_codes, p.n, p.kbytes, BN / CL))
        return set_error(DMPQ_ECUDA, "dmpq_gemm: cuTensorMapEncodeTiled failed (A/B)");
    if constexpr (FP4) {
        if (!make_tmap_sf(&tmSFA, p.sfa, (p.m + 127) / 128, p.kc4, 1) ||
            !make_tmap_sf(&tmSFB, p.sfb, p.sfb_row_tiles, p.kc4, (CL == 4 || DMPQ_SFB_MC) ? 1 : 2))
            return set_error(DMPQ_ECUDA, "dmpq_gemm: cuTensorMapEncodeTiled failed (scales)");
    }
    if (p.Y && !make_tmap_y(&tmY, p.Y, p.m, p.n, p.ldy, L::PAIRED))
        return set_error(DMPQ_ECUDA, "dmpq_gemm: cuTensorMapEncodeTiled failed (Y)");
    if (p.Y && (p.flags & DMPQ_EP_RESIDUAL) && !make_tmap_y(&tmR, p.residual, p.m, p.n, p.ldr, L::PAIRED))
        return set_error(DMPQ_ECUDA, "dmpq_gemm: cuTensorMapEncodeTiled failed (residual)");
    p.num_m_tiles = (p.m + 255) / 256;
    p.num_n_tiles = (p.n + BN - 1) / BN;
    p.num_kb = (p.kbytes + BK_BYTES - 1) / BK_BYTES;
    auto kern = dmpq_gemm_pair_kernel<KIND, BN, STAGES, TDC, QNT, CL>;
    static bool attr_set = false;   // per process and kernel (dmpq_prepare sets them ahead of graph capture)
    if (!attr_set) {
        dmpq_status rc = set_pair_attrs<KIND, BN, STAGES, TDC, QNT, CL>();
        if (rc != DMPQ_OK) return rc;
        attr_set = true;
    }
    const int tiles = (CL == 4 ? (p.num_m_tiles + 1) / 2 : p.num_m_tiles) * p.num_n_tiles;
    int clusters = num_sms() / CL;
    if constexpr (CL == 4) {   // 4-CTA clusters do not tile every GPC: size the persistent grid to what is co-resident
        static int max_active = 0;
        if (max_active == 0) {
            cudaLaunchConfig_t cfg = {};
            cfg.gridDim = dim3(CL * clusters);
            cfg.blockDim = dim3(128 + 32 * EPI_WARPS);
            cfg.dynamicSmemBytes = L::TOTAL;
            int n = 0;
            if (cudaOccupancyMaxActiveClusters(&n, kern, &cfg) != cudaSuccess || n < 1) {
                cudaGetLastError();
                n = clusters;
            }
            max_active = n;
        }
        if (clusters > max_active) clusters = max_active;
    }
    if (clusters > tiles) clusters = tiles;
    kern<<<CL * clusters, 128 + 32 * EPI_WARPS, L::TOTAL, s>>>(tmA, tmB, tmSFA, tmSFB, tmY, tmR, p);
    return check_launch("dmpq_gemm");
}

static dmpq_status launch_gemm_i8b(GemmParams p, const void* a_codes, const void* w_codes, cudaStream_t s) {
    using L = I8BLayout;
    CUtensorMap tmA, tmB;
    if (!make_tmap(&tmA, a_codes, p.m, p.kbytes, BM) || !make_tmap(&tmB, w_codes, p.n, p.kbytes, I8B_BN / 2))
        return set_error(DMPQ_ECUDA, "dmpq_gemm: cuTensorMapEncodeTiled failed (A/B)");
    p.num_m_tiles = (p.m + 255) / 256;
    p.num_n_tiles = (p.n + I8B_BN - 1) / I8B_BN;
    p.num_kb = p.kbytes / BK_BYTES;
    static bool attr_set = false;
    if (!attr_set) {
        if (cudaFuncSetAttribute(dmpq_gemm_i8b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, L::TOTAL) != cudaSuccess)
            return check_launch("dmpq_gemm(smem attribute, per-block INT8)");
        attr_set = true;
    }
    const int tiles = p.num_m_tiles * p.num_n_tiles;
    int clusters = num_sms() / 2;
    if (clusters > tiles) clusters = tiles;
    dmpq_gemm_i8b_kernel<<<2 * clusters, 128 + 32 * I8B_EPI_WARPS, L::TOTAL, s>>>(tmA, tmB, p);
    return check_launch("dmpq_gemm(per-block INT8)");
}

}  // namespace dmpq

using namespace dmpq;

// Stage-ring depth of the GEMM (tuning knob, DMPQ_GEMM_STAGES = 5 | 6; default 5: the 6-stage ring only fits with single-buffered output staging, measured slower on the N = 12288 layer).
// Cluster size of the plain INT8 / NVFP4 GEMMs (experiment knob DMPQ_GEMM_CLUSTER = 2 | 4; 4 = two CTA
// pairs sharing B / SFB tiles by TMA multicast).
static int gemm_cluster() {
    static int c = [] {
        const char* e = std::getenv("DMPQ_GEMM_CLUSTER");
        return (e && std::atoi(e) == 4) ? 4 : 2;
    }();
    return c;
}

static int gemm_stages() {
    static int st = [] {
        const char* e = std::getenv("DMPQ_GEMM_STAGES");
        return (e && std::atoi(e) == 6) ? 6 : 5;
    }();
    return st;
}

// fused TDC refresh workspace: partials of up to 1024 CTAs x EPI_WARPS warps, then the counter
constexpr size_t kTdcPartialBytes = (size_t)1024 * EPI_WARPS * 7 * sizeof(double);
extern "C" size_t dmpq_gemm_tdc_workspace_bytes(void) { return kTdcPartialBytes + 256; }

// NVFP4 tile width (experiment knob DMPQ_FP4_BN = 192 | 256; 256 = single-buffered accumulator).
static int fp4_bn() {
    static int bn = [] {
        const char* e = std::getenv("DMPQ_FP4_BN");
        return (e && std::atoi(e) == 256) ? 256 : 192;
    }();
    return bn;
}

extern "C" dmpq_status dmpq_prepare(void) {
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_prepare: needs an sm_100 device");
    dmpq_status rc = DMPQ_OK;
    if (gemm_stages() == 5) {
        rc = set_pair_attrs<0, 256, 5>();
        if (rc == DMPQ_OK) rc = set_pair_attrs<1, 192, 5>();
        if (rc == DMPQ_OK) rc = set_pair_attrs<2, 256, 5>();
    } else {
        rc = set_pair_attrs<0, 256, 6>();
        if (rc == DMPQ_OK) rc = set_pair_attrs<1, 192, 6>();
        if (rc == DMPQ_OK) rc = set_pair_attrs<2, 256, 6>();
    }
    if (rc == DMPQ_OK && fp4_bn() == 256) rc = set_pair_attrs<1, 256, 5>();
    if (rc == DMPQ_OK && gemm_cluster() == 4) rc = set_pair_attrs<1, 192, 5, false, false, 4>();
    if (rc == DMPQ_OK && gemm_cluster() == 4) rc = set_pair_attrs<0, 256, 5, false, false, 4>();
    if (rc == DMPQ_OK) rc = set_pair_attrs<0, 256, 5, true>();   // fused TDC refresh variants
    if (rc == DMPQ_OK) rc = set_pair_attrs<1, 192, 5, true>();
    if (rc == DMPQ_OK) rc = set_pair_attrs<2, 256, 5, true>();
    if (rc == DMPQ_OK) rc = set_pair_attrs<0, 256, 5, false, true>();   // producer-fused NVFP4 quantizer
    if (rc == DMPQ_OK) rc = set_pair_attrs<1, 192, 5, false, true>();
    if (rc == DMPQ_OK && cudaFuncSetAttribute(dmpq_gemm_i8b_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                              I8BLayout::TOTAL) != cudaSuccess)
        rc = check_launch("dmpq_prepare(per-block INT8 GEMM)");
    if (rc == DMPQ_OK) rc = prepare_quant_tma();
    if (rc == DMPQ_OK) rc = prepare_quant_had();
    return rc;
}

extern "C" dmpq_status dmpq_gemm(const dmpq_act* A, const dmpq_weights* W, const dmpq_epilogue* ep, uint16_t* Y, int ldy,
                                 float* Y32, int32_t* acc_or_null, dmpq_stream_t s) {
    DMPQ_REQUIRE(A && W, DMPQ_EINVAL, "dmpq_gemm: NULL operand");
    DMPQ_REQUIRE(A->fmt == DMPQ_FMT_INT8 || A->fmt == DMPQ_FMT_NVFP4 || A->fmt == DMPQ_FMT_BF16, DMPQ_EINVAL,
                 "dmpq_gemm: unknown format");
    const bool fp4 = A->fmt == DMPQ_FMT_NVFP4;
    const int m = A->m, n = W->n, k = A->k;
    DMPQ_REQUIRE(k == W->k && k > 0 && k % 64 == 0 && n > 0 && n % 32 == 0 && m >= 0, DMPQ_ESHAPE,
                 "dmpq_gemm: need A.k == W.k, k %% 64 == 0, n %% 32 == 0 (m=%d n=%d k=%d Wk=%d)", m, n, k, W->k);
    const bool qnt = ep && (ep->flags & DMPQ_EP_QUANT_NVFP4);
    DMPQ_REQUIRE(Y || Y32 || acc_or_null || qnt, DMPQ_EINVAL, "dmpq_gemm: no output");
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
    if (p.flags & DMPQ_EP_TDC_REFRESH) {
        DMPQ_REQUIRE(Y && ep->tdc_x_in && ep->tdc_delta && ep->tdc_stats && ep->tdc_workspace && aligned16(ep->tdc_x_in) &&
                         aligned16(ep->tdc_delta) && aligned16(ep->tdc_workspace),
                     DMPQ_EALIGN, "dmpq_gemm: DMPQ_EP_TDC_REFRESH needs Y and 16-byte aligned tdc_x_in / tdc_delta / workspace");
        p.tdc_x_in = ep->tdc_x_in; p.tdc_delta = ep->tdc_delta; p.tdc_stats = ep->tdc_stats;
        p.tdc_partials = reinterpret_cast<double*>(ep->tdc_workspace);
        p.tdc_counter = reinterpret_cast<unsigned int*>(reinterpret_cast<uint8_t*>(ep->tdc_workspace) + kTdcPartialBytes);
    }
    p.Y = Y; p.ldy = ldy; p.Y32 = Y32; p.acc_out = acc_or_null;
    if (ep) { p.run_if = ep->run_if; p.run_if_value = ep->run_if_value; }
    if (qnt) {
        const dmpq_act* q = ep->q_out;
        DMPQ_REQUIRE(q && q->fmt == DMPQ_FMT_NVFP4 && q->m == m && q->k == n && n % 64 == 0, DMPQ_ESHAPE,
                     "dmpq_gemm: DMPQ_EP_QUANT_NVFP4 needs an NVFP4 [m x n] q_out and n %% 64 == 0");
        DMPQ_REQUIRE(q->codes && q->sf && q->g && ep->q_amax && aligned16(q->codes) && aligned16(q->sf), DMPQ_EALIGN,
                     "dmpq_gemm: DMPQ_EP_QUANT_NVFP4 output pointers");
        DMPQ_REQUIRE(!(p.flags & DMPQ_EP_TDC_REFRESH) && A->scale_block == 0, DMPQ_EUNSUPPORTED,
                     "dmpq_gemm: the fused quantizer is built for the plain INT8 / NVFP4 kernels");
        p.q_codes = reinterpret_cast<uint8_t*>(q->codes); p.q_sf = q->sf; p.q_g = q->g; p.q_amax = ep->q_amax;
        p.q_kc4 = n / 64; p.q_m_pad = (m + 127) / 128 * 128;
    }
    if (m == 0) {
        if (p.flags & DMPQ_EP_TDC_REFRESH) {   // empty sums
            if (cudaMemsetAsync(ep->tdc_stats, 0, 7 * sizeof(double), reinterpret_cast<cudaStream_t>(s)) != cudaSuccess)
                return check_launch("dmpq_gemm(empty TDC stats)");
        }
        return DMPQ_OK;
    }
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_gemm: needs an sm_100 device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    const bool tdc = (p.flags & DMPQ_EP_TDC_REFRESH) != 0;
    if (fp4) {
        DMPQ_REQUIRE(A->codes && A->sf && A->g && W->fp4_codes && W->fp4_sf && W->fp4_g && aligned16(A->codes) &&
                         aligned16(A->sf) && aligned16(W->fp4_codes) && aligned16(W->fp4_sf),
                     DMPQ_EALIGN, "dmpq_gemm: NVFP4 operand pointers");
        p.kbytes = k / 2;
        p.sfa = A->sf; p.sfb = W->fp4_sf; p.g_a = A->g; p.g_w = W->fp4_g; p.g_w_col = W->fp4_g_col;
        p.kc4 = k / 64;
        p.sfb_row_tiles = (n + 127) / 128;
        if (tdc) return launch_gemm_pair<1, 192, 5, true>(p, A->codes, W->fp4_codes, st);
        if (qnt) return launch_gemm_pair<1, 192, 5, false, true>(p, A->codes, W->fp4_codes, st);
        if (fp4_bn() == 256) return launch_gemm_pair<1, 256, 5>(p, A->codes, W->fp4_codes, st);
        if (gemm_cluster() == 4) return launch_gemm_pair<1, 192, 5, false, false, 4>(p, A->codes, W->fp4_codes, st);
        return gemm_stages() == 5 ? launch_gemm_pair<1, 192, 5>(p, A->codes, W->fp4_codes, st)
                                 : launch_gemm_pair<1, 192, 6>(p, A->codes, W->fp4_codes, st);
    } else if (A->fmt == DMPQ_FMT_BF16) {
        DMPQ_REQUIRE(A->codes && W->bf16_w && aligned16(A->codes) && aligned16(W->bf16_w), DMPQ_EALIGN,
                     "dmpq_gemm: BF16 path needs A->codes (bf16 activation) and W->bf16_w");
        DMPQ_REQUIRE(!qnt, DMPQ_EUNSUPPORTED, "dmpq_gemm: the fused quantizer is built for the INT8 / NVFP4 kernels");
        p.kbytes = 2 * k;
        if (tdc) return launch_gemm_pair<2, 256, 5, true>(p, A->codes, W->bf16_w, st);
        return gemm_stages() == 5 ? launch_gemm_pair<2, 256, 5>(p, A->codes, W->bf16_w, st)
                                 : launch_gemm_pair<2, 256, 6>(p, A->codes, W->bf16_w, st);
    } else {
        DMPQ_REQUIRE(A->codes && A->row_scale && W->i8_codes && W->i8_scale && aligned16(A->codes) && aligned16(W->i8_codes),
                     DMPQ_EALIGN, "dmpq_gemm: INT8 operand pointers");
        p.kbytes = k;
        p.a_scale = A->row_scale; p.w_scale = W->i8_scale;
        if (A->scale_block != 0) {   // per-block symmetric INT8 activations (R17)
            DMPQ_REQUIRE(A->scale_block == 128 && k % 128 == 0, DMPQ_ESHAPE, "dmpq_gemm: per-block INT8 needs scale_block 128, k %% 128 == 0");
            DMPQ_REQUIRE(!tdc && !acc_or_null, DMPQ_EUNSUPPORTED, "dmpq_gemm: per-block INT8 has no fused refresh / raw accumulators");
            DMPQ_REQUIRE(!(p.flags & DMPQ_EP_RESIDUAL) || ep->ldr % 8 == 0, DMPQ_EALIGN, "dmpq_gemm: residual stride");
            return launch_gemm_i8b(p, A->codes, W->i8_codes, st);
        }
        if (tdc) return launch_gemm_pair<0, 256, 5, true>(p, A->codes, W->i8_codes, st);
        if (qnt) return launch_gemm_pair<0, 256, 5, false, true>(p, A->codes, W->i8_codes, st);
        if (gemm_cluster() == 4) return launch_gemm_pair<0, 256, 5, false, false, 4>(p, A->codes, W->i8_codes, st);
        return gemm_stages() == 5 ? launch_gemm_pair<0, 256, 5>(p, A->codes, W->i8_codes, st)
                                 : launch_gemm_pair<0, 256, 6>(p, A->codes, W->i8_codes, st);
    }
}
