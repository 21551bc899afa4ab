// pack.cu — dmpq_pack_weights: offline packing of one linear layer's weights in
// both formats ("all weights are quantized to NVFP4 offline ...
// cast to INT8" for INT8-routed layers; R7: the INT8 form is the
// per-output-channel symmetric INT8 of the dequantized NVFP4 weights).
// Runs once per layer at load time; not on the per-step hot path.
#include "common.cuh"

namespace dmpq {

__global__ void amax_bf16_kernel(const uint16_t* x, long long nvec, float* out) {
    float m = 0.0f;
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += (long long)gridDim.x * blockDim.x) {
        const uint4 v = ldg_stream(x + i * 8);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int j = 0; j < 4; ++j) m = fmaxf(m, fmaxf(fabsf(bf16lo(w[j])), fabsf(bf16hi(w[j]))));
    }
    m = warp_max(m);
    if ((threadIdx.x & 31) == 0) atomic_max_nonneg(out, m);
}

__device__ __forceinline__ float e2m1_value(uint32_t nib) {
    const float mag[8] = {0.0f, 0.5f, 1.0f, 1.5f, 2.0f, 3.0f, 4.0f, 6.0f};
    float v = mag[nib & 7];
    return (nib & 8) ? -v : v;
}

// One CTA per output row: W^ = fl(dec(code) * fl(dec(s_b) * g)); s_w = fl(max|W^|/127);
// code = RNE(fl(W^ * fl(127/max))).
__global__ void __launch_bounds__(256) pack_int8_from_fp4_kernel(const uint8_t* codes, const uint8_t* sf, const float* g_ptr,
                                                                 int n, int k, int kc4, int8_t* i8, float* i8_scale,
                                                                 float* i8_rcp) {
    __shared__ float red[8];
    const int row = blockIdx.x;
    if (row >= n) return;
    const float g = *g_ptr;
    const uint8_t* cr = codes + (size_t)row * (k / 2);
    const uint8_t* sr = sf + (size_t)(row >> 7) * kc4 * 512 + (row & 31) * 16 + ((row & 127) >> 5) * 4;
    auto what = [&](int j) -> float {  // dequantized weight j of this row
        const uint32_t byte = cr[j >> 1];
        const uint32_t nib = (j & 1) ? (byte >> 4) : (byte & 15u);
        const int c = j >> 4;
        const float eff = __fmul_rn(e4m3_decode(sr[(size_t)(c >> 2) * 512 + (c & 3)]), g);
        return __fmul_rn(e2m1_value(nib), eff);
    };
    float a = 0.0f;
    for (int j = threadIdx.x; j < k; j += blockDim.x) a = fmaxf(a, fabsf(what(j)));
    a = warp_max(a);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    a = 0.0f;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a = fmaxf(a, red[w]);
    const float rcp = a > 0.0f ? __fdiv_rn(127.0f, a) : 0.0f;
    if (threadIdx.x == 0) {
        i8_scale[row] = a > 0.0f ? __fdiv_rn(a, 127.0f) : 1.0f;
        if (i8_rcp) i8_rcp[row] = rcp;   // r_w for the on-the-fly cast (dmpq_cast_int8)
    }
    if (!i8) return;                     // NVFP4-only residency: INT8 codes are cast per GEMM
    for (int j = threadIdx.x; j < k; j += blockDim.x) {
        int c = __float2int_rn(__fmul_rn(what(j), rcp));
        i8[(size_t)row * k + j] = (int8_t)max(-128, min(127, c));
    }
}

// g[0] *= f and s[0..n) *= f for an exact power of two f; r[0..n) /= f (the cast's r_w: W^ scales
// by f with g, so fl(W^ f * r_w / f) = fl(W^ r_w) keeps the INT8 codes)
__global__ void scale_pow2_kernel(float* g, float* s, float* r, int n, float f) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i == 0) g[0] = __fmul_rn(g[0], f);
    if (i < n) {
        s[i] = __fmul_rn(s[i], f);
        if (r) r[i] = __fdiv_rn(r[i], f);
    }
}

}  // namespace dmpq

using namespace dmpq;

extern "C" dmpq_status dmpq_pack_weights(const uint16_t* W, int n, int k, dmpq_weights* out, dmpq_stream_t s) {
    return dmpq_pack_weights_ex(W, n, k, 0u, out, s);
}

extern "C" dmpq_status dmpq_pack_weights_ex(const uint16_t* W, int n, int k, uint32_t flags, dmpq_weights* out,
                                            dmpq_stream_t s) {
    DMPQ_REQUIRE(W && out, DMPQ_EINVAL, "dmpq_pack_weights: NULL argument");
    DMPQ_REQUIRE((flags & ~DMPQ_PACK_HADAMARD) == 0, DMPQ_EINVAL, "dmpq_pack_weights: unknown flags 0x%x", flags);
    const bool had = (flags & DMPQ_PACK_HADAMARD) != 0;
    DMPQ_REQUIRE(!had || k % 128 == 0, DMPQ_ESHAPE, "dmpq_pack_weights: DMPQ_PACK_HADAMARD needs k %% 128 == 0");
    DMPQ_REQUIRE(n > 0 && k > 0 && k % 64 == 0 && n % 16 == 0 && k <= 16384, DMPQ_ESHAPE,
                 "dmpq_pack_weights: need n %% 16 == 0, k %% 64 == 0, k <= 16384 (n=%d k=%d)", n, k);
    DMPQ_REQUIRE(out->n == n && out->k == k, DMPQ_ESHAPE, "dmpq_pack_weights: out->n/k mismatch");
    DMPQ_REQUIRE(out->fp4_codes && out->fp4_sf && out->fp4_g && (out->i8_codes || out->i8_rcp) && out->i8_scale &&
                     aligned16(W) && aligned16(out->fp4_codes) && aligned16(out->fp4_sf) && aligned16(out->i8_codes),
                 DMPQ_EALIGN, "dmpq_pack_weights: buffers must be non-NULL (i8_codes may be NULL with i8_rcp), "
                              "16-byte aligned device pointers");
    DMPQ_REQUIRE(device_is_sm100(), DMPQ_EUNSUPPORTED, "dmpq_pack_weights: needs an sm_100 device");
    cudaStream_t st = reinterpret_cast<cudaStream_t>(s);
    if (cudaMemsetAsync(out->fp4_g, 0, sizeof(float), st) != cudaSuccess) return check_launch("dmpq_pack_weights(memset)");
    dmpq_status rc;
    dmpq_act a{};
    a.fmt = DMPQ_FMT_NVFP4; a.m = n; a.k = k; a.codes = out->fp4_codes; a.sf = out->fp4_sf; a.g = out->fp4_g;
    dmpq_quant_opts had_opts{};
    had_opts.flags = DMPQ_QF_HADAMARD;
    if (had) {
        // pass 1: amax of the rotated weights (codes are overwritten by pass 2), with g = 1 in i8_scale[0]
        float* one = out->i8_scale;
        const float h_one = 1.0f;
        if (cudaMemcpyAsync(one, &h_one, sizeof(float), cudaMemcpyHostToDevice, st) != cudaSuccess)
            return check_launch("dmpq_pack_weights(memcpy)");
        dmpq_act probe = a;
        probe.g = one;
        rc = dmpq_quantize_act(W, n, k, k, &had_opts, nullptr, &probe, out->fp4_g, s);
        if (rc != DMPQ_OK) return rc;
    } else {
        const long long nvec = (long long)n * k / 8;
        int grid = num_sms() * 4;
        if ((long long)grid * 256 > nvec) grid = (int)((nvec + 255) / 256);
        amax_bf16_kernel<<<grid, 256, 0, st>>>(W, nvec, out->fp4_g);
        rc = check_launch("dmpq_pack_weights(amax)");
        if (rc != DMPQ_OK) return rc;
    }
    rc = dmpq_global_scale(out->fp4_g, 2688.0f, out->fp4_g, 1, s);
    if (rc != DMPQ_OK) return rc;
    rc = dmpq_quantize_act(W, n, k, k, had ? &had_opts : nullptr, nullptr, &a, nullptr, s);
    if (rc != DMPQ_OK) return rc;
    pack_int8_from_fp4_kernel<<<n, 256, 0, st>>>(out->fp4_codes, out->fp4_sf, out->fp4_g, n, k, ((k / 16) + 3) / 4,
                                                 out->i8_codes, out->i8_scale, out->i8_rcp);
    rc = check_launch("dmpq_pack_weights(int8)");
    if (rc != DMPQ_OK || !had) return rc;
    // R14: the packed forms above are those of U = W . blockdiag(H_128); the rotated weights are
    // W~ = 2^-7 U. Scaling by a power of two commutes with every rounding of the pack (E4M3/E2M1
    // codes are unchanged), so only g_w and the INT8 row scales take the factor (exactly).
    scale_pow2_kernel<<<(n + 1 + 255) / 256, 256, 0, st>>>(out->fp4_g, out->i8_scale, out->i8_rcp, n, 0.0078125f);
    return check_launch("dmpq_pack_weights(hadamard scale)");
}
