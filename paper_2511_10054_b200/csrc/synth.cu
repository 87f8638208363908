// Synthetic expert weights from a counter-based hash (bench inputs, not the
// hot path). Value i of a matrix is lut[16-bit field of mix64(base + i/4)]:
// one splitmix64 finalisation yields four values, and the 65,536-entry lut
// holds bf16 quantiles of N(0, scale^2) (paper_2511_10054_b200/synth.py
// builds it). Pure integer arithmetic, so the host twin in synth.py (numpy
// uint64) produces the same bits: the CPU reference arm of bench.py gets the
// GPU arm's exact weights without touching the GPU.
#include <algorithm>

#include <cuda_bf16.h>

#include "common.cuh"

namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z += 0x9E3779B97F4A7C15ull;
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

// one thread -> 8 values (two hashes), one 16-byte store
__global__ void synth_kernel(const uint16_t *__restrict__ lut, uint64_t base, int64_t n, uint16_t *__restrict__ out) {
    extern __shared__ __align__(16) uint16_t s_lut[];  // 128 KB: the whole lut
    for (int i = threadIdx.x; i < 65536 / 8; i += blockDim.x)
        reinterpret_cast<uint4 *>(s_lut)[i] = reinterpret_cast<const uint4 *>(lut)[i];
    __syncthreads();
    const int64_t groups8 = (n + 7) / 8;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups8; g += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t a = mix64(base + (uint64_t)(2 * g)), b = mix64(base + (uint64_t)(2 * g + 1));
        uint16_t v[8];
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            v[j] = s_lut[(a >> (16 * j)) & 0xFFFFu];
            v[4 + j] = s_lut[(b >> (16 * j)) & 0xFFFFu];
        }
        const int64_t i0 = 8 * g;
        if (i0 + 8 <= n) {
            uint4 w;
            w.x = v[0] | ((uint32_t)v[1] << 16);
            w.y = v[2] | ((uint32_t)v[3] << 16);
            w.z = v[4] | ((uint32_t)v[5] << 16);
            w.w = v[6] | ((uint32_t)v[7] << 16);
            if ((reinterpret_cast<uintptr_t>(out) & 15) == 0) {
                reinterpret_cast<uint4 *>(out)[g] = w;
                continue;
            }
        }
        for (int j = 0; j < 8 && i0 + j < n; ++j) out[i0 + j] = v[j];
    }
}

// clustered experts (the reference's recipe, model.py:161-171): value =
// bf16_rn(base + spread * delta), base and delta two hashed matrices, the sum
// rounded once in fp32 (no contraction) so the host twin reproduces it
__global__ void synth_mix_kernel(const uint16_t *__restrict__ lut, uint64_t base_key, uint64_t delta_key, float spread,
                                 int64_t n, uint16_t *__restrict__ out) {
    extern __shared__ __align__(16) uint16_t s_lut[];
    for (int i = threadIdx.x; i < 65536 / 8; i += blockDim.x)
        reinterpret_cast<uint4 *>(s_lut)[i] = reinterpret_cast<const uint4 *>(lut)[i];
    __syncthreads();
    const int64_t groups = (n + 3) / 4;
    for (int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; g < groups; g += (int64_t)gridDim.x * blockDim.x) {
        const uint64_t zb = mix64(base_key + (uint64_t)g), zd = mix64(delta_key + (uint64_t)g);
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int64_t i = 4 * g + j;
            if (i >= n) break;
            const float b = __uint_as_float((uint32_t)s_lut[(zb >> (16 * j)) & 0xFFFFu] << 16);
            const float dl = __uint_as_float((uint32_t)s_lut[(zd >> (16 * j)) & 0xFFFFu] << 16);
            const float v = __fadd_rn(b, __fmul_rn(spread, dl));
            const __nv_bfloat16 h = __float2bfloat16_rn(v);
            out[i] = *reinterpret_cast<const uint16_t *>(&h);
        }
    }
}

}  // namespace

extern "C" int bm_synth_mix_bf16(const uint16_t *lut, uint64_t base_key, uint64_t delta_key, float spread, int64_t n,
                                 uint16_t *out, bm_stream_t stream) {
    BM_REQUIRE(n >= 0 && (n == 0 || (lut && out)), BM_EINVAL, "bm_synth_mix_bf16: bad arguments");
    BM_REQUIRE((reinterpret_cast<uintptr_t>(lut) & 15) == 0, BM_EINVAL, "bm_synth_mix_bf16: lut must be 16-byte aligned");
    if (n == 0) return BM_OK;
    static bool attr = false;
    if (!attr) {
        BM_CUDA_TRY(cudaFuncSetAttribute(synth_mix_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 * 2));
        attr = true;
    }
    const int64_t groups = (n + 3) / 4;
    const int blocks = (int)std::min<int64_t>((groups + 511) / 512, (int64_t)bm::sm_count());
    synth_mix_kernel<<<blocks, 512, 65536 * 2, bm::as_stream(stream)>>>(lut, base_key, delta_key, spread, n, out);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_synth_bf16(const uint16_t *lut, uint64_t base, int64_t n, uint16_t *out, bm_stream_t stream) {
    BM_REQUIRE(n >= 0 && (n == 0 || (lut && out)), BM_EINVAL, "bm_synth_bf16: bad arguments");
    BM_REQUIRE((reinterpret_cast<uintptr_t>(lut) & 15) == 0, BM_EINVAL, "bm_synth_bf16: lut must be 16-byte aligned");
    if (n == 0) return BM_OK;
    static bool attr = false;
    if (!attr) {
        BM_CUDA_TRY(cudaFuncSetAttribute(synth_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 65536 * 2));
        attr = true;
    }
    const int64_t groups8 = (n + 7) / 8;
    // one CTA per SM (the lut fills most of its shared memory), grid-stride
    const int blocks = (int)std::min<int64_t>((groups8 + 511) / 512, (int64_t)bm::sm_count());
    synth_kernel<<<blocks, 512, 65536 * 2, bm::as_stream(stream)>>>(lut, base, n, out);
    BM_LAUNCH_CHECK();
    return BM_OK;
}
