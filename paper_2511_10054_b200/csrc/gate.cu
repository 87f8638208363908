// K1 — fused router: GEMV + bias + warp top-k + renormalised softmax + TAE /
// margin token gate. One token per CTA cluster. Replaces model.route_batch
// (reference model.py:231-280) and gating.tae/margin/token_gate
// (gating.py:71-108).
#include <float.h>
#include <math.h>

#include <stdlib.h>

#include <algorithm>

#include "common.cuh"
#include "ptx.cuh"

namespace bm {
namespace {

constexpr int kGateThreads = 256;
constexpr int kMaxE = 256;
constexpr int kMaxK = 32;
constexpr int kGateUnroll = 16;  // float4 weight loads in flight per lane (d = 2048: a whole row at once)
constexpr int kGateMaxSplit = 16;  // CTAs per token in a cluster (non-portable size above 8)

template <typename T>
struct Cand {
    T v;
    int i;
};

// Reference order: stable argsort of -z => value descending, ties to the
// lower expert id (model.py:261).
template <typename T>
__device__ __forceinline__ bool better(T av, int ai, T bv, int bi) {
    return av > bv || (av == bv && ai < bi);
}

template <typename T>
__device__ void select_and_gate(const T *z, int E, int k, double temperature, double tau, double gamma,
                                int32_t *topk, float *probs, double *probs64, double *tae, double *margin,
                                uint8_t *allowed, int *sel_i, double *sel_z) {
    // called by one full warp; sel_i / sel_z: that warp's kMaxK shared scratch
    const unsigned lane = lane_id();
    unsigned taken = 0;  // bit j: element lane + 32*j already selected
    for (int s = 0; s < k; ++s) {
        T bv = T(0);
        int bi = INT_MAX;
        bool have = false;
        for (int j = 0; lane + 32 * j < (unsigned)E; ++j) {
            if (taken & (1u << j)) continue;
            int e = lane + 32 * j;
            T v = z[e];
            if (!have || better(v, e, bv, bi)) {
                bv = v;
                bi = e;
                have = true;
            }
        }
        if (!have) bi = INT_MAX;
        for (int off = 16; off > 0; off >>= 1) {
            T ov = __shfl_xor_sync(0xffffffffu, bv, off);
            int oi = __shfl_xor_sync(0xffffffffu, bi, off);
            if (oi != INT_MAX && (bi == INT_MAX || better(ov, oi, bv, bi))) {
                bv = ov;
                bi = oi;
            }
        }
        if ((unsigned)(bi & 31) == lane) taken |= 1u << (bi >> 5);
        if (lane == 0) {
            sel_i[s] = bi;
            sel_z[s] = (double)bv;
        }
    }
    __syncwarp();
    // softmax(z/T) restricted to the selection (model.py:259,262-263): the max
    // over all E of z/T is the top-1's, the full denominator cancels in the
    // renormalisation. Lane i evaluates the exp / log of selected value i (the
    // f64 transcendentals in parallel); the sums run in index order on lane 0,
    // exactly as a sequential loop would add them.
    const double zmax = sel_z[0] / temperature;
    const double ei = lane < (unsigned)k ? exp(sel_z[lane] / temperature - zmax) : 0.0;
    double s = 0.0;
    for (int i = 0; i < k; ++i) s += __shfl_sync(0xffffffffu, ei, i);  // every lane: the same order
    const double pi = ei / s;
    const double hi = (lane < (unsigned)k && pi > 0.0) ? pi * log(pi) : 0.0;
    if (lane < (unsigned)k) {
        topk[lane] = sel_i[lane];
        if (probs) probs[lane] = (float)pi;
        if (probs64) probs64[lane] = pi;
    }
    double h = 0.0;
    for (int i = 0; i < k; ++i) h -= __shfl_sync(0xffffffffu, hi, i);
    const double p0 = __shfl_sync(0xffffffffu, pi, 0), p1 = __shfl_sync(0xffffffffu, pi, 1);
    if (lane == 0) {
        double t = 0.0, m = 1.0;
        if (k > 1) {
            t = fmin(1.0, fmax(0.0, h / log((double)k)));
            m = p0 - p1;
        }
        if (tae) *tae = t;
        if (margin) *margin = m;
        bool ok = !(t <= tau);
        if (gamma >= 0.0 && m >= gamma) ok = false;
        if (allowed) *allowed = ok ? 1 : 0;
    }
}

// Two layouts, one per batch regime, with the same per-logit arithmetic (a
// warp's lane-strided float4 dot product, kGateUnroll loads in flight, then
// the xor-shuffle reduction), so the logits are bitwise independent of both:
//  - decode (TOK = 1): one token per cluster of `nsplit` CTAs (grid B *
//    nsplit). CTA r computes the logits of experts [r*epc, (r+1)*epc), one
//    warp per expert, and stores them straight into CTA 0's z through
//    distributed shared memory; after the cluster barrier CTA 0 selects. One
//    CTA per token kept 16 SMs streaming E*d*4 B of router weights each at
//    B = 16 (Qwen3: 55 us per layer).
//  - prefill (TOK = 8): a CTA owns 8 tokens and each weight row it loads
//    serves all 8 (2048 CTAs each re-reading the 1 MB router from L2 took
//    210 us per Qwen3 chunk); warps 0..7 then select one token each.
template <int TOK>
__global__ void __launch_bounds__(kGateThreads) gate_kernel(const float *__restrict__ x, const float *__restrict__ wg,
                                                            const float *__restrict__ bias, int B, int E, int d,
                                                            int k, int nsplit, double temperature, double tau,
                                                            double gamma, float *logits, int32_t *topk, float *probs,
                                                            double *tae, double *margin, uint8_t *allowed) {
    extern __shared__ __align__(16) float smem_x[];  // [TOK][d]
    __shared__ float z[TOK][kMaxE];
    __shared__ int sel_i[TOK][kMaxK];
    __shared__ double sel_z[TOK][kMaxK];
    const int grp = blockIdx.x / nsplit, rank = blockIdx.x % nsplit;
    const int b0 = grp * TOK, nt = min(TOK, B - b0);
    const int epc = (E + nsplit - 1) / nsplit;
    const int e0 = rank * epc, e1 = min(E, e0 + epc);
    const bool vec = (d % 4) == 0;
    // every CTA of the cluster must have started before CTA 0's shared memory
    // is written remotely: arrive now, wait after the row load
    if (nsplit > 1) asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
    for (int t = 0; t < nt; ++t) {
        const float *xr = x + (size_t)(b0 + t) * d;
        float *xs = smem_x + (size_t)t * d;
        if (vec) {
            const float4 *src = reinterpret_cast<const float4 *>(xr);
            float4 *dst = reinterpret_cast<float4 *>(xs);
            for (int i = threadIdx.x; i < d / 4; i += blockDim.x) dst[i] = src[i];
        } else {
            for (int i = threadIdx.x; i < d; i += blockDim.x) xs[i] = xr[i];
        }
    }
    if (nsplit > 1) asm volatile("barrier.cluster.wait.aligned;" ::: "memory");
    __syncthreads();
    const uint32_t z0 = nsplit > 1 ? ptx::mapa(ptx::smem_u32(&z[0][0]), 0) : 0;
    const int warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const unsigned lane = lane_id();
    for (int e = e0 + warp; e < e1; e += nwarps) {
        const float *w = wg + (size_t)e * d;
        float acc[TOK];
#pragma unroll
        for (int t = 0; t < TOK; ++t) acc[t] = 0.f;
        if (vec) {
            const float4 *w4 = reinterpret_cast<const float4 *>(w);
            const int n4 = d / 4;
            for (int i0 = lane; i0 < n4; i0 += 32 * kGateUnroll) {
                float4 a[kGateUnroll];
#pragma unroll
                for (int j = 0; j < kGateUnroll; ++j)
                    a[j] = i0 + 32 * j < n4 ? __ldg(w4 + i0 + 32 * j) : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
                for (int t = 0; t < TOK; ++t) {
                    if (t >= nt) break;
                    const float4 *x4 = reinterpret_cast<const float4 *>(smem_x + (size_t)t * d);
#pragma unroll
                    for (int j = 0; j < kGateUnroll; ++j) {
                        if (i0 + 32 * j >= n4) break;
                        const float4 c = x4[i0 + 32 * j];
                        acc[t] = fmaf(a[j].x, c.x, acc[t]);
                        acc[t] = fmaf(a[j].y, c.y, acc[t]);
                        acc[t] = fmaf(a[j].z, c.z, acc[t]);
                        acc[t] = fmaf(a[j].w, c.w, acc[t]);
                    }
                }
            }
        } else {
            for (int i = lane; i < d; i += 32) {
                const float a = __ldg(w + i);
#pragma unroll
                for (int t = 0; t < TOK; ++t)
                    if (t < nt) acc[t] = fmaf(a, smem_x[(size_t)t * d + i], acc[t]);
            }
        }
#pragma unroll
        for (int t = 0; t < TOK; ++t) {
            float v = acc[t];
            for (int off = 16; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off);
            if (lane == 0 && t < nt) {
                v += bias ? bias[e] : 0.f;
                if (nsplit > 1)
                    asm volatile("st.shared::cluster.f32 [%0], %1;" ::"r"(z0 + 4u * (uint32_t)e), "f"(v) : "memory");
                else
                    z[t][e] = v;
                if (logits) logits[(size_t)(b0 + t) * E + e] = v;
            }
        }
    }
    if (nsplit > 1) {
        ptx::cluster_sync();  // release the remote stores / acquire them in CTA 0
        if (rank != 0) return;
    } else {
        __syncthreads();
    }
    if (warp < nt) {
        const int b = b0 + warp;
        select_and_gate<float>(z[warp], E, k, temperature, tau, gamma, topk + (size_t)b * k,
                               probs ? probs + (size_t)b * k : nullptr, nullptr, tae ? tae + b : nullptr,
                               margin ? margin + b : nullptr, allowed ? allowed + b : nullptr, sel_i[warp],
                               sel_z[warp]);
    }
}

__global__ void __launch_bounds__(32) select_f64_kernel(const double *__restrict__ logits, int E, int k,
                                                        double temperature, double tau, double gamma,
                                                        int32_t *topk, float *probs, double *probs64,
                                                        double *tae, double *margin, uint8_t *allowed) {
    __shared__ double z[kMaxE];
    __shared__ int sel_i[kMaxK];
    __shared__ double sel_z[kMaxK];
    const int b = blockIdx.x;
    for (int e = threadIdx.x; e < E; e += 32) z[e] = logits[(size_t)b * E + e];
    __syncwarp();
    select_and_gate<double>(z, E, k, temperature, tau, gamma, topk + (size_t)b * k,
                            probs ? probs + (size_t)b * k : nullptr, probs64 ? probs64 + (size_t)b * k : nullptr,
                            tae ? tae + b : nullptr, margin ? margin + b : nullptr, allowed ? allowed + b : nullptr,
                            sel_i, sel_z);
}

}  // namespace
}  // namespace bm

using namespace bm;

extern "C" int bm_gate_topk(const float *x, const float *wg, const float *bias, int64_t B, int64_t E, int64_t d,
                            int64_t k, double temperature, double tau, double gamma, float *logits, int32_t *topk,
                            float *probs, double *tae, double *margin, uint8_t *token_allowed, bm_stream_t stream) {
    BM_REQUIRE(B >= 0 && E >= 1 && E <= kMaxE && d >= 1 && k >= 1 && k <= kMaxK && k <= E, BM_EINVAL,
               "bm_gate_topk: bad shape B=%lld E=%lld d=%lld k=%lld", (long long)B, (long long)E, (long long)d,
               (long long)k);
    BM_REQUIRE(temperature > 0.0, BM_EINVAL, "temperature must be > 0");
    if (B == 0) return BM_OK;  // empty batch (its tensors may have null data pointers)
    BM_REQUIRE(x && wg && topk, BM_EINVAL, "bm_gate_topk: null pointer");
    BM_REQUIRE((size_t)d * sizeof(float) <= 200 * 1024, BM_EINVAL, "bm_gate_topk: d=%lld too large", (long long)d);
    // small batches: split each token over a cluster; large ones: 8 tokens per CTA
    const char *wide_env = getenv("BMOE_GATE_WIDE");  // A/B knob: 0 = one token per CTA at any B
    const bool wide = B >= 4 * 148 && (size_t)8 * d * sizeof(float) <= 200 * 1024 && !(wide_env && atoi(wide_env) == 0);
    // small batches: up to 16 CTAs per token (8 experts each), so every warp owns about one expert
    // row and loads it in one round; the per-logit arithmetic does not depend on the split
    int nsplit = wide ? 1 : (B >= 4 * 148 ? 1 : (int)std::min<int64_t>(kGateMaxSplit, (E + 7) / 8));
    if (const char *ev = getenv("BMOE_GATE_SPLIT"))  // A/B knob: forced cluster size (1..16)
        if (atoi(ev) > 0 && !wide) nsplit = std::min(atoi(ev), kGateMaxSplit);
    const int tok = wide ? 8 : 1;
    const size_t smem = (size_t)tok * d * sizeof(float);
    auto kern = wide ? gate_kernel<8> : gate_kernel<1>;
    if (smem > 48 * 1024)
        BM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    if (nsplit > 8) {
        static bool nonportable = false;
        if (!nonportable) {
            BM_CUDA_TRY(cudaFuncSetAttribute(gate_kernel<1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
            nonportable = true;
        }
    }
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3((unsigned)(((B + tok - 1) / tok) * nsplit));
    lc.blockDim = dim3(kGateThreads);
    lc.dynamicSmemBytes = smem;
    lc.stream = as_stream(stream);
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = (unsigned)nsplit;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    BM_CUDA_TRY(cudaLaunchKernelEx(&lc, kern, x, wg, bias, (int)B, (int)E, (int)d, (int)k, nsplit, temperature, tau,
                                   gamma, logits, topk, probs, tae, margin, token_allowed));
    return BM_OK;
}

extern "C" int bm_select_topk_f64(const double *logits, int64_t B, int64_t E, int64_t k, double temperature,
                                  double tau, double gamma, int32_t *topk, float *probs, double *probs64,
                                  double *tae, double *margin, uint8_t *token_allowed, bm_stream_t stream) {
    BM_REQUIRE(B >= 0 && E >= 1 && E <= kMaxE && k >= 1 && k <= kMaxK && k <= E, BM_EINVAL,
               "bm_select_topk_f64: bad shape");
    BM_REQUIRE(temperature > 0.0, BM_EINVAL, "temperature must be > 0");
    if (B == 0) return BM_OK;
    BM_REQUIRE(logits && topk, BM_EINVAL, "bm_select_topk_f64: null pointer");
    select_f64_kernel<<<(unsigned)B, 32, 0, as_stream(stream)>>>(logits, (int)E, (int)k, temperature, tau, gamma,
                                                                topk, probs, probs64, tae, margin, token_allowed);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

// ---------------------------------------------------------------- gates from given probabilities
namespace bm {
namespace {
// TAE / margin / token gate of given renormalised probabilities p[B][k]
// (gating.tae / margin / token_gate, gating.py:71-108): one thread per token.
__global__ void gate_from_probs_kernel(const double *__restrict__ p, int B, int k, double tau, double gamma,
                                       double *tae, double *margin, uint8_t *allowed) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const double *r = p + (size_t)b * k;
    double h = 0.0, top1 = -1.0, top2 = -1.0;
    for (int i = 0; i < k; ++i) {
        const double v = r[i];
        if (v > 0.0) h -= v * log(v);
        if (v > top1) {
            top2 = top1;
            top1 = v;
        } else if (v > top2) {
            top2 = v;
        }
    }
    double t = 0.0, m = 1.0;
    if (k > 1) {
        t = fmin(1.0, fmax(0.0, h / log((double)k)));
        m = top1 - top2;
    }
    if (tae) tae[b] = t;
    if (margin) margin[b] = m;
    bool ok = !(t <= tau);
    if (gamma >= 0.0 && m >= gamma) ok = false;
    if (allowed) allowed[b] = ok ? 1 : 0;
}
}  // namespace
}  // namespace bm

extern "C" int bm_gate_from_probs(const double *probs, int64_t B, int64_t k, double tau, double gamma, double *tae,
                                  double *margin, uint8_t *token_allowed, bm_stream_t stream) {
    BM_REQUIRE(probs && B >= 0 && k >= 1, BM_EINVAL, "bm_gate_from_probs: bad args");
    if (B == 0) return BM_OK;
    bm::gate_from_probs_kernel<<<(unsigned)((B + 127) / 128), 128, 0, bm::as_stream(stream)>>>(
        probs, (int)B, (int)k, tau, gamma, tae, margin, token_allowed);
    BM_LAUNCH_CHECK();
    return BM_OK;
}
