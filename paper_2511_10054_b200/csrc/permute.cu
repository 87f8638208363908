// K3 permute (warp-scan histogram, stable), row gather into the GEMM's
// operand layout, and K5 combine + layer_update epilogue.
// Reference semantics: model._plan_arrays / forward_batch / layer_update
// (model.py:294-347).
#include <cuda_bf16.h>

#include <algorithm>

#include "combine.cuh"
#include "common.cuh"

namespace bm {
namespace {

constexpr int kPermThreads = 1024;
constexpr int kPermMaxE = 256;

__global__ void __launch_bounds__(kPermThreads) permute_kernel(const int32_t *__restrict__ executed,
                                                               const uint8_t *__restrict__ kind, int nslots, int k,
                                                               int E, int align, int32_t *expert_count,
                                                               int32_t *expert_offset, int32_t *row_token,
                                                               int32_t *slot_row) {
    __shared__ int cnt[kPermMaxE];
    __shared__ int off[kPermMaxE + 1];
    __shared__ int base[kPermMaxE];
    __shared__ int warp_cnt[kPermThreads / 32][kPermMaxE];
    const int tid = threadIdx.x, warp = tid >> 5;
    const unsigned lane = lane_id();
    for (int e = tid; e < E; e += blockDim.x) {
        cnt[e] = 0;
        base[e] = 0;
    }
    __syncthreads();
    // pass 1: histogram of executed experts (dropped slots excluded)
    for (int i = tid; i < nslots; i += blockDim.x)
        if (kind[i] != BM_KIND_DROPPED) atomicAdd(&cnt[executed[i]], 1);
    __syncthreads();
    if (warp == 0) {  // segment offsets: one warp scans the padded counts (8 experts per lane)
        constexpr int kPer = kPermMaxE / 32;
        int v[kPer], sum = 0;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const int e = (int)lane * kPer + j;
            v[j] = e < E ? (cnt[e] + align - 1) / align * align : 0;
            sum += v[j];
        }
        int incl = sum;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
            const int y = __shfl_up_sync(0xffffffffu, incl, o);
            if (lane >= (unsigned)o) incl += y;
        }
        int run = incl - sum;
#pragma unroll
        for (int j = 0; j < kPer; ++j) {
            const int e = (int)lane * kPer + j;
            if (e < E) off[e] = run;
            run += v[j];
        }
        if (lane == 31) off[E] = incl;
    }
    __syncthreads();
    for (int e = tid; e < E; e += blockDim.x) expert_count[e] = cnt[e];
    for (int e = tid; e <= E; e += blockDim.x) expert_offset[e] = off[e];
    // padding rows (fewer than `align` per expert)
    for (int e = tid; e < E; e += blockDim.x)
        for (int r = off[e] + cnt[e]; r < off[e + 1]; ++r) row_token[r] = -1;
    // pass 2: stable rank of each slot inside its expert segment, chunk by chunk
    const int nw = blockDim.x >> 5;
    for (int c0 = 0; c0 < nslots; c0 += blockDim.x) {
        for (int i = tid; i < nw * E; i += blockDim.x) (&warp_cnt[0][0])[(i / E) * kPermMaxE + (i % E)] = 0;
        __syncthreads();
        const int i = c0 + tid;
        int e = -1;
        if (i < nslots && kind[i] != BM_KIND_DROPPED) e = executed[i];
        const unsigned peers = __match_any_sync(0xffffffffu, e);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        if (e >= 0 && rank == 0) warp_cnt[warp][e] = __popc(peers);
        __syncthreads();
        // exclusive prefix over warps, per expert
        for (int x = tid; x < E; x += blockDim.x) {
            int run = 0;
            for (int w = 0; w < nw; ++w) {
                int v = warp_cnt[w][x];
                warp_cnt[w][x] = run;
                run += v;
            }
            cnt[x] = run;  // reuse cnt as this chunk's total
        }
        __syncthreads();
        if (i < nslots) {
            if (e >= 0) {
                const int row = off[e] + base[e] + warp_cnt[warp][e] + rank;
                row_token[row] = i / k;
                slot_row[i] = row;
            } else {
                slot_row[i] = -1;
            }
        }
        __syncthreads();
        for (int x = tid; x < E; x += blockDim.x) base[x] += cnt[x];
        __syncthreads();
    }
}

// Multi-CTA permute for prefill-size plans (B*k > one chunk): the single
// CTA above walks 1024-slot chunks one after another (16 at a 2048-token
// top-8 chunk, ~78 us). Here chunk c is CTA c: (1) every CTA histograms its
// chunk, (2) one CTA turns the chunk histograms into expert offsets and each
// chunk's per-expert base (exclusive prefix over chunks = the running base
// of the single CTA), (3) every CTA ranks its chunk exactly like pass 2
// above. Same rows for every slot, bit for bit.
constexpr int kChunk = kPermThreads;

__global__ void __launch_bounds__(kPermThreads) permute_hist_kernel(const int32_t *__restrict__ executed,
                                                                    const uint8_t *__restrict__ kind, int nslots,
                                                                    int E, int32_t *__restrict__ chunk_hist) {
    __shared__ int cnt[kPermMaxE];
    for (int e = threadIdx.x; e < E; e += blockDim.x) cnt[e] = 0;
    __syncthreads();
    const int i = blockIdx.x * kChunk + threadIdx.x;
    if (i < nslots && kind[i] != BM_KIND_DROPPED) atomicAdd(&cnt[executed[i]], 1);
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) chunk_hist[(size_t)blockIdx.x * E + e] = cnt[e];
}

__global__ void __launch_bounds__(kPermThreads) permute_scan_kernel(int32_t *__restrict__ chunk_hist, int nchunks,
                                                                    int E, int align, int32_t *expert_count,
                                                                    int32_t *expert_offset, int32_t *row_token) {
    __shared__ int tot[kPermMaxE];
    __shared__ int off[kPermMaxE + 1];
    for (int e = threadIdx.x; e < E; e += blockDim.x) {  // per expert: exclusive prefix over chunks, in place
        int run = 0;
        for (int c = 0; c < nchunks; ++c) {
            const int v = chunk_hist[(size_t)c * E + e];
            chunk_hist[(size_t)c * E + e] = run;
            run += v;
        }
        tot[e] = run;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int run = 0;
        for (int e = 0; e < E; ++e) {
            off[e] = run;
            run += (tot[e] + align - 1) / align * align;
        }
        off[E] = run;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += blockDim.x) expert_count[e] = tot[e];
    for (int e = threadIdx.x; e <= E; e += blockDim.x) expert_offset[e] = off[e];
    for (int e = 0; e < E; ++e)  // padding rows
        for (int r = off[e] + tot[e] + threadIdx.x; r < off[e + 1]; r += blockDim.x) row_token[r] = -1;
}

__global__ void __launch_bounds__(kPermThreads) permute_scatter_kernel(const int32_t *__restrict__ executed,
                                                                       const uint8_t *__restrict__ kind, int nslots,
                                                                       int k, int E,
                                                                       const int32_t *__restrict__ chunk_base,
                                                                       const int32_t *__restrict__ expert_offset,
                                                                       int32_t *row_token, int32_t *slot_row) {
    __shared__ int warp_cnt[kPermThreads / 32][kPermMaxE];
    const int tid = threadIdx.x, warp = tid >> 5, nw = blockDim.x >> 5;
    const unsigned lane = lane_id();
    for (int i = tid; i < nw * E; i += blockDim.x) (&warp_cnt[0][0])[(i / E) * kPermMaxE + (i % E)] = 0;
    __syncthreads();
    const int i = blockIdx.x * kChunk + tid;
    int e = -1;
    if (i < nslots && kind[i] != BM_KIND_DROPPED) e = executed[i];
    const unsigned peers = __match_any_sync(0xffffffffu, e);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (e >= 0 && rank == 0) warp_cnt[warp][e] = __popc(peers);
    __syncthreads();
    for (int x = tid; x < E; x += blockDim.x) {
        int run = 0;
        for (int w = 0; w < nw; ++w) {
            const int v = warp_cnt[w][x];
            warp_cnt[w][x] = run;
            run += v;
        }
    }
    __syncthreads();
    if (i < nslots) {
        if (e >= 0) {
            const int row = expert_offset[e] + chunk_base[(size_t)blockIdx.x * E + e] + warp_cnt[warp][e] + rank;
            row_token[row] = i / k;
            slot_row[i] = row;
        } else {
            slot_row[i] = -1;
        }
    }
}

// layout 0: fp32 row-major [r_max][d]
__global__ void gather_f32_kernel(const float *__restrict__ x, int d, const int32_t *__restrict__ row_token,
                                  const int32_t *__restrict__ expert_offset, int E, float *__restrict__ out) {
    const int rows = expert_offset[E];
    const int r = blockIdx.x;
    if (r >= rows) return;
    const int t = row_token[r];
    float *dst = out + (size_t)r * d;
    if ((d & 3) == 0) {
        float4 *d4 = reinterpret_cast<float4 *>(dst);
        const float4 *s4 = reinterpret_cast<const float4 *>(x + (size_t)(t < 0 ? 0 : t) * d);
        for (int i = threadIdx.x; i < d / 4; i += blockDim.x) d4[i] = t < 0 ? make_float4(0.f, 0.f, 0.f, 0.f) : s4[i];
    } else {
        for (int i = threadIdx.x; i < d; i += blockDim.x) dst[i] = t < 0 ? 0.f : x[(size_t)t * d + i];
    }
}

// layout 1: bf16 SW128 K-major planes [d/64][r_max][64], 16-byte chunk j of
// row r at chunk position j ^ (r & 7) — the smem image of a 128B-swizzled
// UMMA operand, so the GEMM moves it with a plain bulk copy.
__global__ void gather_sw128_kernel(const float *__restrict__ x, int d, const int32_t *__restrict__ row_token,
                                    const int32_t *__restrict__ expert_offset, int E, int r_max,
                                    uint4 *__restrict__ out) {
    const int rows = expert_offset[E];
    const int chunks_per_row = d / 8;
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (idx >= (long long)rows * chunks_per_row) return;
    const int r = (int)(idx / chunks_per_row);
    const int c = (int)(idx % chunks_per_row);  // 8-column chunk index along d
    const int plane = c >> 3, j = c & 7;
    const int t = row_token[r];
    uint4 v = make_uint4(0, 0, 0, 0);
    if (t >= 0) {
        const float4 *s = reinterpret_cast<const float4 *>(x + (size_t)t * d + (size_t)c * 8);
        float4 a = s[0], b = s[1];
        __nv_bfloat162 p0 = __floats2bfloat162_rn(a.x, a.y), p1 = __floats2bfloat162_rn(a.z, a.w);
        __nv_bfloat162 p2 = __floats2bfloat162_rn(b.x, b.y), p3 = __floats2bfloat162_rn(b.z, b.w);
        v.x = *reinterpret_cast<uint32_t *>(&p0);
        v.y = *reinterpret_cast<uint32_t *>(&p1);
        v.z = *reinterpret_cast<uint32_t *>(&p2);
        v.w = *reinterpret_cast<uint32_t *>(&p3);
    }
    out[((size_t)plane * r_max + r) * 8 + (j ^ (r & 7))] = v;
}

template <typename T, int VEC>
__global__ void __launch_bounds__(kCombineThreads) combine_kernel(const T *__restrict__ y_perm,
                                                                  const int32_t *__restrict__ slot_row,
                                                                  const T *__restrict__ probs,
                                                                  const uint8_t *__restrict__ kind, int k, int d,
                                                                  const T *h_in, T scale,
                                                                  T *out) {  // out may alias h_in
    extern __shared__ __align__(16) uint8_t hraw[];
    __shared__ CombineShared<T> sh;
    combine_token<T, VEC, false>(blockIdx.x, y_perm, slot_row, probs, kind, k, d, h_in, scale, out,
                                 reinterpret_cast<T *>(hraw), sh);
}

template <typename T, int VEC>
int launch_combine(const T *y_perm, const int32_t *slot_row, const T *probs, const uint8_t *kind, int64_t B,
                   int64_t k, int64_t d, const T *h_in, T scale, T *out, cudaStream_t s) {
    const size_t smem = h_in ? (size_t)d * sizeof(T) : 0;
    BM_REQUIRE(smem <= 200 * 1024, BM_EINVAL, "bm_combine: d too large");
    if (smem > 48 * 1024)
        BM_CUDA_TRY(cudaFuncSetAttribute(combine_kernel<T, VEC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
    combine_kernel<T, VEC><<<(unsigned)B, kCombineThreads, smem, s>>>(y_perm, slot_row, probs, kind, (int)k, (int)d,
                                                                      h_in, scale, out);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

// layout 0 in f64: row-major [r_max][d] (the reference-precision forward)
__global__ void gather_f64_kernel(const double *__restrict__ x, int d, const int32_t *__restrict__ row_token,
                                  const int32_t *__restrict__ expert_offset, int E, double *__restrict__ out) {
    const int rows = expert_offset[E];
    const int r = blockIdx.x;
    if (r >= rows) return;
    const int t = row_token[r];
    for (int i = threadIdx.x; i < d; i += blockDim.x) out[(size_t)r * d + i] = t < 0 ? 0.0 : x[(size_t)t * d + i];
}

__global__ void split_counts_kernel(const int32_t *__restrict__ count, const int32_t *__restrict__ mask, int E,
                                    int32_t *ca, int32_t *cb) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= E) return;
    const int c = count[e];
    ca[e] = mask[e] ? 0 : c;
    cb[e] = mask[e] ? c : 0;
}

__global__ void append_shared_kernel(const int32_t *__restrict__ ex, const uint8_t *__restrict__ kd,
                                     const float *__restrict__ pr, int B, int k, int E, int S, int32_t *ex2,
                                     uint8_t *kd2, float *pr2) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B) return;
    const int kt = k + S;
    for (int s = 0; s < k; ++s) {
        ex2[b * kt + s] = ex[b * k + s];
        kd2[b * kt + s] = kd[b * k + s];
        pr2[b * kt + s] = pr[b * k + s];
    }
    for (int s = 0; s < S; ++s) {
        ex2[b * kt + k + s] = E + s;
        kd2[b * kt + k + s] = BM_KIND_KEPT;
        pr2[b * kt + k + s] = 1.0f;
    }
}

}  // namespace
}  // namespace bm

using namespace bm;

extern "C" int bm_split_counts(const int32_t *expert_count, const int32_t *mask, int64_t E, int32_t *count_a,
                               int32_t *count_b, bm_stream_t stream) {
    BM_REQUIRE(expert_count && mask && count_a && count_b && E >= 1, BM_EINVAL, "bm_split_counts: bad args");
    split_counts_kernel<<<(unsigned)((E + 255) / 256), 256, 0, as_stream(stream)>>>(expert_count, mask, (int)E, count_a,
                                                                                  count_b);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_append_shared(const int32_t *executed, const uint8_t *kind, const float *probs, int64_t B, int64_t k,
                                int64_t E, int64_t S, int32_t *executed_ext, uint8_t *kind_ext, float *probs_ext,
                                bm_stream_t stream) {
    BM_REQUIRE(executed && kind && probs && executed_ext && kind_ext && probs_ext && B >= 0 && S >= 0, BM_EINVAL,
               "bm_append_shared: bad args");
    if (B == 0) return BM_OK;
    append_shared_kernel<<<(unsigned)((B + 127) / 128), 128, 0, as_stream(stream)>>>(
        executed, kind, probs, (int)B, (int)k, (int)E, (int)S, executed_ext, kind_ext, probs_ext);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int64_t bm_permute_rows_max(int64_t B, int64_t k, int64_t E, int64_t row_align) {
    int64_t n = B * k;
    int64_t segs = n < E ? n : E;
    return n + segs * (row_align - 1);
}

extern "C" int bm_permute_scratch_elems(int64_t B, int64_t k, int64_t E) {
    return (int)(((B * k + kChunk - 1) / kChunk) * E);
}

extern "C" int bm_permute_ws(const int32_t *executed, const uint8_t *kind, int64_t B, int64_t k, int64_t E,
                             int64_t row_align, int32_t *expert_count, int32_t *expert_offset, int32_t *row_token,
                             int32_t *slot_row, int32_t *chunk_scratch, int64_t scratch_elems, bm_stream_t stream) {
    BM_REQUIRE(B >= 0 && k >= 1 && E >= 1 && E <= kPermMaxE && row_align >= 1 && row_align <= 256, BM_EINVAL,
               "bm_permute: bad shape");
    BM_REQUIRE(expert_count && expert_offset && (B == 0 || (executed && kind && row_token && slot_row)), BM_EINVAL,
               "bm_permute: null pointer");
    const int64_t nslots = B * k, nchunks = (nslots + kChunk - 1) / kChunk;
    static const int multi_env = [] {
        const char *ev = getenv("BMOE_PERMUTE_MULTI");  // A/B switch: 0 = always one CTA
        return ev ? atoi(ev) : -1;
    }();
    const bool multi = chunk_scratch && scratch_elems >= nchunks * E && nchunks >= 2 &&
                       (multi_env < 0 ? nchunks >= 4 : multi_env != 0);
    cudaStream_t st = as_stream(stream);
    if (multi) {  // per-chunk histograms -> chunk bases (in place) + offsets -> scatter
        permute_hist_kernel<<<(unsigned)nchunks, kPermThreads, 0, st>>>(executed, kind, (int)nslots, (int)E,
                                                                       chunk_scratch);
        BM_LAUNCH_CHECK();
        permute_scan_kernel<<<1, kPermThreads, 0, st>>>(chunk_scratch, (int)nchunks, (int)E, (int)row_align,
                                                         expert_count, expert_offset, row_token);
        BM_LAUNCH_CHECK();
        permute_scatter_kernel<<<(unsigned)nchunks, kPermThreads, 0, st>>>(executed, kind, (int)nslots, (int)k,
                                                                           (int)E, chunk_scratch, expert_offset,
                                                                           row_token, slot_row);
        BM_LAUNCH_CHECK();
        return BM_OK;
    }
    // one CTA, as many warps as the slots need (a decode plan of 128 slots: 4 warps, so the
    // per-chunk loops over warps and the barriers stay short); ranks do not depend on it
    const int threads = (int)std::min<int64_t>(kPermThreads, std::max<int64_t>(64, (nslots + 31) / 32 * 32));
    permute_kernel<<<1, threads, 0, st>>>(executed, kind, (int)nslots, (int)k, (int)E, (int)row_align,
                                          expert_count, expert_offset, row_token, slot_row);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_permute(const int32_t *executed, const uint8_t *kind, int64_t B, int64_t k, int64_t E,
                          int64_t row_align, int32_t *expert_count, int32_t *expert_offset, int32_t *row_token,
                          int32_t *slot_row, bm_stream_t stream) {
    return bm_permute_ws(executed, kind, B, k, E, row_align, expert_count, expert_offset, row_token, slot_row,
                         nullptr, 0, stream);
}

extern "C" int bm_gather_rows(const float *x, int64_t B, int64_t d, const int32_t *row_token,
                              const int32_t *expert_offset, int64_t E, int64_t r_max, int32_t layout, void *x_perm,
                              bm_stream_t stream) {
    BM_REQUIRE(d >= 1 && r_max >= 0 && B >= 0, BM_EINVAL, "bm_gather_rows: bad args");
    if (r_max == 0 || B == 0) return BM_OK;
    BM_REQUIRE(x && row_token && expert_offset && x_perm, BM_EINVAL, "bm_gather_rows: null pointer");
    if (layout == 0) {
        gather_f32_kernel<<<(unsigned)r_max, 256, 0, as_stream(stream)>>>(x, (int)d, row_token, expert_offset,
                                                                          (int)E, static_cast<float *>(x_perm));
    } else if (layout == 1) {
        BM_REQUIRE(d % 64 == 0, BM_EINVAL, "SW128 layout needs d %% 64 == 0");
        long long n = r_max * (d / 8);
        gather_sw128_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(
            x, (int)d, row_token, expert_offset, (int)E, (int)r_max, static_cast<uint4 *>(x_perm));
    } else {
        BM_REQUIRE(false, BM_EINVAL, "bm_gather_rows: unknown layout %d", layout);
    }
    BM_LAUNCH_CHECK();
    return BM_OK;
}

template <typename T>
static int combine_any(const T *y_perm, const int32_t *slot_row, const T *probs, const uint8_t *kind, int64_t B,
                       int64_t k, int64_t d, const T *h_in, T residual_scale, T *out, bm_stream_t stream) {
    BM_REQUIRE(B >= 0 && k >= 1 && d >= 1, BM_EINVAL, "bm_combine: bad args");
    BM_REQUIRE(k <= kCombineMaxSlots, BM_EINVAL, "bm_combine: k=%lld slots exceeds %d", (long long)k,
               kCombineMaxSlots);
    if (B == 0) return BM_OK;
    BM_REQUIRE(y_perm && slot_row && probs && kind && out, BM_EINVAL, "bm_combine: null pointer");
    constexpr int VEC = 16 / sizeof(T);
    const bool vec = d % VEC == 0 && ((reinterpret_cast<uintptr_t>(y_perm) | reinterpret_cast<uintptr_t>(out) |
                                       reinterpret_cast<uintptr_t>(h_in)) & 15) == 0;
    cudaStream_t s = as_stream(stream);
    return vec ? launch_combine<T, VEC>(y_perm, slot_row, probs, kind, B, k, d, h_in, residual_scale, out, s)
               : launch_combine<T, 1>(y_perm, slot_row, probs, kind, B, k, d, h_in, residual_scale, out, s);
}

extern "C" int bm_combine(const float *y_perm, const int32_t *slot_row, const float *probs, const uint8_t *kind,
                          int64_t B, int64_t k, int64_t d, const float *h_in, float residual_scale, float *out,
                          bm_stream_t stream) {
    return combine_any<float>(y_perm, slot_row, probs, kind, B, k, d, h_in, residual_scale, out, stream);
}

extern "C" int bm_combine_f64(const double *y_perm, const int32_t *slot_row, const double *probs,
                              const uint8_t *kind, int64_t B, int64_t k, int64_t d, const double *h_in,
                              double residual_scale, double *out, bm_stream_t stream) {
    return combine_any<double>(y_perm, slot_row, probs, kind, B, k, d, h_in, residual_scale, out, stream);
}

extern "C" int bm_gather_rows_f64(const double *x, int64_t B, int64_t d, const int32_t *row_token,
                                  const int32_t *expert_offset, int64_t E, int64_t r_max, double *x_perm,
                                  bm_stream_t stream) {
    BM_REQUIRE(d >= 1 && r_max >= 0 && B >= 0, BM_EINVAL, "bm_gather_rows_f64: bad args");
    if (r_max == 0 || B == 0) return BM_OK;
    BM_REQUIRE(x && row_token && expert_offset && x_perm, BM_EINVAL, "bm_gather_rows_f64: null pointer");
    gather_f64_kernel<<<(unsigned)r_max, 256, 0, as_stream(stream)>>>(x, (int)d, row_token, expert_offset, (int)E,
                                                                      x_perm);
    BM_LAUNCH_CHECK();
    return BM_OK;
}
