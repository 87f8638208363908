// K2 — buddy remap (Alg. 1): one warp per token, the residency snapshot as
// a bitmap in shared memory, the token's assigned set as a 256-bit register
// mask, and one warp ballot per missing slot over the candidate list.
// Bit-exact with substitution.substitute_token (reference
// substitution.py:146-190) including the Psi ordering (:98-143) and the
// batch distribution gate (gating.py:126-165).
#include <math.h>

#include "common.cuh"
#include "numpy_order.cuh"

namespace bm {
namespace {

constexpr int kRemapThreads = 256;
constexpr int kWarps = kRemapThreads / 32;
constexpr int kMaxE = 256;
constexpr int kMaxH = 256;
constexpr int kMaxK = 32;
constexpr double kZClamp = 3.0;  // substitution.py:33

// The engine's packed plan in mapped pinned host memory: the kernel writes its
// plan (and the router's top-k and token gate it read) straight to the host,
// so the engine's layer-step has no readback copy (null fields: none).
struct HostPlan {
    int32_t *topk, *executed;
    uint8_t *kind, *allowed, *batch_ok;
};

struct RemapArgs {
    const int32_t *topk;
    const uint8_t *token_allowed;
    const void *logits;
    int logits_f64;
    int B, k, E;
    const uint32_t *bitmap;
    const int32_t *ids;
    const double *w;
    const int32_t *len;
    int stride, H;
    long long rho;
    int fallback, method;
    double beta, eta, kappa;
    int use_local_logit;
    const int32_t *partition_of;
    double hop;
    int32_t *executed;
    uint8_t *kind;
    int32_t *used;
    double *delta_out;
    uint8_t *batch_allowed_out;
    const double *beta_dev;  // when set, beta is read from device memory (the engine's adaptive beta)
    HostPlan hp;             // the engine's mapped host plan (null: none)
};

__device__ __forceinline__ bool bit_of(const uint32_t *m, int e) { return (m[e >> 5] >> (e & 31)) & 1u; }

template <bool kPsi>
__global__ void __launch_bounds__(kRemapThreads) remap_kernel(RemapArgs a) {
    __shared__ uint32_t res[kMaxE / 32];
    __shared__ int miss_warp[kWarps];
    __shared__ double zrow[kPsi ? kWarps : 1][kPsi ? kMaxE : 1];
    __shared__ double score[kPsi ? kWarps : 1][kPsi ? kMaxH : 1];
    __shared__ int cand_sorted[kPsi ? kWarps : 1][kPsi ? kMaxH : 1];

    const int nwords = (a.E + 31) >> 5;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) res[i] = a.bitmap[i];
    __syncthreads();

    // distribution gate: delta over the batch's requested slots, duplicates
    // counted (gating.py:138-145). Every CTA recomputes it: deterministic,
    // and B*k is small at decode.
    const long long nreq = (long long)a.B * a.k;
    int miss = 0;
    for (long long i = threadIdx.x; i < nreq; i += blockDim.x) miss += bit_of(res, a.topk[i]) ? 0 : 1;
    for (int off = 16; off > 0; off >>= 1) miss += __shfl_xor_sync(0xffffffffu, miss, off);
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    if (lane == 0) miss_warp[warp] = miss;
    __syncthreads();
    int total_miss = 0;
    for (int w = 0; w < kWarps; ++w) total_miss += miss_warp[w];
    const double delta = nreq > 0 ? ddiv((double)total_miss, (double)nreq) : 0.0;
    const double beta = a.beta_dev ? *a.beta_dev : a.beta;
    const bool batch_ok = !(delta >= beta);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
        if (a.delta_out) *a.delta_out = delta;
        if (a.batch_allowed_out) *a.batch_allowed_out = batch_ok ? 1 : 0;
        if (a.hp.batch_ok) *a.hp.batch_ok = batch_ok ? 1 : 0;
    }

    const int b = blockIdx.x * kWarps + warp;
    if (b >= a.B) return;
    const int k = a.k;
    const int my_e = (lane < (unsigned)k) ? a.topk[(size_t)b * k + lane] : -1;
    int32_t *ex = a.executed + (size_t)b * k;
    uint8_t *kd = a.kind + (size_t)b * k;

    if (a.hp.topk) {  // the router's part of the host plan
        if (lane < (unsigned)k) a.hp.topk[(size_t)b * k + lane] = my_e;
        if (lane == 0) a.hp.allowed[b] = a.token_allowed ? a.token_allowed[b] : 1;
    }
    if (a.method != BM_METHOD_BUDDY) {
        if (lane < (unsigned)k) {
            const uint8_t kk = (a.method == BM_METHOD_IDENTITY || bit_of(res, my_e)) ? BM_KIND_KEPT : BM_KIND_ONDEMAND;
            ex[lane] = my_e;
            kd[lane] = kk;
            if (a.hp.executed) {
                a.hp.executed[(size_t)b * k + lane] = my_e;
                a.hp.kind[(size_t)b * k + lane] = kk;
            }
        }
        if (lane == 0 && a.used) a.used[b] = 0;
        return;
    }

    // assigned set U_t = all k originals (SPEC: includes not-yet-processed
    // missing slots, substitution.py:160), kept as a warp-uniform bitmask.
    uint32_t assigned[kMaxE / 32];
#pragma unroll
    for (int w = 0; w < kMaxE / 32; ++w) {
        uint32_t bit = (my_e >= 0 && (my_e >> 5) == w) ? (1u << (my_e & 31)) : 0u;
        assigned[w] = __reduce_or_sync(0xffffffffu, bit);
    }

    const bool allowed = a.token_allowed[b] && batch_ok;
    const int fb_kind = a.fallback == BM_FALLBACK_PREFETCH ? BM_KIND_ONDEMAND : BM_KIND_DROPPED;
    const long long budget = a.rho < 0 ? (long long)1 << 62 : a.rho;

    double zmean = 0.0, zsd = 0.0;
    if (kPsi && allowed && a.use_local_logit && a.eta != 0.0) {
        // _zscore (substitution.py:98-104): numpy mean/std of the logit row,
        // pairwise summation order, f64.
        for (int e = lane; e < a.E; e += 32)
            zrow[warp][e] = a.logits_f64 ? static_cast<const double *>(a.logits)[(size_t)b * a.E + e]
                                         : (double)static_cast<const float *>(a.logits)[(size_t)b * a.E + e];
        __syncwarp();
        if (lane == 0) {
            zmean = ddiv(pairwise_sum(zrow[warp], a.E), (double)a.E);
            zsd = sqrt(ddiv(pairwise_sum_sq_dev(zrow[warp], a.E, zmean), (double)a.E));
        }
        zmean = __shfl_sync(0xffffffffu, zmean, 0);
        zsd = __shfl_sync(0xffffffffu, zsd, 0);
    }

    long long used = 0;
    int out_e = my_e, out_kind = BM_KIND_KEPT;
    for (int s = 0; s < k; ++s) {
        const int orig = __shfl_sync(0xffffffffu, my_e, s);
        int picked = -1;
        if (!bit_of(res, orig)) {
            if (allowed && used < budget) {
                const int n = min(a.len[orig], a.H);
                const int32_t *cids = a.ids + (size_t)orig * a.stride;
                if (kPsi && (a.eta != 0.0 || a.kappa != 0.0)) {
                    // psi_score (substitution.py:107-130): q*(1+eta*z)*(1-kappa*hops);
                    // the diversity factor cannot reorder viable candidates (they
                    // are outside the assigned set) and is omitted.
                    for (int r = lane; r < n; r += 32) {
                        int j = cids[r];
                        double q = a.w[(size_t)orig * a.stride + r];
                        double zh = 0.0;
                        if (a.use_local_logit && a.eta != 0.0 && zsd > 0.0) {
                            double v = ddiv(dsub(zrow[warp][j], zmean), zsd);
                            zh = fmin(kZClamp, fmax(-kZClamp, v));
                        }
                        double hops = 0.0;
                        if (a.partition_of && a.partition_of[orig] != a.partition_of[j]) hops = a.hop;
                        score[warp][r] = dmul(dmul(q, dadd(1.0, dmul(a.eta, zh))), dsub(1.0, dmul(a.kappa, hops)));
                    }
                    __syncwarp();
                    // stable argsort(-score): rank = #(better score) + #(equal, earlier)
                    for (int r = lane; r < n; r += 32) {
                        double sr = score[warp][r];
                        int rank = 0;
                        for (int t = 0; t < n; ++t) {
                            double st = score[warp][t];
                            rank += (st > sr || (st == sr && t < r)) ? 1 : 0;
                        }
                        cand_sorted[warp][rank] = cids[r];
                    }
                    __syncwarp();
                    for (int base = 0; base < n && picked < 0; base += 32) {
                        int r = base + lane;
                        bool ok = false;
                        if (r < n) {
                            int j = cand_sorted[warp][r];
                            ok = bit_of(res, j) && !((assigned[j >> 5] >> (j & 31)) & 1u);
                        }
                        unsigned m = __ballot_sync(0xffffffffu, ok);
                        if (m) picked = cand_sorted[warp][base + __ffs(m) - 1];
                    }
                    __syncwarp();
                } else {
                    for (int base = 0; base < n && picked < 0; base += 32) {
                        int r = base + lane;
                        int j = r < n ? cids[r] : -1;
                        bool ok = j >= 0 && bit_of(res, j) && !((assigned[j >> 5] >> (j & 31)) & 1u);
                        unsigned m = __ballot_sync(0xffffffffu, ok);
                        if (m) picked = __shfl_sync(0xffffffffu, j, __ffs(m) - 1);
                    }
                }
            }
            if (picked >= 0) {
                assigned[picked >> 5] |= 1u << (picked & 31);
                ++used;
            }
            if (lane == (unsigned)s) {
                out_e = picked >= 0 ? picked : orig;
                out_kind = picked >= 0 ? BM_KIND_SUBSTITUTED : fb_kind;
            }
        }
    }
    if (lane < (unsigned)k) {
        ex[lane] = out_e;
        kd[lane] = (uint8_t)out_kind;
        if (a.hp.executed) {
            a.hp.executed[(size_t)b * k + lane] = out_e;
            a.hp.kind[(size_t)b * k + lane] = (uint8_t)out_kind;
        }
    }
    if (lane == 0 && a.used) a.used[b] = (int32_t)used;
}

}  // namespace
}  // namespace bm

namespace bm {
// bm_buddy_remap with an optional device-resident beta (engine.cpp: the
// adaptive BetaController changes beta between CUDA-graph replays).
int buddy_remap_impl(const int32_t *topk, const uint8_t *token_allowed, const void *logits, int32_t logits_f64,
                     int64_t B, int64_t k, int64_t E, const uint32_t *resident_bitmap, const int32_t *tbl_ids,
                     const double *tbl_w, const int32_t *tbl_len, int64_t tbl_stride, int64_t H, int64_t rho,
                     int32_t fallback, int32_t method, double beta, const double *beta_dev, double eta, double kappa,
                     int32_t use_local_logit, const int32_t *partition_of, double hop, int32_t *executed,
                     uint8_t *kind, int32_t *used, double *delta_out, uint8_t *batch_allowed_out,
                     bm_stream_t stream, int32_t *hp_topk, int32_t *hp_executed, uint8_t *hp_kind,
                     uint8_t *hp_allowed, uint8_t *hp_batch_ok) {
    BM_REQUIRE(B >= 0 && k >= 1 && k <= kMaxK && E >= 1 && E <= kMaxE, BM_EINVAL,
               "bm_buddy_remap: bad shape B=%lld k=%lld E=%lld", (long long)B, (long long)k, (long long)E);
    BM_REQUIRE(resident_bitmap && (B == 0 || (topk && executed && kind)), BM_EINVAL, "bm_buddy_remap: null pointer");
    BM_REQUIRE(method >= BM_METHOD_BUDDY && method <= BM_METHOD_IDENTITY, BM_EINVAL, "bad method %d", method);
    const bool psi = eta != 0.0 || kappa != 0.0;
    if (method == BM_METHOD_BUDDY) {
        BM_REQUIRE((B == 0 || token_allowed) && tbl_ids && tbl_len, BM_EINVAL,
                   "bm_buddy_remap: buddy method needs gates and a table");
        BM_REQUIRE(H >= 1 && H <= kMaxH && tbl_stride >= 1, BM_ECONFIG, "search rank H=%lld out of range", (long long)H);
        BM_REQUIRE(fallback == BM_FALLBACK_PREFETCH || fallback == BM_FALLBACK_DROP, BM_ECONFIG, "bad fallback");
        BM_REQUIRE(eta >= 0.0 && kappa >= 0.0, BM_ECONFIG, "eta and kappa must be nonnegative");
        if (psi) {
            BM_REQUIRE(tbl_w, BM_EINVAL, "Psi ordering needs table weights");
            BM_REQUIRE(!(use_local_logit && eta != 0.0) || logits, BM_EINVAL, "Psi z-scores need logits");
        }
    }
    RemapArgs a{topk, token_allowed, logits, logits_f64, (int)B, (int)k, (int)E, resident_bitmap, tbl_ids,
                tbl_w, tbl_len, (int)tbl_stride, (int)H, (long long)rho, fallback, method, beta, eta, kappa,
                use_local_logit, partition_of, hop, executed, kind, used, delta_out, batch_allowed_out, beta_dev,
                HostPlan{hp_topk, hp_executed, hp_kind, hp_allowed, hp_batch_ok}};
    unsigned grid = (unsigned)((B + kWarps - 1) / kWarps);
    if (grid == 0) grid = 1;  // still publish delta for an empty batch
    if (psi && method == BM_METHOD_BUDDY)
        remap_kernel<true><<<grid, kRemapThreads, 0, as_stream(stream)>>>(a);
    else
        remap_kernel<false><<<grid, kRemapThreads, 0, as_stream(stream)>>>(a);
    BM_LAUNCH_CHECK();
    return BM_OK;
}
}  // namespace bm

using namespace bm;

extern "C" int bm_buddy_remap(const int32_t *topk, const uint8_t *token_allowed, const void *logits,
                              int32_t logits_f64, int64_t B, int64_t k, int64_t E, const uint32_t *resident_bitmap,
                              const int32_t *tbl_ids, const double *tbl_w, const int32_t *tbl_len,
                              int64_t tbl_stride, int64_t H, int64_t rho, int32_t fallback, int32_t method,
                              double beta, double eta, double kappa, int32_t use_local_logit,
                              const int32_t *partition_of, double hop, int32_t *executed, uint8_t *kind,
                              int32_t *used, double *delta_out, uint8_t *batch_allowed_out, bm_stream_t stream) {
    return buddy_remap_impl(topk, token_allowed, logits, logits_f64, B, k, E, resident_bitmap, tbl_ids, tbl_w,
                            tbl_len, tbl_stride, H, rho, fallback, method, beta, nullptr, eta, kappa,
                            use_local_logit, partition_of, hop, executed, kind, used, delta_out, batch_allowed_out,
                            stream, nullptr, nullptr, nullptr, nullptr, nullptr);
}

// ---------------------------------------------------------------- distribution gate alone
namespace bm {
namespace {
__global__ void __launch_bounds__(256) distribution_gate_kernel(const int32_t *__restrict__ req, long long n,
                                                                const uint32_t *__restrict__ bitmap, double beta,
                                                                double *delta_out, uint8_t *allowed_out) {
    __shared__ int part[8];
    int miss = 0;
    for (long long i = threadIdx.x; i < n; i += blockDim.x) {
        const int e = req[i];
        miss += ((bitmap[e >> 5] >> (e & 31)) & 1u) ? 0 : 1;
    }
    for (int off = 16; off > 0; off >>= 1) miss += __shfl_xor_sync(0xffffffffu, miss, off);
    if ((threadIdx.x & 31) == 0) part[threadIdx.x >> 5] = miss;
    __syncthreads();
    if (threadIdx.x == 0) {
        long long tot = 0;
        for (int w = 0; w < 8; ++w) tot += part[w];
        const double d = ddiv((double)tot, (double)n);  // np.mean of bools: exact integer / count
        *delta_out = d;
        if (allowed_out) *allowed_out = !(d >= beta) ? 1 : 0;
    }
}
}  // namespace
}  // namespace bm

// gating.distribution_gate (gating.py:126-145) over n requested ids (duplicates counted).
extern "C" int bm_distribution_gate(const int32_t *requested, int64_t n, const uint32_t *resident_bitmap,
                                    double beta, double *delta_out, uint8_t *allowed_out, bm_stream_t stream) {
    BM_REQUIRE(requested && resident_bitmap && delta_out && n >= 1, BM_EINVAL,
               "requested expert set is empty or null");
    bm::distribution_gate_kernel<<<1, 256, 0, bm::as_stream(stream)>>>(requested, n, resident_bitmap, beta, delta_out,
                                                                       allowed_out);
    BM_LAUNCH_CHECK();
    return BM_OK;
}
