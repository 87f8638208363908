// C-ABI of the bf16 grouped expert FFN (K4): bm_expert_ffn_bf16 picks the
// decode kernel (one cooperative launch, ffn_decode.cu) or the prefill GEMMs
// (ffn_prefill.cu) for a call; weight packing into the UMMA-tiled layout,
// the workspace layout and the optional kernel-timing hook live here.
#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"
#include "ffn_common.cuh"

namespace bm {
namespace ffn {

// Pack a row-major bf16 matrix W[M][K] into the UMMA-tiled expert layout:
// 16 KB block (mt, kb, slot) at ((mt*K/64 + kb)*nmat + slot) * 16 KB holds
// rows mt*128.. of columns kb*64.., row r's 16-byte chunk j at
// r*128 + (j ^ (r & 7))*16 — the SW128 K-major smem image, so the GEMM's
// producer moves whole k-steps of every matrix with one contiguous bulk copy.
__global__ void pack_tiles_kernel(const uint4 *__restrict__ src, int M, int K, int nmat, int slot,
                                  uint8_t *__restrict__ dst) {
    const long long idx = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    const long long cpr = K / 8;  // 16-byte chunks per row
    if (idx >= (long long)M * cpr) return;
    const int row = (int)(idx / cpr), c = (int)(idx % cpr);
    const int kb = c >> 3, j = c & 7, mt = row >> 7, r = row & 127;
    const long long off =
        (((long long)mt * (K / 64) + kb) * nmat + slot) * kATileBytes + r * 128 + ((j ^ (r & 7)) << 4);
    *reinterpret_cast<uint4 *>(dst + off) = src[idx];
}

long long max_tiles(long long E, long long M, long long r_max, long long n_tile) {
    const long long segs = std::min(E, std::max(1LL, r_max / 16));
    return (M / kBM) * (segs + r_max / n_tile + 1);
}

// kernel timing (for the bench's roofline), off by default. Each timed call
// is a record of 4 events (before/after GEMM1, before/after GEMM2; a fused
// decode call is one kernel: events 2-3 null) and, for fused calls, an
// on-device span slot [first CTA entry, last CTA exit] (globaltimer ns).
// Eager calls' records are read when the times are asked for. Calls made
// while the stream is being captured record their events as external
// event nodes of the graph: their records go to the capture's group
// (ffn_timing_take_capture), the engine marks the group after each replay
// of its graph (ffn_timing_replayed) and reads it back before the next
// replay (ffn_timing_harvest), so CUDA graphs time their FFN launches too.
struct CallRec {
    cudaEvent_t ev[4] = {nullptr, nullptr, nullptr, nullptr};
    int64_t span_slot = -1;
};
struct Timing {
    bool enabled = false;
    std::vector<CallRec> eager;              // eager calls since timing was enabled, unread
    std::vector<CallRec> capturing;          // calls recorded into the graph being captured
    std::vector<std::vector<CallRec> *> replayed;  // graph groups replayed since the last harvest
    std::vector<float> res_ms;               // 2 per read call (GEMM1 ms, GEMM2 ms)
    std::vector<float> res_span;             // 1 per read call (span ms, 0 without one)
    unsigned long long *span = nullptr;      // slots: eager ones from the bottom, graph ones from the top
    int64_t span_cap = 0, span_n = 0, span_graph_n = 0;
    std::mutex mu;
} g_timing;

bool capturing(cudaStream_t s) {
    cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
    return cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive;
}

CallRec &new_call(cudaStream_t s) {
    auto &v = capturing(s) ? g_timing.capturing : g_timing.eager;
    v.emplace_back();
    return v.back();
}

// a span slot (reset to [UINT64_MAX, 0] on s, as graph nodes when capturing) for the
// fused call `rec` being timed, or null
unsigned long long *next_span(cudaStream_t s, CallRec &rec) {
    if (!g_timing.span) return nullptr;  // allocated when timing is switched on (not during a capture)
    int64_t slot;
    if (capturing(s)) {
        if (g_timing.span_n + g_timing.span_graph_n >= g_timing.span_cap) return nullptr;
        slot = g_timing.span_cap - 1 - g_timing.span_graph_n++;
    } else {
        if (g_timing.span_n + g_timing.span_graph_n >= g_timing.span_cap) return nullptr;
        slot = g_timing.span_n++;
    }
    unsigned long long *p = g_timing.span + 2 * slot;
    cudaMemsetAsync(p, 0xff, sizeof(unsigned long long), s);
    cudaMemsetAsync(p + 1, 0, sizeof(unsigned long long), s);
    rec.span_slot = slot;
    return p;
}

int record_event(cudaStream_t s, CallRec &rec, int i) {
    cudaEvent_t e;
    BM_CUDA_TRY(cudaEventCreate(&e));
    if (capturing(s))
        BM_CUDA_TRY(cudaEventRecordWithFlags(e, s, cudaEventRecordExternal));  // a node the host can read
    else
        BM_CUDA_TRY(cudaEventRecord(e, s));
    rec.ev[i] = e;
    return BM_OK;
}

// read one record's times into the results (its events must have completed)
int read_call(const CallRec &r) {
    float a = 0.f, b = 0.f, sp = 0.f;
    if (cudaEventElapsedTime(&a, r.ev[0], r.ev[1]) != cudaSuccess) return BM_ECUDA;
    if (r.ev[2] && cudaEventElapsedTime(&b, r.ev[2], r.ev[3]) != cudaSuccess) return BM_ECUDA;
    if (r.span_slot >= 0) {
        unsigned long long v[2];
        if (cudaMemcpy(v, g_timing.span + 2 * r.span_slot, sizeof(v), cudaMemcpyDeviceToHost) != cudaSuccess)
            return BM_ECUDA;
        sp = (float)((double)(v[1] - v[0]) * 1e-6);
    }
    g_timing.res_ms.push_back(a);
    g_timing.res_ms.push_back(b);
    g_timing.res_span.push_back(sp);
    return BM_OK;
}

void destroy_call(CallRec &r) {
    for (cudaEvent_t &e : r.ev)
        if (e) {
            cudaEventDestroy(e);
            e = nullptr;
        }
}

}  // namespace ffn
}  // namespace bm

namespace bm {
namespace ffn {
// workspace: [persistent state: grid barrier, launch count, H readiness, split-tile
// arrival counters | fp32 partial slots (2 sets) | bf16 SW128 H planes]; the state must
// start at zero (the kernels keep it consistent from then on).
struct WsLayout {
    long long slot_set_bytes, partial_off, partial_bytes, h_off, h_bytes, ctr_off, bar_off, tile_cap, total;
};
WsLayout ws_layout(long long E, long long d, long long f, long long r_max, long long n_tile) {
    WsLayout w;
    const long long M = std::max(d, f);
    // Persistent state first, at offsets that do not depend on the call's token tile (a
    // workspace serves calls of any n_tile up to the one it was sized for, and the counters
    // must survive between them): [grid barrier u64 | launch count u64 | h_ready[2][kMaxE] |
    // split-tile arrival counters, 2 phases x the tile count of the narrowest tile (16)].
    w.tile_cap = max_tiles(E, M, r_max, 16);
    w.bar_off = 0;
    w.ctr_off = 16 + 2 * kMaxE * 4;
    const long long state = ((w.ctr_off + 2 * w.tile_cap * 4 + 1023) / 1024) * 1024;
    // scratch: two split-tile slot sets (the fused decode kernel's GEMM2 may run while GEMM1
    // split tiles are still being reduced, per-expert H readiness), then the H planes
    const long long slots = max_tiles(E, M, r_max, n_tile) + kMaxGroups * sm_count() + 1;  // + group offsets
    w.slot_set_bytes = ((slots * 2 * n_tile * kBM * 4 + 1023) / 1024) * 1024;
    w.partial_off = state;
    w.partial_bytes = 2 * w.slot_set_bytes;
    w.h_off = w.partial_off + w.partial_bytes;
    w.h_bytes = (((f / 64) * r_max * 128 + 1023) / 1024) * 1024;
    w.total = w.h_off + w.h_bytes;
    return w;
}
}  // namespace ffn
}  // namespace bm

using namespace bm;
using namespace bm::ffn;

// Diagnostics (BMOE_FFN_TRACE=1): per-CTA globaltimer stamps of the fused
// decode kernel's phases (ffn_decode.cu), overwritten by every fused call.
static unsigned long long *g_trace = nullptr;
static int g_trace_ctas = 0;
static unsigned long long *trace_buffer(int G, cudaStream_t s) {
    const char *ev = getenv("BMOE_FFN_TRACE");  // read per call (tests switch it)
    if (!ev || atoi(ev) == 0) return nullptr;
    if (!g_trace) {
        if (cudaMalloc(&g_trace, (size_t)G * kTracePts * sizeof(unsigned long long)) != cudaSuccess) return nullptr;
        g_trace_ctas = G;
    }
    cudaMemsetAsync(g_trace, 0, (size_t)G * kTracePts * sizeof(unsigned long long), s);  // unset stamps read 0
    return g_trace;
}

extern "C" int64_t bm_ffn_trace_read(uint64_t *out_host, int64_t cap) {
    if (!g_trace || !out_host) return 0;
    const int64_t n = std::min<int64_t>(cap, (int64_t)g_trace_ctas * kTracePts);
    if (cudaMemcpy(out_host, g_trace, (size_t)n * sizeof(uint64_t), cudaMemcpyDeviceToHost) != cudaSuccess) return -1;
    return n;
}

extern "C" int64_t bm_expert_ffn_bf16_workspace(int64_t E, int64_t d, int64_t f, int64_t r_max, int64_t n_tile) {
    return ws_layout(E, d, f, r_max, n_tile).total;
}

static int ffn_bf16_impl(const void *x_perm, const int32_t *expert_count, const int32_t *expert_offset, int64_t E,
                         int64_t d, int64_t f, int32_t act, const void *w_arena, int64_t n_bufs,
                         const int32_t *buf_of_expert, int64_t r_max, int64_t n_tile, void *workspace,
                         int64_t workspace_bytes, float *y_perm, bm_stream_t stream, const CombineArgs *cmb);

extern "C" int bm_expert_ffn_bf16(const void *x_perm, const int32_t *expert_count, const int32_t *expert_offset,
                                  int64_t E, int64_t d, int64_t f, int32_t act, const void *w_arena, int64_t n_bufs,
                                  const int32_t *buf_of_expert, int64_t r_max, int64_t n_tile, void *workspace,
                                  int64_t workspace_bytes, float *y_perm, bm_stream_t stream) {
    return ffn_bf16_impl(x_perm, expert_count, expert_offset, E, d, f, act, w_arena, n_bufs, buf_of_expert, r_max,
                         n_tile, workspace, workspace_bytes, y_perm, stream, nullptr);
}

extern "C" int bm_expert_ffn_bf16_combine(const void *x_perm, const int32_t *expert_count,
                                          const int32_t *expert_offset, int64_t E, int64_t d, int64_t f, int32_t act,
                                          const void *w_arena, int64_t n_bufs, const int32_t *buf_of_expert,
                                          int64_t r_max, int64_t n_tile, void *workspace, int64_t workspace_bytes,
                                          float *y_perm, const int32_t *slot_row, const float *probs,
                                          const uint8_t *kind, int64_t B, int64_t k, float *h, float residual_scale,
                                          bm_stream_t stream) {
    BM_REQUIRE(B >= 0 && k >= 1 && k <= 64, BM_EINVAL, "bm_expert_ffn_bf16_combine: bad B/k");
    if (B == 0) return BM_OK;
    BM_REQUIRE(slot_row && probs && kind && h, BM_EINVAL, "bm_expert_ffn_bf16_combine: null pointer");
    const CombineArgs cmb{slot_row, probs, kind, h, residual_scale, (int)B, (int)k};
    return ffn_bf16_impl(x_perm, expert_count, expert_offset, E, d, f, act, w_arena, n_bufs, buf_of_expert, r_max,
                         n_tile, workspace, workspace_bytes, y_perm, stream, &cmb);
}

static int ffn_bf16_impl(const void *x_perm, const int32_t *expert_count, const int32_t *expert_offset, int64_t E,
                         int64_t d, int64_t f, int32_t act, const void *w_arena, int64_t n_bufs,
                         const int32_t *buf_of_expert, int64_t r_max, int64_t n_tile, void *workspace,
                         int64_t workspace_bytes, float *y_perm, bm_stream_t stream, const CombineArgs *cmb) {
    // the combine (if any) after the FFN, as its own launch: bm_combine's exact computation
    auto separate_combine = [&]() -> int {
        if (!cmb) return BM_OK;
        return bm_combine(y_perm, cmb->slot_row, cmb->probs, cmb->kind, cmb->B, cmb->k, d, cmb->h, cmb->scale,
                          cmb->h, stream);
    };
    BM_REQUIRE(r_max >= 0, BM_EINVAL, "r_max must be >= 0");
    if (r_max == 0) return separate_combine();  // no rows (an empty batch): nothing to compute
    BM_REQUIRE(x_perm && expert_count && expert_offset && w_arena && buf_of_expert && workspace && y_perm,
               BM_EINVAL, "bm_expert_ffn_bf16: null pointer");
    BM_REQUIRE(E >= 1 && E <= kMaxE, BM_EINVAL, "E out of range");
    BM_REQUIRE(d % kBM == 0 && f % kBM == 0 && d > 0 && f > 0, BM_EINVAL, "d and f must be multiples of 128");
    BM_REQUIRE(n_tile >= 16 && n_tile <= 256 && n_tile % 16 == 0, BM_EINVAL, "n_tile must be 16..256, multiple of 16");
    BM_REQUIRE(act == BM_ACT_SWIGLU || act == BM_ACT_TANH, BM_EINVAL, "bad activation");
    BM_REQUIRE(r_max % 16 == 0, BM_EINVAL, "r_max must be a multiple of 16");
    BM_REQUIRE(workspace_bytes >= bm_expert_ffn_bf16_workspace(E, d, f, r_max, n_tile), BM_EINVAL,
               "workspace too small");
    if (r_max == 0) return BM_OK;
    cudaStream_t s = as_stream(stream);
    const long long buf_bytes = (act == BM_ACT_SWIGLU ? 3 : 2) * d * f * 2;
    const WsLayout wl = ws_layout(E, d, f, r_max, n_tile);
    float *partials = reinterpret_cast<float *>(static_cast<uint8_t *>(workspace) + wl.partial_off);
    uint8_t *h_planes = static_cast<uint8_t *>(workspace) + wl.h_off;
    int *counters = reinterpret_cast<int *>(static_cast<uint8_t *>(workspace) + wl.ctr_off);
    const int G = sm_count();
    const uint8_t *arena = static_cast<const uint8_t *>(w_arena);
    const int nmat1 = act == BM_ACT_SWIGLU ? 2 : 1;
    // Decode-width tiles (n_tile <= 64) run the single fused launch; for
    // wide prefill tiles the accumulator is single-buffered and the MMA would
    // wait on the longer epilogue, so they use GEMM + fixup kernels.
    int fused = n_tile <= 64 ? 1 : 0;
    if (const char *ev = getenv("BMOE_FUSED")) fused = fused && atoi(ev) != 0;
    // Wide (prefill) tiles are data-parallel and finished in the GEMM
    // epilogue: no partials, no fixup kernels (BMOE_DP=0: stream-K + fixups).
    int dp = n_tile > 64 ? 1 : 0;
    if (const char *ev = getenv("BMOE_DP")) dp = dp && atoi(ev) != 0;
    int fuse = (n_tile <= 64 || dp) ? 1 : 0;
    if (const char *ev = getenv("BMOE_FUSE")) fuse = dp ? 1 : atoi(ev);
    int probe = 0;
    if (const char *ev = getenv("BMOE_PROBE")) probe = dp ? atoi(ev) : 0;
    GemmParams g1{expert_count, expert_offset, buf_of_expert, (int)E, (int)f, (int)d, nmat1, (int)n_tile,
                  kps_for(nmat1, d, n_tile), arena, buf_bytes, 0, static_cast<const uint8_t *>(x_perm),
                  r_max * 128, partials, G, act == BM_ACT_SWIGLU ? 0 : 1, fuse, dp, probe, h_planes, (int)r_max,
                  nullptr};
    GemmParams g2{expert_count, expert_offset, buf_of_expert, (int)E, (int)d, (int)f, 1, (int)n_tile,
                  kps_for(1, f, n_tile), arena, buf_bytes, (long long)nmat1 * f * d * 2, h_planes, r_max * 128,
                  partials, G, 2, fuse, dp, probe, nullptr, 0, y_perm};

    g1.arena_bytes = g2.arena_bytes = n_bufs * buf_bytes;
    const bool timing = g_timing.enabled;
    std::lock_guard<std::mutex> lk(g_timing.mu);
    CallRec *rec = timing ? &new_call(s) : nullptr;
    if (fused) {
        int k1 = 1, k2 = 1;
        fused_kps(nmat1, d, f, n_tile, &k1, &k2);
        g1.kps = k1;
        g2.kps = k2;
        g1.fuse = g2.fuse = 1;
        g1.dp = g2.dp = 0;
        int pre = 1;
        if (const char *ev = getenv("BMOE_PREFETCH_W2")) pre = atoi(ev);
        FusedParams fp{{g1, g2}, counters, (int)wl.tile_cap,
                       reinterpret_cast<unsigned long long *>(static_cast<uint8_t *>(workspace) + wl.bar_off),
                       pre, trace_buffer(G, s), CombineArgs{}, 0, nullptr, nullptr, nullptr, 1, 12, 2};
        if (const char *mi = getenv("BMOE_FFN_MIN_ITERS")) fp.min_iters = std::max(1, atoi(mi));
        const char *gv = getenv("BMOE_FFN_GROUPS");  // read per call: tests switch it
        fp.groups = std::max(1, std::min(gv ? atoi(gv) : 3, kMaxGroups));
        if (const char *mi = getenv("BMOE_FFN_GROUP_ITERS")) fp.group_min_iters = std::max(0, atoi(mi));
        static const int h_ready = getenv("BMOE_H_READY") ? atoi(getenv("BMOE_H_READY")) : 1;
        fp.g[1].partials = reinterpret_cast<float *>(static_cast<uint8_t *>(workspace) + wl.partial_off +
                                                     wl.slot_set_bytes);
        if (h_ready) {
            fp.launch_count = reinterpret_cast<unsigned long long *>(static_cast<uint8_t *>(workspace) + wl.bar_off + 8);
            fp.h_ready = reinterpret_cast<int *>(static_cast<uint8_t *>(workspace) + wl.bar_off + 16);
        }
        static const int pdl = getenv("BMOE_PDL") ? atoi(getenv("BMOE_PDL")) : 0;
        fp.pdl = pdl;
        // the combine joins the launch when bm_combine would take its 16-byte vector path (same code then)
        const bool fuse_cmb = cmb && d % 4 == 0 && d * 4 <= 200 * 1024 &&  // h row in the pipeline smem (as bm_combine)
                              ((reinterpret_cast<uintptr_t>(y_perm) | reinterpret_cast<uintptr_t>(cmb->h)) & 15) == 0;
        if (fuse_cmb) fp.cmb = *cmb;
        // timing record: [start, end] of the one kernel, then an empty GEMM2 interval
        if (timing) fp.span = next_span(s, *rec);
        if (timing && record_event(s, *rec, 0)) return BM_ECUDA;
        const int rc = launch_fused_dispatch(fp, nmat1, k1, k2, G, s);
        if (rc) return rc;
        if (timing && record_event(s, *rec, 1)) return BM_ECUDA;  // one kernel: GEMM2 interval reported as 0
        return fuse_cmb ? BM_OK : separate_combine();
    }
    if (timing && record_event(s, *rec, 0)) return BM_ECUDA;
    if (int rc = launch_gemm_dispatch(g1, G, s)) return rc;
    if (timing && record_event(s, *rec, 1)) return BM_ECUDA;
    if (dp) {  // every tile was finished by its GEMM epilogue
        // GEMM2 (one accumulator per tile) keeps a double-buffered 256-token
        // tile on CTA pairs: wider tiles halve its per-MAC operand traffic
        if (n_tile >= 128 && use_2sm(g2)) {
            const char *ev = getenv("BMOE_NT2");
            g2.n_tile = ev ? atoi(ev) : 256;
        }
        if (timing && record_event(s, *rec, 2)) return BM_ECUDA;
        if (int rc = launch_gemm_dispatch(g2, G, s)) return rc;
        if (timing && record_event(s, *rec, 3)) return BM_ECUDA;
        return separate_combine();
    }
    const int fix_blocks = 4 * G;
    if (int rc = launch_fixup(g1, act == BM_ACT_SWIGLU ? 0 : 1, reinterpret_cast<uint4 *>(h_planes), (int)r_max,
                              nullptr, fix_blocks, s))
        return rc;
    if (timing && record_event(s, *rec, 2)) return BM_ECUDA;
    if (int rc = launch_gemm_dispatch(g2, G, s)) return rc;
    if (timing && record_event(s, *rec, 3)) return BM_ECUDA;
    if (int rc = launch_fixup(g2, 2, nullptr, 0, y_perm, fix_blocks, s)) return rc;
    return separate_combine();
}

extern "C" int bm_set_kernel_timing(int32_t enable) {
    std::lock_guard<std::mutex> lk(g_timing.mu);
    for (CallRec &r : g_timing.eager) destroy_call(r);
    g_timing.eager.clear();
    g_timing.replayed.clear();
    g_timing.res_ms.clear();
    g_timing.res_span.clear();
    g_timing.span_n = 0;
    g_timing.enabled = enable != 0;
    if (g_timing.enabled && !g_timing.span) {
        g_timing.span_cap = 1 << 16;
        BM_CUDA_TRY(cudaMalloc(&g_timing.span, (size_t)g_timing.span_cap * 2 * sizeof(unsigned long long)));
    }
    return BM_OK;
}

namespace bm {
namespace ffn {
// the engine's side of graph timing (see Timing)
void *ffn_timing_take_capture() {
    std::lock_guard<std::mutex> lk(g_timing.mu);
    if (g_timing.capturing.empty()) return nullptr;
    auto *grp = new std::vector<CallRec>(std::move(g_timing.capturing));
    g_timing.capturing.clear();
    return grp;
}
void ffn_timing_replayed(void *group) {
    if (!group) return;
    std::lock_guard<std::mutex> lk(g_timing.mu);
    if (g_timing.enabled) g_timing.replayed.push_back(static_cast<std::vector<CallRec> *>(group));
}
int ffn_timing_harvest() {  // the replayed graphs' launches must have completed
    std::lock_guard<std::mutex> lk(g_timing.mu);
    for (auto *grp : g_timing.replayed)
        for (const CallRec &r : *grp)
            if (int rc = read_call(r)) return rc;
    g_timing.replayed.clear();
    return BM_OK;
}
void ffn_timing_release(void *group) {
    if (!group) return;
    std::lock_guard<std::mutex> lk(g_timing.mu);
    auto *grp = static_cast<std::vector<CallRec> *>(group);
    for (CallRec &r : *grp) destroy_call(r);
    delete grp;
}
// eager records -> results (synchronises on their last events)
int read_eager() {
    for (CallRec &r : g_timing.eager) {
        cudaEvent_t last = r.ev[3] ? r.ev[3] : r.ev[1];
        if (cudaEventSynchronize(last) != cudaSuccess) return BM_ECUDA;
        if (int rc = read_call(r)) return rc;
        destroy_call(r);
    }
    g_timing.eager.clear();
    return BM_OK;
}
}  // namespace ffn
}  // namespace bm

// One float per bm_expert_ffn_bf16 call since timing was enabled: the fused
// decode kernel's on-device span in ms (first CTA entry to last CTA exit,
// globaltimer), 0 for calls without one (prefill GEMMs). Synchronises.
extern "C" int64_t bm_kernel_spans(float *out_host, int64_t cap) {
    std::lock_guard<std::mutex> lk(g_timing.mu);
    if (read_eager() != BM_OK) return -1;
    int64_t n = 0;
    for (float v : g_timing.res_span) {
        if (n >= cap) break;
        out_host[n++] = v;
    }
    return n;
}

extern "C" int bm_kernel_timing_enabled(void) { return g_timing.enabled ? 1 : 0; }

// Two floats per bm_expert_ffn_bf16 call since timing was enabled: GEMM1
// and GEMM2 kernel durations in ms (CUDA events on the launching stream,
// inside the captured graph for calls replayed from one).
extern "C" int64_t bm_kernel_times(float *out_host, int64_t cap) {
    std::lock_guard<std::mutex> lk(g_timing.mu);
    if (read_eager() != BM_OK) return -1;
    int64_t n = 0;
    for (float v : g_timing.res_ms) {
        if (n >= cap) break;
        out_host[n++] = v;
    }
    return n;
}

extern "C" int bm_pack_expert_bf16(const void *w1, const void *w3, const void *w2, int64_t d, int64_t f, int32_t act,
                                   void *dst, bm_stream_t stream) {
    BM_REQUIRE(w1 && w2 && dst && (act == BM_ACT_TANH || w3), BM_EINVAL, "bm_pack_expert_bf16: null pointer");
    BM_REQUIRE(d % kBM == 0 && f % kBM == 0, BM_EINVAL, "d and f must be multiples of 128");
    cudaStream_t s = as_stream(stream);
    uint8_t *out = static_cast<uint8_t *>(dst);
    const long long n1 = f * d / 8;
    const unsigned g = (unsigned)((n1 + 255) / 256);
    if (act == BM_ACT_SWIGLU) {
        pack_tiles_kernel<<<g, 256, 0, s>>>(static_cast<const uint4 *>(w1), (int)f, (int)d, 2, 0, out);
        pack_tiles_kernel<<<g, 256, 0, s>>>(static_cast<const uint4 *>(w3), (int)f, (int)d, 2, 1, out);
        pack_tiles_kernel<<<g, 256, 0, s>>>(static_cast<const uint4 *>(w2), (int)d, (int)f, 1, 0, out + 2 * f * d * 2);
    } else {
        pack_tiles_kernel<<<g, 256, 0, s>>>(static_cast<const uint4 *>(w1), (int)f, (int)d, 1, 0, out);
        pack_tiles_kernel<<<g, 256, 0, s>>>(static_cast<const uint4 *>(w2), (int)d, (int)f, 1, 0, out + f * d * 2);
    }
    BM_LAUNCH_CHECK();
    return BM_OK;
}
