// Offloaded-MoE decode engine: the reference's per-layer decode loop
// (harness.py:315-393) driven over real memory. The control plane
// (cache.cpp) makes every hit / miss / eviction / prefetch decision exactly
// like memtier; this file is the data plane that makes those decisions
// physical: a pool of equally sized HBM expert buffers (capacity per layer
// plus transient staging), H2D fetches from a pinned host mirror on copy
// streams, CUDA events ordering buffer reuse, and the kernel sequence
// gate -> remap -> permute -> grouped FFN -> combine per layer.
#include <cuda_runtime.h>
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <vector>

#include "../../include/bmoe.h"

namespace bm {
void set_error(const char *fmt, ...);
int buddy_remap_impl(const int32_t *topk, const uint8_t *token_allowed, const void *logits, int32_t logits_f64,
                     int64_t B, int64_t k, int64_t E, const uint32_t *resident_bitmap, const int32_t *tbl_ids,
                     const double *tbl_w, const int32_t *tbl_len, int64_t tbl_stride, int64_t H, int64_t rho,
                     int32_t fallback, int32_t method, double beta, const double *beta_dev, double eta, double kappa,
                     int32_t use_local_logit, const int32_t *partition_of, double hop, int32_t *executed,
                     uint8_t *kind, int32_t *used, double *delta_out, uint8_t *batch_allowed_out,
                     bm_stream_t stream, int32_t *hp_topk, int32_t *hp_executed, uint8_t *hp_kind,
                     uint8_t *hp_allowed, uint8_t *hp_batch_ok);
int random_plan_batch(const int32_t *topk, int64_t B, int64_t k, const uint32_t *resident_bits, int64_t E,
                      bm_pcg64 *rng, int32_t *executed, uint8_t *kind, int32_t *used);
namespace ffn {  // timing of FFN launches inside captured graphs (ffn_tc.cu)
void *ffn_timing_take_capture();
void ffn_timing_replayed(void *group);
int ffn_timing_harvest();
void ffn_timing_release(void *group);
}  // namespace ffn
}

#define ENG_CUDA(expr)                                                                                    \
    do {                                                                                                  \
        cudaError_t _e = (expr);                                                                          \
        if (_e != cudaSuccess) {                                                                          \
            bm::set_error("engine %s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e));      \
            return BM_ECUDA;                                                                              \
        }                                                                                                 \
    } while (0)
#define ENG_TRY(expr)             \
    do {                          \
        int _rc = (expr);         \
        if (_rc != BM_OK) return _rc; \
    } while (0)

namespace {

// gating.BetaController (gating.py:168-221) over the shared host
// implementation in beta.cpp (bm_beta_*), on the default candidate grid.
struct BetaController {
    bm_beta_state st{};
    bool active = false;
    double beta = 1.0;
    bool on() const { return active; }
    int init(double budget, double expert_bytes, double initial) {
        beta = initial;
        active = budget >= 0.0;
        if (!active) return BM_OK;
        double grid[11];
        for (int i = 0; i < 11; ++i) grid[i] = (double)i / 10.0;  // DEFAULT_BETA_GRID (gating.py:170)
        return bm_beta_init(&st, budget, expert_bytes, initial, grid, 11, 0.9, 64);
    }
    int record(double delta, int64_t miss_count) { return bm_beta_record(&st, delta, miss_count, &beta); }
    // beta_wire_bytes: the budget check prices a miss at what a fetch measurably moved
    void set_miss_bytes(double b) { st.expert_bytes = b; }
};

struct Buffer {
    void *dev = nullptr;
    cudaEvent_t free_ev = nullptr;  // last compute that read it (borrowed per-layer event)
};

// Staging ring of the coded fetch path: coded pieces land in a slot on the
// copy stream, a high-priority decode stream rebuilds them into the target
// HBM buffer; a slot is refilled only after its previous decode finished.
constexpr int kRingSlots = 4;
struct Ring {
    uint8_t *slot[kRingSlots] = {};
    cudaEvent_t copied[kRingSlots] = {}, decoded[kRingSlots] = {};
    bool used[kRingSlots] = {};
    int next = 0;
    cudaStream_t dec = nullptr;
};

// Bounded pool of timing-event pairs (stall and copy-engine busy time). A
// pair is harvested into the running sum when its slot comes round again
// (by then it completed long ago, so the synchronize does not block the
// step) or when the stats are read; no event is created per step.
struct TimingRing {
    static constexpr int kPairs = 256;
    cudaEvent_t a[kPairs] = {}, b[kPairs] = {};
    bool live[kPairs] = {};
    int head = 0;
    double acc_ms = 0.0;
    int init() {
        for (int i = 0; i < kPairs; ++i) {
            if (cudaEventCreate(&a[i]) != cudaSuccess || cudaEventCreate(&b[i]) != cudaSuccess) return BM_ECUDA;
        }
        return BM_OK;
    }
    int harvest(int i) {
        if (!live[i]) return BM_OK;
        ENG_CUDA(cudaEventSynchronize(b[i]));
        float ms = 0.f;
        ENG_CUDA(cudaEventElapsedTime(&ms, a[i], b[i]));
        acc_ms += ms;
        live[i] = false;
        return BM_OK;
    }
    // the next pair to record into (its previous use harvested first)
    int next(cudaEvent_t *ea, cudaEvent_t *eb) {
        const int i = head;
        head = (head + 1) % kPairs;
        ENG_TRY(harvest(i));
        live[i] = true;
        *ea = a[i];
        *eb = b[i];
        return BM_OK;
    }
    int drain(double *out_ms) {
        for (int i = 0; i < kPairs; ++i) ENG_TRY(harvest(i));
        *out_ms = acc_ms;
        acc_ms = 0.0;
        return BM_OK;
    }
    void release() {
        for (int i = 0; i < kPairs; ++i) {
            if (a[i]) cudaEventDestroy(a[i]);
            if (b[i]) cudaEventDestroy(b[i]);
        }
    }
};

}  // namespace

struct bm_engine {
    bm_engine_config cfg{};
    int L = 0, E = 0, k = 0, d = 0, f = 0, cap = 0, S = 0, nbufs = 0, reserve = 0, K = 0;
    size_t buf_bytes = 0;
    int64_t buf_elems = 0;
    uint8_t *arena = nullptr;
    std::vector<Buffer> bufs;
    std::vector<int> free_list;
    std::vector<std::vector<int>> phys;            // [L][E] buffer id or -1
    std::vector<std::vector<cudaEvent_t>> ready;   // [L][E] copy-complete events
    std::vector<std::vector<uint8_t>> ready_pending;
    std::vector<std::vector<cudaStream_t>> ready_stream;  // [L][E] stream the ready event was recorded on
    std::vector<cudaEvent_t> buf_ev;                      // [nbufs] free events of buffers released in flight
    std::vector<cudaEvent_t> layer_done;           // [L]
    std::vector<const uint8_t *> host_mirror;
    bool coded = false;       // host_mirror[l] is an exponent-coded layer image (cfg.fetch_codec)
    size_t ring_slot_bytes = 0;
    Ring ring_copy, ring_prefetch;
    const float *gate_w = nullptr, *gate_b = nullptr;
    // Psi ordering of the candidates (substitution.py:107-143; bm_engine_set_psi)
    bool psi = false;
    const double *tbl_w = nullptr;
    double eta = 0.0, kappa = 0.0, hop = 1.0;
    int32_t use_local_logit = 1;
    const int32_t *partition_of = nullptr;
    const int32_t *tbl_ids = nullptr, *tbl_len = nullptr;
    std::vector<double> tau;
    bm_cache *cache = nullptr;
    // device workspaces
    float *logits = nullptr, *probs = nullptr, *y_perm = nullptr, *h_ws = nullptr;
    double *tae = nullptr, *margin = nullptr, *delta = nullptr;
    int32_t *used = nullptr;
    // views into the packed plan buffers, re-carved per batch size (carve())
    int32_t *topk = nullptr, *executed = nullptr;
    uint8_t *kind = nullptr, *allowed = nullptr, *batch_ok = nullptr;
    int32_t *count = nullptr, *offset = nullptr, *row_token = nullptr, *slot_row = nullptr;
    int32_t *perm_scratch = nullptr;  // chunk histograms of the multi-CTA permute (prefill plans)
    int64_t perm_scratch_elems = 0;
    // shared experts (always resident, outside the budget): plan extended to k + Ssh slots
    int Ssh = 0;
    int32_t *exec_ext = nullptr;
    uint8_t *kind_ext = nullptr;
    float *probs_ext = nullptr;
    std::vector<int> shared_buf;  // [L][Ssh] buffer ids
    void *x_perm = nullptr, *ffn_ws = nullptr;
    int64_t ffn_ws_bytes = 0, r_max = 0, device_bytes = 0;
    // host views into the pinned plan pack
    int32_t *topk_h = nullptr, *exec_h = nullptr;
    uint8_t *kind_h = nullptr, *allowed_h = nullptr, *batch_ok_h = nullptr;
    cudaEvent_t plan_ev = nullptr;
    cudaStream_t copy_stream = nullptr, prefetch_stream = nullptr;
    std::vector<std::vector<int32_t>> prev_counts;  // [L][E]
    // packed plan readback, per-layer staging (graph-stable addresses), graphs
    uint8_t *plan_dev = nullptr, *plan_host = nullptr;
    uint8_t *plan_host_dev = nullptr;  // the same pinned plan seen from the device (mapped)
    int32_t *topk_hd = nullptr, *exec_hd = nullptr;
    uint8_t *kind_hd = nullptr, *allowed_hd = nullptr, *batch_ok_hd = nullptr;
    float *h_int = nullptr;                       // engine-owned hidden state [max_batch][d]
    uint32_t *bm_dev_all = nullptr, *bm_host_all = nullptr;
    int32_t *bo_dev_all = nullptr, *bo_host_all = nullptr;
    std::vector<uint32_t *> bm_dev_l, bm_host_l;  // per-layer residency bitmaps (+ the beta the remap uses)
    std::vector<uint32_t *> bm_hostdev_l;         // bm_host_l seen from the device (mapped pinned memory)
    // the remap reads the snapshot and writes the packed plan through mapped pinned memory: no
    // upload or readback copy on the layer-step's host round trip (BMOE_ZERO_COPY=0: the copies)
    bool zero_copy = true;
    int bm_stride = 0, beta_word = 0;            // u32 words per layer slot; beta (f64) at word beta_word
    BetaController beta_ctl;
    int64_t wire_total = 0, fetch_total = 0;  // every physical fetch since creation (stats resets keep them)
    bm_pcg64 rng{};  // method RANDOM: numpy's PCG64 stream of harness.py:299-300, advanced on the host
    std::vector<int32_t *> bo_dev_l, bo_host_l;   // per-layer buffer maps (E + shared)
    cudaStream_t cap_stream = nullptr;
    bool use_graphs = true;
    std::map<std::pair<int, int64_t>, std::pair<int, cudaGraphExec_t>> g_pre, g_post, g_post2;
    std::map<cudaGraphExec_t, void *> timing_groups;  // timed FFN calls captured in a graph
    // split expert counts: resident | fetched (early + late) -> early | late
    int32_t *count_a = nullptr, *count_b = nullptr, *count_bc = nullptr, *count_c = nullptr;
    bool overlap_fetch = true;  // run resident experts' GEMMs while misses stream in (BMOE_OVERLAP=0 disables)
    // early fetched experts' GEMMs while the last one streams in (BMOE_SPLIT_FETCHED=1): measured
    // +0.7% Mixtral / +0.8% Qwen3 decode tokens/s (within run-to-run noise), at the price of
    // a third, smaller FFN launch per layer-step (FFN roofline 0.84 -> 0.81, 0.49 -> 0.36); off
    bool split_fetched = false;
    // K5 joins the layer-step's last bf16 FFN launch (bm_expert_ffn_bf16_combine; BMOE_FUSE_COMBINE=0: own launch)
    bool fuse_combine = true;
    // CTAs for the decode of pieces off the critical path (BMOE_DECODE_NARROW; 0: full grid)
    int32_t decode_narrow = 296;
    bm_engine_stats stats{};
    TimingRing stall_ev, copy_ev;
    std::vector<uint8_t> mask_tmp;
    std::vector<double> pend_done;
    std::vector<int32_t> pend_exp;
    // optional per-layer-step trace (routing, gates, snapshot, plan) for parity checks
    bool tracing = false;
    bool copy_timing = false;
    std::vector<int32_t> tr_layer, tr_B, tr_topk, tr_exec;
    std::vector<uint8_t> tr_allowed, tr_batch_ok, tr_kind;
    std::vector<uint32_t> tr_bitmap;
    std::vector<double> tr_tae, tr_margin, tr_delta;

    template <typename T>
    int dmalloc(T **p, size_t n) {
        ENG_CUDA(cudaMalloc(reinterpret_cast<void **>(p), n * sizeof(T) + 16));
        device_bytes += (int64_t)(n * sizeof(T));
        return BM_OK;
    }
    template <typename T>
    int hmalloc(T **p, size_t n) {
        ENG_CUDA(cudaHostAlloc(reinterpret_cast<void **>(p), n * sizeof(T) + 16, cudaHostAllocPortable | cudaHostAllocMapped));
        return BM_OK;
    }

    std::vector<int> pending_experts(int layer) {
        int64_t sc[4];
        bm_cache_layer_state(cache, layer, nullptr, nullptr, sc);
        pend_done.resize(sc[1] + 1);
        pend_exp.resize(sc[1] + 1);
        bm_cache_pending(cache, layer, pend_done.data(), pend_exp.data(), sc[1]);
        return std::vector<int>(pend_exp.begin(), pend_exp.begin() + sc[1]);
    }

    int alloc_buffer(int *out) {
        if (free_list.empty()) {
            bm::set_error("engine: expert buffer pool exhausted (staging too small)");
            return BM_EINVARIANT;
        }
        *out = free_list.back();
        free_list.pop_back();
        return BM_OK;
    }

    const bm_xfer_blob_header *blob_of(int l, int e) const {
        const auto *lh = reinterpret_cast<const bm_xfer_layer_header *>(host_mirror[l]);
        return reinterpret_cast<const bm_xfer_blob_header *>(host_mirror[l] + lh->blob_off[e]);
    }

    // Coded transfer of expert e of layer l into dst: each piece is copied
    // into a ring slot on stream s and decoded on the ring's decode stream.
    // Returns the wire bytes; the decode stream holds the completion.
    // critical: the expert whose arrival the layer-step's last FFN waits for; only its last
    // piece is decoded on the full grid
    int enqueue_coded(int l, int e, void *dst, cudaStream_t s, Ring &r, int64_t *wire, bool critical = true) {
        const bm_xfer_blob_header *bh = blob_of(l, e);
        const uint8_t *blob = reinterpret_cast<const uint8_t *>(bh);
        *wire = 0;
        for (uint32_t p = 0; p < bh->n_pieces; ++p) {
            const int j = r.next;
            r.next = (r.next + 1) % kRingSlots;
            if (r.used[j]) ENG_CUDA(cudaStreamWaitEvent(s, r.decoded[j], 0));
            const size_t sz = (size_t)(bh->piece_off[p + 1] - bh->piece_off[p]);
            ENG_CUDA(cudaMemcpyAsync(r.slot[j], blob + bh->piece_off[p], sz, cudaMemcpyHostToDevice, s));
            ENG_CUDA(cudaEventRecord(r.copied[j], s));
            ENG_CUDA(cudaStreamWaitEvent(r.dec, r.copied[j], 0));
            const auto *ph = reinterpret_cast<const bm_xfer_piece_header *>(blob + bh->piece_off[p]);
            // an expert's last piece gates its FFN: full grid; the others only have to keep
            // up with the copy of the next piece, so they take a narrow grid (decode_narrow)
            const bool last = critical && p + 1 == bh->n_pieces;
            ENG_TRY(bm_xfer_decode_piece_ctas(r.slot[j],
                                              static_cast<uint16_t *>(dst) + (size_t)p * bh->piece_values,
                                              ph->n_chunks, last ? 0 : decode_narrow, r.dec));
            ENG_CUDA(cudaEventRecord(r.decoded[j], r.dec));
            r.used[j] = true;
            *wire += (int64_t)sz;
            ++stats.kernel_launches;
        }
        return BM_OK;
    }

    // H2D of expert e of layer l into a fresh buffer on stream s
    int fetch(int l, int e, cudaStream_t s, bool critical = true) {
        int b;
        ENG_TRY(alloc_buffer(&b));
        cudaEvent_t c0 = nullptr, c1 = nullptr;  // copy-engine busy time, for the PCIe roofline
        if (copy_timing) ENG_TRY(copy_ev.next(&c0, &c1));
        cudaStream_t done = s;
        if (coded) {
            Ring &r = (s == prefetch_stream) ? ring_prefetch : ring_copy;
            if (bufs[b].free_ev) ENG_CUDA(cudaStreamWaitEvent(r.dec, bufs[b].free_ev, 0));  // the decode writes it
            if (c0) ENG_CUDA(cudaEventRecord(c0, s));
            int64_t wire = 0;
            ENG_TRY(enqueue_coded(l, e, bufs[b].dev, s, r, &wire, critical));
            if (c1) ENG_CUDA(cudaEventRecord(c1, s));
            stats.wire_bytes += wire;
            wire_total += wire;
            done = r.dec;
        } else {
            if (bufs[b].free_ev) ENG_CUDA(cudaStreamWaitEvent(s, bufs[b].free_ev, 0));
            if (c0) ENG_CUDA(cudaEventRecord(c0, s));
            ENG_CUDA(cudaMemcpyAsync(bufs[b].dev, host_mirror[l] + (size_t)e * buf_bytes, buf_bytes,
                                     cudaMemcpyHostToDevice, s));
            if (c1) ENG_CUDA(cudaEventRecord(c1, s));
            stats.wire_bytes += (int64_t)buf_bytes;
            wire_total += (int64_t)buf_bytes;
        }
        ++fetch_total;
        ENG_CUDA(cudaEventRecord(ready[l][e], done));
        ready_pending[l][e] = 1;
        ready_stream[l][e] = done;
        phys[l][e] = b;
        stats.h2d_bytes += (int64_t)buf_bytes;
        return BM_OK;
    }

    // synchronous upload (initial residents, shared experts)
    int upload(int l, int e, int b) {
        if (!coded) {
            ENG_CUDA(cudaMemcpy(bufs[b].dev, host_mirror[l] + (size_t)e * buf_bytes, buf_bytes,
                                cudaMemcpyHostToDevice));
            return BM_OK;
        }
        int64_t wire = 0;
        ENG_TRY(enqueue_coded(l, e, bufs[b].dev, copy_stream, ring_copy, &wire));
        ENG_CUDA(cudaStreamSynchronize(ring_copy.dec));
        ENG_CUDA(cudaStreamSynchronize(copy_stream));
        return BM_OK;
    }

    // plan pack [topk | executed | kind | allowed | batch_ok] for batch B (device + pinned host)
    void carve(int64_t B) {
        topk = reinterpret_cast<int32_t *>(plan_dev);
        executed = topk + B * k;
        kind = reinterpret_cast<uint8_t *>(executed + B * k);
        allowed = kind + B * k;
        batch_ok = allowed + B;
        topk_h = reinterpret_cast<int32_t *>(plan_host);
        exec_h = topk_h + B * k;
        kind_h = reinterpret_cast<uint8_t *>(exec_h + B * k);
        allowed_h = kind_h + B * k;
        batch_ok_h = allowed_h + B;
        topk_hd = reinterpret_cast<int32_t *>(plan_host_dev);
        exec_hd = topk_hd + B * k;
        kind_hd = reinterpret_cast<uint8_t *>(exec_hd + B * k);
        allowed_hd = kind_hd + B * k;
        batch_ok_hd = allowed_hd + B;
    }
    static size_t plan_bytes(int64_t B, int k) { return (size_t)B * k * 9 + (size_t)B + 1; }

    // K1 gate, snapshot upload, K2 remap, packed plan readback
    int enqueue_pre(int l, float *h, int64_t B, cudaStream_t s) {
        ENG_TRY(bm_gate_topk(h, gate_w + (size_t)l * E * d, gate_b + (size_t)l * E, B, E, d, k, cfg.temperature,
                             tau[l], cfg.gamma, logits, topk, probs, tae, margin, allowed, s));
        const bool zc = zero_copy && plan_host_dev;
        if (!zc)
            ENG_CUDA(cudaMemcpyAsync(bm_dev_l[l], bm_host_l[l], bm_stride * sizeof(uint32_t), cudaMemcpyHostToDevice,
                                     s));
        uint32_t *bits = zc ? bm_hostdev_l[l] : bm_dev_l[l];
        const bool p = psi && cfg.method == BM_METHOD_BUDDY;
        ENG_TRY(bm::buddy_remap_impl(topk, allowed, p ? logits : nullptr, 0, B, k, E, bits,
                                     tbl_ids ? tbl_ids + (size_t)l * E * K : nullptr,
                                     p ? tbl_w + (size_t)l * E * K : nullptr,
                                     tbl_len ? tbl_len + (size_t)l * E : nullptr, K > 0 ? K : 1, cfg.search_rank_h,
                                     cfg.rho, cfg.fallback,
                                     cfg.method == BM_METHOD_RANDOM ? BM_METHOD_ORIGINAL : cfg.method, cfg.beta,
                                     reinterpret_cast<const double *>(bits + beta_word), p ? eta : 0.0,
                                     p ? kappa : 0.0, use_local_logit, p ? partition_of : nullptr, hop, executed, kind,
                                     used, delta, batch_ok, s, zc ? topk_hd : nullptr, zc ? exec_hd : nullptr,
                                     zc ? kind_hd : nullptr, zc ? allowed_hd : nullptr, zc ? batch_ok_hd : nullptr));
        if (!zc) ENG_CUDA(cudaMemcpyAsync(plan_host, plan_dev, plan_bytes(B, k), cudaMemcpyDeviceToHost, s));
        return BM_OK;
    }

    // Post phase, part 1 (before the fetch waits): buffer map + fetch mask
    // upload, K3 permute, gather, and — bf16 path — K4 over the experts that
    // are already in HBM, overlapping the H2D copies of the missing ones.
    int enqueue_post1(int l, float *h, int64_t B, bool with_combine, cudaStream_t s) {
        const int Et = E + Ssh, kt = k + Ssh;
        ENG_CUDA(cudaMemcpyAsync(bo_dev_l[l], bo_host_l[l], 3 * Et * sizeof(int32_t), cudaMemcpyHostToDevice, s));
        if (cfg.method == BM_METHOD_RANDOM)  // the host-drawn plan [executed | kind] replaces K2's on-demand plan
            ENG_CUDA(cudaMemcpyAsync(executed, exec_h, (size_t)B * k * 5, cudaMemcpyHostToDevice, s));
        const int32_t *pe = executed;
        const uint8_t *pk = kind;
        if (Ssh) {  // every token also runs the shared experts with weight 1
            ENG_TRY(bm_append_shared(executed, kind, probs, B, k, E, Ssh, exec_ext, kind_ext, probs_ext, s));
            pe = exec_ext;
            pk = kind_ext;
        }
        ENG_TRY(bm_permute_ws(pe, pk, B, kt, Et, 16, count, offset, row_token, slot_row, perm_scratch,
                              perm_scratch_elems, s));
        if (cfg.fp32_weights) {
            ENG_TRY(bm_gather_rows(h, B, d, row_token, offset, Et, r_max, 0, x_perm, s));
            return BM_OK;  // the fp32 parity path runs in one piece after the waits
        }
        ENG_TRY(bm_gather_rows(h, B, d, row_token, offset, Et, r_max, 1, x_perm, s));
        ENG_TRY(bm_split_counts(count, bo_dev_l[l] + Et, Et, count_a, count_bc, s));
        ENG_TRY(bm_split_counts(count_bc, bo_dev_l[l] + 2 * Et, Et, count_b, count_c, s));
        return ffn_bf16(l, h, B, count_a, with_combine, s);
    }

    // no expert gets more than B rows: the token tile is sized to the batch
    int token_tile(int64_t B) const { return std::min(cfg.n_tile, std::max(16, (int)((B + 15) / 16 * 16))); }

    // K4 over the experts with rows in cnt; with_combine: K5 (+ layer_update, in place on h)
    // joins it (one launch at decode widths, bm_expert_ffn_bf16_combine)
    int ffn_bf16(int l, float *h, int64_t B, const int32_t *cnt, bool with_combine, cudaStream_t s) {
        const int Et = E + Ssh;
        const int nt = token_tile(B);
        if (with_combine)
            return bm_expert_ffn_bf16_combine(x_perm, cnt, offset, Et, d, f, cfg.act, arena, nbufs, bo_dev_l[l],
                                              r_max, nt, ffn_ws, ffn_ws_bytes, y_perm, slot_row,
                                              Ssh ? probs_ext : probs, Ssh ? kind_ext : kind, B, k + Ssh, h, 0.5f,
                                              s);
        return bm_expert_ffn_bf16(x_perm, cnt, offset, Et, d, f, cfg.act, arena, nbufs, bo_dev_l[l], r_max, nt,
                                  ffn_ws, ffn_ws_bytes, y_perm, s);
    }

    // Post phase, part 2 (after the waits): K4 over the fetched experts (only the last-fetched
    // one when the others already ran while it was on the wire), K5 combine (in place)
    int enqueue_post2(int l, float *h, int64_t B, bool fetched, bool late_only, cudaStream_t s) {
        const int Et = E + Ssh, kt = k + Ssh;
        if (cfg.fp32_weights) {
            ENG_TRY(bm_expert_ffn_f32(static_cast<float *>(x_perm), count, offset, Et, d, f, cfg.act,
                                      reinterpret_cast<const float *>(arena), buf_elems, bo_dev_l[l], r_max, h_ws,
                                      y_perm, s));
        } else if (fetched) {  // the last FFN call of the layer-step carries the combine
            ENG_TRY(ffn_bf16(l, h, B, late_only ? count_c : count_b, fuse_combine, s));
            if (fuse_combine) return BM_OK;
        } else if (fuse_combine) {
            return BM_OK;  // it ran with the resident experts' FFN (post1)
        }
        ENG_TRY(bm_combine(y_perm, slot_row, Ssh ? probs_ext : probs, Ssh ? kind_ext : kind, B, kt, d, h, 0.5f, h, s));
        return BM_OK;
    }

    // Replay a per-(layer, B) CUDA graph of enqueue_pre/post (captured on the
    // second occurrence; the first runs eagerly and warms lazy attributes).
    // With kernel timing on, separate graphs are captured whose FFN launches are bracketed
    // by external event nodes (and span stamps), so the timing pass measures the kernels as
    // the timed run launches them; each replay's times are read back after the step.
    template <typename Body>
    int run(std::map<std::pair<int, int64_t>, std::pair<int, cudaGraphExec_t>> &cache_g, int l, int variant,
            float *h, int64_t B, cudaStream_t s, Body body) {
        (void)h;
        if (!use_graphs) return body(s);
        const bool timing = bm_kernel_timing_enabled() != 0;
        auto &slot = cache_g[{l * 3 + variant + (timing ? (1 << 20) : 0), B}];
        if (slot.second == nullptr) {
            if (!timing && slot.first++ == 0) return body(s);
            cudaGraph_t g;
            ENG_CUDA(cudaStreamBeginCapture(cap_stream, cudaStreamCaptureModeThreadLocal));
            int rc = body(cap_stream);
            cudaError_t ce = cudaStreamEndCapture(cap_stream, &g);
            void *grp = bm::ffn::ffn_timing_take_capture();
            if (rc != BM_OK || ce != cudaSuccess) bm::ffn::ffn_timing_release(grp);
            if (rc != BM_OK) return rc;
            ENG_CUDA(ce);
            ENG_CUDA(cudaGraphInstantiate(&slot.second, g, 0));
            cudaGraphDestroy(g);
            if (grp) timing_groups[slot.second] = grp;
        }
        ENG_CUDA(cudaGraphLaunch(slot.second, s));
        if (timing) {
            auto it = timing_groups.find(slot.second);
            if (it != timing_groups.end()) bm::ffn::ffn_timing_replayed(it->second);
        }
        return BM_OK;
    }

    int layer_step(int l, float *h, int64_t B, const int32_t *tokens, cudaStream_t s) {
        carve(B);
        // 1. speculative loads for the next layer (harness.py:321-326)
        if (cfg.prefetch_enabled && L > 1) {
            const int t = l + 1 < L ? l + 1 : 0;
            int32_t preds[1024];
            int64_t np = 0;
            ENG_TRY(bm_cache_predict(cache, t, prev_counts[t].data(), preds, &np));
            if (np > 0) {
                std::vector<int> before = pending_experts(t);
                ENG_TRY(bm_cache_prefetch(cache, t, preds, np));
                std::vector<int> after = pending_experts(t);
                for (int e : after) {
                    if (std::find(before.begin(), before.end(), e) != before.end()) continue;
                    if (phys[t][e] >= 0 || (int)free_list.size() <= reserve) continue;  // keep the on-demand reserve
                    ENG_TRY(fetch(t, e, prefetch_stream, false));  // speculative: never critical
                    ++stats.prefetch_copies;
                }
            }
        }
        // 2. commit completed transfers (harness.py:327-329)
        ENG_TRY(bm_cache_settle(cache, l));
        // 3-5. K1 router, snapshot, K2 remap, plan readback (harness.py:331-361)
        const int words = (E + 31) / 32;
        ENG_TRY(bm_cache_snapshot(cache, l, nullptr, bm_host_l[l]));
        *reinterpret_cast<double *>(bm_host_l[l] + beta_word) = beta_ctl.beta;  // harness.py:336-337
        ENG_TRY(run(g_pre, l, 0, h, B, s, [&](cudaStream_t st) { return enqueue_pre(l, h, B, st); }));
        ENG_CUDA(cudaEventRecord(plan_ev, s));
        ENG_CUDA(cudaEventSynchronize(plan_ev));
        if (cfg.method == BM_METHOD_RANDOM)  // substitution.random_plan per token (harness.py:358-359)
            ENG_TRY(bm::random_plan_batch(topk_h, B, k, bm_host_l[l], E, &rng, exec_h, kind_h, nullptr));
        if (cfg.method == BM_METHOD_BUDDY) {
            for (int64_t b = 0; b < B; ++b) stats.gate_forbidden += allowed_h[b] ? 0 : 1;
            stats.batch_bypassed += batch_ok_h[0] ? 0 : 1;
            if (beta_ctl.on()) {  // controller.record(delta, miss_count) (harness.py:354-357)
                const uint32_t *bits = bm_host_l[l];
                auto resident = [&](int e) { return (bits[e >> 5] >> (e & 31)) & 1u; };
                int64_t miss_slots = 0, miss_unique = 0;
                std::vector<uint8_t> seen(E, 0);
                for (int64_t i = 0; i < B * k; ++i) {
                    const int e = topk_h[i];
                    if (!resident(e)) {
                        ++miss_slots;
                        if (!seen[e]) ++miss_unique;
                    }
                    seen[e] = 1;
                }
                if (cfg.beta_wire_bytes && fetch_total > 0)
                    beta_ctl.set_miss_bytes((double)wire_total / (double)fetch_total);
                ENG_TRY(beta_ctl.record((double)miss_slots / (double)(B * k), miss_unique));  // delta as in K2
            }
        }
        if (tracing) {
            tr_layer.push_back(l);
            tr_B.push_back((int32_t)B);
            tr_topk.insert(tr_topk.end(), topk_h, topk_h + B * k);
            tr_exec.insert(tr_exec.end(), exec_h, exec_h + B * k);
            tr_kind.insert(tr_kind.end(), kind_h, kind_h + B * k);
            tr_allowed.insert(tr_allowed.end(), allowed_h, allowed_h + B);
            tr_batch_ok.push_back(batch_ok_h[0]);
            tr_bitmap.insert(tr_bitmap.end(), bm_host_l[l], bm_host_l[l] + words);
            // gate record fields (harness.py:345-350): K1's f64 TAE and margin, K2's delta
            const size_t t0 = tr_tae.size();
            tr_tae.resize(t0 + B);
            tr_margin.resize(t0 + B);
            tr_delta.resize(tr_delta.size() + 1);
            ENG_CUDA(cudaMemcpy(tr_tae.data() + t0, tae, B * sizeof(double), cudaMemcpyDeviceToHost));
            ENG_CUDA(cudaMemcpy(tr_margin.data() + t0, margin, B * sizeof(double), cudaMemcpyDeviceToHost));
            ENG_CUDA(cudaMemcpy(&tr_delta.back(), delta, sizeof(double), cudaMemcpyDeviceToHost));
        }
        std::vector<int32_t> &cnt = prev_counts[l];  // harness.py:384-389
        std::fill(cnt.begin(), cnt.end(), 0);
        for (int64_t i = 0; i < B * k; ++i) {
            if (kind_h[i] == BM_KIND_DROPPED) {
                ++stats.drops;
                continue;
            }
            ++cnt[exec_h[i]];
        }
        // 7. data plane: every executed expert must be in HBM before the GEMM. The copies
        // depend only on the plan and on which experts hold HBM buffers (buffers freed by
        // this step's evictions are released after its compute), not on the replay, so
        // they are enqueued first and the replay below runs on the CPU while they move.
        std::vector<cudaEvent_t> waits;
        std::vector<int> wait_experts;
        ++stats.ffn_calls;
        int last_fetch = -1;  // the copies go out in expert order: the last one gates the FFN
        for (int e = 0; e < E; ++e)
            if (cnt[e] && phys[l][e] < 0) last_fetch = e;
        for (int e = 0; e < E; ++e) {
            if (!cnt[e]) continue;
            ++stats.ffn_experts;
            stats.ffn_rows += cnt[e];
            if (phys[l][e] < 0) {
                ENG_TRY(fetch(l, e, copy_stream, e == last_fetch));
                ++stats.physical_fetches;
            }
            if (ready_pending[l][e]) {
                waits.push_back(ready[l][e]);
                wait_experts.push_back(e);
                ready_pending[l][e] = 0;
            }
        }
        // 6. control plane: replay accesses in (token, slot) order (harness.py:363-382),
        // overlapping the copies enqueued above
        int64_t out4[4];
        ENG_TRY(bm_cache_apply_plan(cache, l, B, k, tokens, topk_h, exec_h, kind_h, out4));
        stats.executed_slots += out4[0];
        stats.ondemand_misses += out4[1];
        stats.substitutions += out4[2];
        ENG_TRY(bm_cache_advance(cache, cfg.compute_ms * (double)out4[0]));
        const int Et = E + Ssh;
        int32_t *bo = bo_host_l[l];  // [buffer map (Et) | fetched-this-step mask (Et) | late mask (Et)]
        for (int e = 0; e < E; ++e) {
            bo[e] = phys[l][e] >= 0 ? phys[l][e] : 0;
            bo[Et + e] = 0;
        }
        for (int sx = 0; sx < Ssh; ++sx) {
            bo[E + sx] = shared_buf[(size_t)l * Ssh + sx];
            bo[Et + E + sx] = 0;
        }
        for (int e = 0; e < Et; ++e) bo[2 * Et + e] = 0;
        for (int e : wait_experts) bo[Et + e] = 1;
        if (!overlap_fetch && !waits.empty())  // A/B switch: everything after the waits
            for (int e = 0; e < Et; ++e) bo[Et + e] = 1;
        // With two or more experts in flight, all but the last one (the last copy enqueued)
        // run their FFN while it is still on the wire; only its FFN follows its arrival.
        const bool split_late = overlap_fetch && split_fetched && !cfg.fp32_weights && waits.size() >= 2;
        if (split_late) bo[2 * Et + wait_experts.back()] = 1;
        stats.ffn_experts += Ssh;
        stats.ffn_rows += (int64_t)B * Ssh;
        // 8. K3 -> K4 (resident experts) || H2D of the missing ones -> K4 (fetched) -> K5
        const bool fetched = !waits.empty();
        ENG_TRY(run(g_post, l, fetched ? 0 : 1, h, B, s,
                    [&](cudaStream_t st) { return enqueue_post1(l, h, B, fuse_combine && !fetched, st); }));
        if (fetched) {
            cudaEvent_t a, bb;
            ENG_TRY(stall_ev.next(&a, &bb));
            ENG_CUDA(cudaEventRecord(a, s));
            if (split_late) {
                for (size_t i = 0; i + 1 < waits.size(); ++i) ENG_CUDA(cudaStreamWaitEvent(s, waits[i], 0));
                ENG_TRY(ffn_bf16(l, h, B, count_b, false, s));  // the early fetched experts
                ENG_CUDA(cudaStreamWaitEvent(s, waits.back(), 0));
            } else {
                for (cudaEvent_t w : waits) ENG_CUDA(cudaStreamWaitEvent(s, w, 0));
            }
            ENG_CUDA(cudaEventRecord(bb, s));
        }
        ENG_TRY(run(g_post2, l, split_late ? 2 : (fetched ? 1 : 0), h, B, s,
                    [&](cudaStream_t st) { return enqueue_post2(l, h, B, fetched, split_late, st); }));
        {  // gate, remap, permute (3 kernels at prefill sizes), gather, combine (+ append_shared) + the FFN kernels
            int64_t n = 5 + (Ssh ? 1 : 0) + ((int64_t)B * (k + Ssh) >= 4 * 1024 ? 2 : 0);
            if (cfg.fp32_weights) {
                n += 2;
            } else {
                const int nt = std::min(cfg.n_tile, std::max(16, (int)((B + 15) / 16 * 16)));
                // decode width: one fused launch; prefill: GEMM1 + GEMM2 (data-parallel);
                // the A/B switches restore GEMM + fixup pairs
                const char *ev = getenv(nt <= 64 ? "BMOE_FUSED" : "BMOE_DP");
                const int per_call = (ev && atoi(ev) == 0) ? 4 : (nt <= 64 ? 1 : 2);
                n += 2 + per_call * (1 + (fetched ? 1 : 0) + (split_late ? 1 : 0));  // split_counts x2 + FFN calls
                if (fuse_combine && nt <= 64 && per_call == 1) --n;  // K5 ran inside the last fused FFN launch
            }
            stats.kernel_launches += n;
        }
        // 9. release buffers of experts the control plane no longer holds
        ENG_CUDA(cudaEventRecord(layer_done[l], s));
        ENG_TRY(bm_cache_snapshot(cache, l, mask_tmp.data(), nullptr));
        std::vector<int> pend = pending_experts(l);
        for (int e = 0; e < E; ++e) {
            const int b = phys[l][e];
            if (b < 0 || mask_tmp[e] || std::find(pend.begin(), pend.end(), e) != pend.end()) continue;
            if (ready_pending[l][e]) {
                // Prefetched, settled and evicted before any step used it: its copy/decode may
                // still be writing the buffer, and layer_done[l] does not follow it. The
                // buffer's next writer waits for both (recorded on the producing stream, so
                // the compute stream never waits for a speculative copy).
                cudaStream_t ps = ready_stream[l][e];
                ENG_CUDA(cudaStreamWaitEvent(ps, layer_done[l], 0));
                ENG_CUDA(cudaEventRecord(buf_ev[b], ps));
                bufs[b].free_ev = buf_ev[b];
                ++stats.inflight_releases;
            } else {
                bufs[b].free_ev = layer_done[l];
            }
            free_list.push_back(b);
            phys[l][e] = -1;
            ready_pending[l][e] = 0;
        }
        return BM_OK;
    }

    void release() {
        if (arena) cudaFree(arena);
        for (auto &v : ready)
            for (cudaEvent_t e : v)
                if (e) cudaEventDestroy(e);
        for (cudaEvent_t e : layer_done)
            if (e) cudaEventDestroy(e);
        stall_ev.release();
        copy_ev.release();
        for (cudaEvent_t e : buf_ev)
            if (e) cudaEventDestroy(e);
        for (auto *m : {&g_pre, &g_post, &g_post2})
            for (auto &kv : *m)
                if (kv.second.second) cudaGraphExecDestroy(kv.second.second);
        for (auto &kv : timing_groups) bm::ffn::ffn_timing_release(kv.second);
        void *dptrs[] = {exec_ext, kind_ext, probs_ext, logits, probs, y_perm, h_ws, tae, margin, delta, used,
                         plan_dev, h_int, bm_dev_all, bo_dev_all, count, offset, row_token, slot_row, perm_scratch,
                         x_perm, ffn_ws,
                         count_a, count_b, count_bc, count_c};
        for (void *p : dptrs)
            if (p) cudaFree(p);
        void *hptrs[] = {plan_host, bm_host_all, bo_host_all};
        for (void *p : hptrs)
            if (p) cudaFreeHost(p);
        if (plan_ev) cudaEventDestroy(plan_ev);
        if (cap_stream) cudaStreamDestroy(cap_stream);
        for (Ring *r : {&ring_copy, &ring_prefetch}) {
            for (int j = 0; j < kRingSlots; ++j) {
                if (r->slot[j]) cudaFree(r->slot[j]);
                if (r->copied[j]) cudaEventDestroy(r->copied[j]);
                if (r->decoded[j]) cudaEventDestroy(r->decoded[j]);
            }
            if (r->dec) cudaStreamDestroy(r->dec);
        }
        if (copy_stream) cudaStreamDestroy(copy_stream);
        if (prefetch_stream) cudaStreamDestroy(prefetch_stream);
        if (cache) bm_cache_destroy(cache);
    }
};

static int engine_init(bm_engine *g, const bm_engine_config *c, const void *const *host_mirror, const float *gate_w,
                       const float *gate_b, const int32_t *tbl_ids, const int32_t *tbl_len, int32_t tbl_k,
                       const double *tau_host, const int32_t *initial_host, const double *static_freq_host) {
    g->cfg = *c;
    g->L = c->num_layers;
    g->E = c->num_experts;
    g->k = c->top_k;
    g->d = c->d;
    g->f = c->f;
    g->cap = c->capacity;
    g->K = tbl_k;
    const int L = g->L, E = g->E, k = g->k;
    if (L < 1 || E < 1 || E + (c->num_shared > 0 ? c->num_shared : 0) > 256 || k < 1 || k > E ||
        c->max_batch < 1 || g->cap < 0 || g->cap > E) {
        bm::set_error("engine: bad configuration");
        return BM_ECONFIG;
    }
    if (c->method < BM_METHOD_BUDDY || c->method > BM_METHOD_RANDOM) {
        bm::set_error("engine: unknown method %d", c->method);
        return BM_ECONFIG;
    }
    if (c->method == BM_METHOD_BUDDY && (!tbl_ids || !tbl_len || tbl_k < 1)) {
        bm::set_error("engine: buddy method needs a buddy table per layer");
        return BM_ECONFIG;
    }
    g->buf_elems = (int64_t)(c->act == BM_ACT_SWIGLU ? 3 : 2) * c->d * c->f;
    g->buf_bytes = (size_t)g->buf_elems * (c->fp32_weights ? 4 : 2);
    g->reserve = std::min(E - g->cap, c->max_batch * k);
    g->S = c->staging > 0 ? c->staging : g->reserve + g->cap;
    if (g->S < g->reserve) {
        bm::set_error("engine: staging (%d) below the on-demand reserve (%d)", g->S, g->reserve);
        return BM_ECONFIG;
    }
    g->Ssh = c->num_shared > 0 ? c->num_shared : 0;
    g->nbufs = L * (g->cap + g->Ssh) + g->S;
    g->host_mirror.resize(L);
    for (int l = 0; l < L; ++l) g->host_mirror[l] = static_cast<const uint8_t *>(host_mirror[l]);
    g->coded = c->fetch_codec == 1;
    if (c->fetch_codec != 0 && !(g->coded && !c->fp32_weights)) {
        bm::set_error("engine: fetch_codec %d unsupported (0 raw, 1 exponent-coded bf16)", c->fetch_codec);
        return BM_ECONFIG;
    }
    if (g->coded) {  // validate every layer image, size the staging ring by the largest piece
        const int cnt = E + (c->num_shared > 0 ? c->num_shared : 0);
        for (int l = 0; l < L; ++l) {
            const auto *lh = reinterpret_cast<const bm_xfer_layer_header *>(g->host_mirror[l]);
            if (lh->magic != 0x314C5842u || (int)lh->count != cnt || lh->raw_bytes != g->buf_bytes) {
                bm::set_error("engine: layer %d mirror is not a coded image of %d experts x %zu bytes", l, cnt,
                              g->buf_bytes);
                return BM_ECONFIG;
            }
            for (int e = 0; e < cnt; ++e) {
                const bm_xfer_blob_header *bh = g->blob_of(l, e);
                if (bh->magic != 0x31435842u || bh->n_values * 2 != g->buf_bytes) {
                    bm::set_error("engine: layer %d expert %d blob is corrupt", l, e);
                    return BM_ECONFIG;
                }
                for (uint32_t p = 0; p < bh->n_pieces; ++p)
                    g->ring_slot_bytes = std::max<size_t>(g->ring_slot_bytes, bh->piece_off[p + 1] - bh->piece_off[p]);
            }
        }
    }
    g->gate_w = gate_w;
    g->gate_b = gate_b;
    g->tbl_ids = tbl_ids;
    g->tbl_len = tbl_len;
    g->tau.assign(tau_host, tau_host + L);
    // control plane
    std::vector<int32_t> init((size_t)L * std::max(g->cap, 1), -1);
    if (initial_host) memcpy(init.data(), initial_host, (size_t)L * g->cap * sizeof(int32_t));
    ENG_TRY(bm_cache_create(L, E, g->cap, c->policy, init.data(), static_freq_host, c->load_ms, c->hit_ms,
                            c->prefetch_ms, c->expert_bytes, &g->cache));
    // data plane
    ENG_CUDA(cudaMalloc(&g->arena, (size_t)g->nbufs * g->buf_bytes));
    g->device_bytes += (int64_t)g->nbufs * (int64_t)g->buf_bytes;
    g->bufs.resize(g->nbufs);
    for (int b = 0; b < g->nbufs; ++b) g->bufs[b].dev = g->arena + (size_t)b * g->buf_bytes;
    for (int b = g->nbufs - 1; b >= 0; --b) g->free_list.push_back(b);
    g->phys.assign(L, std::vector<int>(E, -1));
    g->ready.assign(L, std::vector<cudaEvent_t>(E, nullptr));
    g->ready_pending.assign(L, std::vector<uint8_t>(E, 0));
    g->ready_stream.assign(L, std::vector<cudaStream_t>(E, nullptr));
    g->buf_ev.assign(g->nbufs, nullptr);
    for (int b = 0; b < g->nbufs; ++b) ENG_CUDA(cudaEventCreateWithFlags(&g->buf_ev[b], cudaEventDisableTiming));
    ENG_TRY(g->stall_ev.init());
    ENG_TRY(g->copy_ev.init());
    g->layer_done.assign(L, nullptr);
    for (int l = 0; l < L; ++l) {
        for (int e = 0; e < E; ++e) ENG_CUDA(cudaEventCreateWithFlags(&g->ready[l][e], cudaEventDisableTiming));
        ENG_CUDA(cudaEventCreateWithFlags(&g->layer_done[l], cudaEventDisableTiming));
    }
    // spin-wait on the plan readback: the host round trip is on the critical path
    ENG_CUDA(cudaEventCreateWithFlags(&g->plan_ev, cudaEventDisableTiming));
    ENG_CUDA(cudaStreamCreateWithFlags(&g->cap_stream, cudaStreamNonBlocking));
    if (const char *ev = getenv("BMOE_GRAPHS")) g->use_graphs = atoi(ev) != 0;
    if (const char *ev = getenv("BMOE_OVERLAP")) g->overlap_fetch = atoi(ev) != 0;
    if (const char *ev = getenv("BMOE_SPLIT_FETCHED")) g->split_fetched = atoi(ev) != 0;  // A/B switch
    if (const char *ev = getenv("BMOE_FUSE_COMBINE")) g->fuse_combine = atoi(ev) != 0;  // A/B switch
    if (const char *ev = getenv("BMOE_DECODE_NARROW")) g->decode_narrow = atoi(ev);       // A/B switch
    if (g->cfg.fp32_weights) g->fuse_combine = false;  // the fp32 parity path keeps K5 separate
    ENG_CUDA(cudaStreamCreateWithFlags(&g->copy_stream, cudaStreamNonBlocking));
    ENG_CUDA(cudaStreamCreateWithFlags(&g->prefetch_stream, cudaStreamNonBlocking));
    if (g->coded) {
        int lo = 0, hi = 0;
        ENG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        for (Ring *r : {&g->ring_copy, &g->ring_prefetch}) {
            ENG_CUDA(cudaStreamCreateWithPriority(&r->dec, cudaStreamNonBlocking, hi));
            for (int j = 0; j < kRingSlots; ++j) {
                ENG_CUDA(cudaMalloc(&r->slot[j], g->ring_slot_bytes));
                g->device_bytes += (int64_t)g->ring_slot_bytes;
                ENG_CUDA(cudaEventCreateWithFlags(&r->copied[j], cudaEventDisableTiming));
                ENG_CUDA(cudaEventCreateWithFlags(&r->decoded[j], cudaEventDisableTiming));
            }
        }
    }
    // initial residents: synchronous upload
    std::vector<uint8_t> mask(E);
    for (int l = 0; l < L; ++l) {
        ENG_TRY(bm_cache_snapshot(g->cache, l, mask.data(), nullptr));
        for (int e = 0; e < E; ++e) {
            if (!mask[e]) continue;
            int b;
            ENG_TRY(g->alloc_buffer(&b));
            ENG_TRY(g->upload(l, e, b));
            g->phys[l][e] = b;
        }
    }
    // shared experts: permanent buffers, outside the budget
    g->shared_buf.assign((size_t)L * g->Ssh, -1);
    for (int l = 0; l < L; ++l)
        for (int sx = 0; sx < g->Ssh; ++sx) {
            int b;
            ENG_TRY(g->alloc_buffer(&b));
            ENG_TRY(g->upload(l, E + sx, b));
            g->shared_buf[(size_t)l * g->Ssh + sx] = b;
        }
    // workspaces
    const int64_t Bm = c->max_batch;
    const int Et = E + g->Ssh, kt = k + g->Ssh;
    g->r_max = bm_permute_rows_max(Bm, kt, Et, 16);
    g->r_max = (g->r_max + 15) / 16 * 16;
    ENG_TRY(g->dmalloc(&g->logits, Bm * E));
    ENG_TRY(g->dmalloc(&g->probs, Bm * k));
    ENG_TRY(g->dmalloc(&g->tae, Bm));
    ENG_TRY(g->dmalloc(&g->margin, Bm));
    ENG_TRY(g->dmalloc(&g->delta, 1));
    ENG_TRY(g->dmalloc(&g->used, Bm));
    const size_t pb = bm_engine::plan_bytes(Bm, k) + 64;
    ENG_TRY(g->dmalloc(&g->plan_dev, pb));
    ENG_TRY(g->hmalloc(&g->plan_host, pb));
    if (const char *ev = getenv("BMOE_ZERO_COPY")) g->zero_copy = atoi(ev) != 0;
    if (g->zero_copy) {  // pinned allocations are mapped (portable, UVA): their device-side addresses
        void *pd = nullptr;
        if (cudaHostGetDevicePointer(&pd, g->plan_host, 0) == cudaSuccess)
            g->plan_host_dev = static_cast<uint8_t *>(pd);
        else
            cudaGetLastError();
    }
    ENG_TRY(g->dmalloc(&g->h_int, (size_t)Bm * g->d));
    const int words = (E + 31) / 32;
    g->beta_word = (words + 1) & ~1;  // 8-byte aligned f64 after the bitmap
    g->bm_stride = g->beta_word + 2;
    ENG_TRY(g->dmalloc(&g->bm_dev_all, (size_t)L * g->bm_stride));
    ENG_TRY(g->hmalloc(&g->bm_host_all, (size_t)L * g->bm_stride));
    g->rng = c->rng;
    ENG_TRY(g->beta_ctl.init(c->pcie_budget_bytes, (double)c->expert_bytes, c->beta));
    ENG_TRY(g->dmalloc(&g->bo_dev_all, (size_t)L * 3 * Et));
    ENG_TRY(g->hmalloc(&g->bo_host_all, (size_t)L * 3 * Et));
    ENG_TRY(g->dmalloc(&g->count_a, Et));
    ENG_TRY(g->dmalloc(&g->count_b, Et));
    ENG_TRY(g->dmalloc(&g->count_bc, Et));
    ENG_TRY(g->dmalloc(&g->count_c, Et));
    for (int l = 0; l < L; ++l) {
        g->bm_dev_l.push_back(g->bm_dev_all + (size_t)l * g->bm_stride);
        g->bm_host_l.push_back(g->bm_host_all + (size_t)l * g->bm_stride);
        if (g->plan_host_dev) {
            void *pd = nullptr;
            ENG_CUDA(cudaHostGetDevicePointer(&pd, g->bm_host_l.back(), 0));
            g->bm_hostdev_l.push_back(static_cast<uint32_t *>(pd));
        }
        g->bo_dev_l.push_back(g->bo_dev_all + (size_t)l * 3 * Et);
        g->bo_host_l.push_back(g->bo_host_all + (size_t)l * 3 * Et);
    }
    ENG_TRY(g->dmalloc(&g->count, Et));
    ENG_TRY(g->dmalloc(&g->offset, Et + 1));
    ENG_TRY(g->dmalloc(&g->row_token, g->r_max + 16));
    ENG_TRY(g->dmalloc(&g->slot_row, Bm * kt));
    g->perm_scratch_elems = bm_permute_scratch_elems(Bm, kt, Et);
    ENG_TRY(g->dmalloc(&g->perm_scratch, (size_t)std::max<int64_t>(g->perm_scratch_elems, 1)));
    if (g->Ssh) {
        ENG_TRY(g->dmalloc(&g->exec_ext, Bm * kt));
        ENG_TRY(g->dmalloc(&g->kind_ext, Bm * kt));
        ENG_TRY(g->dmalloc(&g->probs_ext, Bm * kt));
    }
    ENG_TRY(g->dmalloc(&g->y_perm, (size_t)g->r_max * g->d));
    if (c->fp32_weights) {
        ENG_TRY(g->dmalloc(reinterpret_cast<float **>(&g->x_perm), (size_t)g->r_max * g->d));
        ENG_TRY(g->dmalloc(&g->h_ws, (size_t)g->r_max * g->f));
    } else {
        ENG_TRY(g->dmalloc(reinterpret_cast<uint16_t **>(&g->x_perm), (size_t)g->r_max * g->d));
        ENG_CUDA(cudaMemset(g->x_perm, 0, (size_t)g->r_max * g->d * 2));
        g->ffn_ws_bytes = bm_expert_ffn_bf16_workspace(Et, g->d, g->f, g->r_max, c->n_tile);
        ENG_TRY(g->dmalloc(reinterpret_cast<uint8_t **>(&g->ffn_ws), (size_t)g->ffn_ws_bytes));
        ENG_CUDA(cudaMemset(g->ffn_ws, 0, (size_t)g->ffn_ws_bytes));  // self-cleaning counters start at zero
    }
    g->prev_counts.assign(L, std::vector<int32_t>(E, 0));
    g->mask_tmp.assign(E, 0);
    g->stats = bm_engine_stats{};  // the initial uploads are not part of any step
    return BM_OK;
}

extern "C" int bm_engine_create(const bm_engine_config *cfg, const void *const *host_mirror, const float *gate_w,
                                const float *gate_b, const int32_t *tbl_ids, const int32_t *tbl_len, int32_t tbl_k,
                                const double *tau_host, const int32_t *initial_host, const double *static_freq_host,
                                bm_engine **out) {
    if (!cfg || !host_mirror || !gate_w || !gate_b || !tau_host || !out) {
        bm::set_error("bm_engine_create: null argument");
        return BM_EINVAL;
    }
    bm_engine *g = new bm_engine();
    int rc = engine_init(g, cfg, host_mirror, gate_w, gate_b, tbl_ids, tbl_len, tbl_k, tau_host, initial_host,
                         static_freq_host);
    if (rc != BM_OK) {
        g->release();
        delete g;
        return rc;
    }
    *out = g;
    return BM_OK;
}

extern "C" void bm_engine_destroy(bm_engine *e) {
    if (!e) return;
    cudaDeviceSynchronize();
    e->release();
    delete e;
}

extern "C" int bm_engine_step(bm_engine *e, float *h, int64_t B, const int32_t *tokens_host, bm_stream_t stream) {
    if (!e || !h || B < 1 || B > e->cfg.max_batch) {
        bm::set_error("bm_engine_step: bad arguments (B=%lld)", (long long)B);
        return BM_EINVAL;
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // the layers run on an engine-owned copy of h so captured graphs see fixed addresses
    ENG_CUDA(cudaMemcpyAsync(e->h_int, h, (size_t)B * e->d * sizeof(float), cudaMemcpyDeviceToDevice, s));
    for (int l = 0; l < e->L; ++l) ENG_TRY(e->layer_step(l, e->h_int, B, tokens_host, s));
    ENG_CUDA(cudaMemcpyAsync(h, e->h_int, (size_t)B * e->d * sizeof(float), cudaMemcpyDeviceToDevice, s));
    if (bm_kernel_timing_enabled()) {  // read the timed graph launches before their next replay
        ENG_CUDA(cudaStreamSynchronize(s));
        ENG_TRY(bm::ffn::ffn_timing_harvest());
    }
    e->stats.tokens += B;
    return BM_OK;
}

extern "C" int bm_engine_stats_get(bm_engine *e, bm_engine_stats *out, int32_t reset) {
    if (!e || !out) return BM_EINVAL;
    double st = 0.0, cp = 0.0;
    ENG_TRY(e->stall_ev.drain(&st));
    ENG_TRY(e->copy_ev.drain(&cp));
    e->stats.stall_ms += st;
    e->stats.copy_ms += cp;
    ENG_TRY(bm_cache_now(e->cache, &e->stats.sim_now_ms));
    e->stats.beta = e->beta_ctl.beta;
    *out = e->stats;
    if (reset) e->stats = bm_engine_stats{};
    return BM_OK;
}

extern "C" bm_cache *bm_engine_cache(bm_engine *e) { return e ? e->cache : nullptr; }

extern "C" int bm_engine_set_copy_timing(bm_engine *e, int32_t enable) {
    if (!e) return BM_EINVAL;
    e->copy_timing = enable != 0;
    return BM_OK;
}

extern "C" int bm_engine_set_trace(bm_engine *e, int32_t enable) {
    if (!e) return BM_EINVAL;
    e->tracing = enable != 0;
    e->tr_layer.clear();
    e->tr_B.clear();
    e->tr_topk.clear();
    e->tr_exec.clear();
    e->tr_kind.clear();
    e->tr_allowed.clear();
    e->tr_batch_ok.clear();
    e->tr_bitmap.clear();
    e->tr_tae.clear();
    e->tr_margin.clear();
    e->tr_delta.clear();
    return BM_OK;
}

extern "C" int bm_engine_trace_gates(const bm_engine *e, double *tae_host, double *margin_host, double *delta_host) {
    if (!e) return BM_EINVAL;
    if (tae_host && !e->tr_tae.empty()) memcpy(tae_host, e->tr_tae.data(), e->tr_tae.size() * sizeof(double));
    if (margin_host && !e->tr_margin.empty())
        memcpy(margin_host, e->tr_margin.data(), e->tr_margin.size() * sizeof(double));
    if (delta_host && !e->tr_delta.empty())
        memcpy(delta_host, e->tr_delta.data(), e->tr_delta.size() * sizeof(double));
    return BM_OK;
}

extern "C" int bm_engine_set_psi(bm_engine *e, const double *tbl_w, double eta, double kappa, int32_t use_local_logit,
                                 const int32_t *partition_of, double hop) {
    if (!e || eta < 0.0 || kappa < 0.0) {
        bm::set_error("bm_engine_set_psi: bad arguments");
        return BM_EINVAL;
    }
    const bool on = eta != 0.0 || kappa != 0.0;
    if (on && (!tbl_w || e->cfg.method != BM_METHOD_BUDDY)) {
        bm::set_error("bm_engine_set_psi: Psi ordering needs the buddy method and table weights");
        return BM_ECONFIG;
    }
    // captured graphs hold the old remap arguments: drop them
    for (auto *m : {&e->g_pre}) {
        for (auto &kv : *m)
            if (kv.second.second) cudaGraphExecDestroy(kv.second.second);
        m->clear();
    }
    e->psi = on;
    e->tbl_w = tbl_w;
    e->eta = eta;
    e->kappa = kappa;
    e->use_local_logit = use_local_logit;
    e->partition_of = partition_of;
    e->hop = hop;
    return BM_OK;
}

extern "C" int bm_engine_trace_size(const bm_engine *e, int64_t *records, int64_t *tokens) {
    if (!e || !records || !tokens) return BM_EINVAL;
    *records = (int64_t)e->tr_layer.size();
    *tokens = (int64_t)e->tr_allowed.size();
    return BM_OK;
}

extern "C" int bm_engine_trace_get(const bm_engine *e, int32_t *layer, int32_t *B, uint32_t *bitmaps, uint8_t *batch_ok,
                                   int32_t *topk, uint8_t *allowed, int32_t *executed, uint8_t *kind) {
    if (!e) return BM_EINVAL;
    auto cp = [](auto &v, auto *dst) {
        if (dst && !v.empty()) memcpy(dst, v.data(), v.size() * sizeof(v[0]));
    };
    cp(e->tr_layer, layer);
    cp(e->tr_B, B);
    cp(e->tr_bitmap, bitmaps);
    cp(e->tr_batch_ok, batch_ok);
    cp(e->tr_topk, topk);
    cp(e->tr_allowed, allowed);
    cp(e->tr_exec, executed);
    cp(e->tr_kind, kind);
    return BM_OK;
}

extern "C" int64_t bm_engine_device_bytes(const bm_engine *e) { return e ? e->device_bytes : 0; }

extern "C" int bm_host_alloc(int64_t bytes, void **out) {
    if (!out || bytes <= 0) return BM_EINVAL;
    ENG_CUDA(cudaHostAlloc(out, (size_t)bytes, cudaHostAllocPortable));
    return BM_OK;
}

extern "C" int bm_host_register(void *p, int64_t bytes, int32_t read_only) {
    if (!p || bytes <= 0) return BM_EINVAL;
    unsigned flags = cudaHostRegisterPortable | (read_only ? cudaHostRegisterReadOnly : 0u);
    ENG_CUDA(cudaHostRegister(p, (size_t)bytes, flags));
    return BM_OK;
}

extern "C" int bm_host_unregister(void *p) {
    if (p) ENG_CUDA(cudaHostUnregister(p));
    return BM_OK;
}

extern "C" int bm_host_free(void *p) {
    if (p) ENG_CUDA(cudaFreeHost(p));
    return BM_OK;
}

extern "C" int bm_memcpy(void *dst, const void *src, int64_t bytes, bm_stream_t stream) {
    ENG_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDefault, reinterpret_cast<cudaStream_t>(stream)));
    return BM_OK;
}
