// Expert-cache control plane: an exact C++ replica of the reference's
// residency state machine and transfer clock (memtier.py:72-300) and the
// next-layer predictor (harness.py:209-218). Host-only; the HBM data plane
// (engine.cpp) follows its decisions.
#include <math.h>
#include <stdarg.h>
#include <string.h>

#include <algorithm>
#include <utility>
#include <vector>

#include "../../include/bmoe.h"

namespace bm {
void set_error(const char *fmt, ...);
}

namespace {

struct Layer {
    int layer = 0, E = 0, cap = 0, policy = 0;
    std::vector<uint8_t> mask;
    std::vector<int64_t> last_use;
    std::vector<double> freq;
    std::vector<double> stat;
    std::vector<uint8_t> unused_prefetch;
    std::vector<std::pair<double, int>> pending;  // (ready_ms, expert), issue order
    int64_t tick = 0;
    int64_t waste = 0;
    int resident = 0;

    // LRU recency list of the residents, least recent first. Every touch and
    // prefetch insert takes a fresh tick, so last_use is unique among
    // residents and the list head is exactly memtier's argmin victim: O(1)
    // instead of a scan over E per miss (a 2048-token prefill chunk replays
    // ~10^4 misses per layer).
    std::vector<int> prv, nxt;
    std::vector<uint8_t> linked;
    int head = -1, tail = -1;
    void lru_unlink(int e) {
        if (!linked[e]) return;
        if (prv[e] >= 0) nxt[prv[e]] = nxt[e]; else head = nxt[e];
        if (nxt[e] >= 0) prv[nxt[e]] = prv[e]; else tail = prv[e];
        linked[e] = 0;
    }
    void lru_to_tail(int e) {
        lru_unlink(e);
        prv[e] = tail;
        nxt[e] = -1;
        if (tail >= 0) nxt[tail] = e; else head = e;
        tail = e;
        linked[e] = 1;
    }
    void init_lists(int n) {
        prv.assign(n, -1);
        nxt.assign(n, -1);
        linked.assign(n, 0);
        head = tail = -1;
    }

    void touch(int e) {  // memtier.py:156-160
        ++tick;
        last_use[e] = tick;
        freq[e] += 1.0;
        unused_prefetch[e] = 0;
        if (mask[e]) lru_to_tail(e);
    }
    int victim() const {  // memtier.py:162-170: argmin over residents, ties -> lowest id
        if (policy == BM_POLICY_LRU) return head;
        int best = -1;
        for (int e = 0; e < E; ++e) {
            if (!mask[e]) continue;
            if (best < 0) {
                best = e;
                continue;
            }
            bool lt;
            if (policy == BM_POLICY_LRU) lt = last_use[e] < last_use[best];
            else if (policy == BM_POLICY_LFU) lt = freq[e] < freq[best];
            else lt = stat[e] < stat[best];
            if (lt) best = e;
        }
        return best;
    }
    int insert(int e, bool via_prefetch) {  // memtier.py:172-195
        if (cap == 0) return -1;
        int v = -1;
        if (!mask[e]) {
            if (resident >= cap) {
                v = victim();
                mask[v] = 0;
                lru_unlink(v);
                --resident;
                if (unused_prefetch[v]) {
                    ++waste;
                    unused_prefetch[v] = 0;
                }
                freq[v] = 0.0;
            }
            mask[e] = 1;
            ++resident;
        }
        if (via_prefetch) {
            freq[e] = 0.0;
            ++tick;
            last_use[e] = tick;
            unused_prefetch[e] = 1;
            lru_to_tail(e);
        } else {
            touch(e);
        }
        return v;
    }
};

}  // namespace

struct bm_cache {
    std::vector<Layer> layers;
    double now = 0.0, free_at = 0.0;  // SimClock.now, PcieChannel.free_at
    double load_ms = 9.5, hit_ms = 0.0, prefetch_ms = 0.0;
    int64_t expert_bytes = 0;
    std::vector<bm_event> events;

    double acquire(double t, double dur) {  // memtier.py:78-82
        double start = t > free_at ? t : free_at;
        double done = start + dur;
        free_at = done;
        return done;
    }
    void log(double t, int kind, int layer, int token, int expert, int64_t bytes, double stall) {
        events.push_back(bm_event{t, kind, layer, token, expert, bytes, stall});
    }
    // memtier.py:217-254
    bm_event access(Layer &L, int e, bool substituted_away, int token) {
        const double start = now;
        if (L.mask[e]) {
            L.touch(e);
            now += hit_ms;
            log(start, BM_EV_HIT, L.layer, token, e, 0, hit_ms);
            return events.back();
        }
        if (substituted_away) {
            now += hit_ms;
            log(start, BM_EV_MISS_SUBSTITUTED, L.layer, token, e, 0, hit_ms);
            return events.back();
        }
        const double done = acquire(start, load_ms);
        const double stall = done - start;
        now = done;
        const int v = L.insert(e, false);
        log(start, BM_EV_MISS_ONDEMAND, L.layer, token, e, expert_bytes, stall);
        bm_event ev = events.back();
        if (v >= 0) log(now, BM_EV_EVICT, L.layer, -1, v, 0, 0.0);
        return ev;
    }
};

extern "C" int bm_cache_create(int32_t num_layers, int32_t num_experts, int32_t capacity, int32_t policy,
                               const int32_t *initial_host, const double *static_freq_host, double expert_load_ms,
                               double hit_ms, double prefetch_ms, int64_t expert_bytes, bm_cache **out) {
    if (!out || num_layers < 1 || num_experts < 1 || capacity < 0 || capacity > num_experts) {
        bm::set_error("bm_cache_create: capacity must be in [0, num_experts]");
        return BM_ECONFIG;
    }
    if (policy < BM_POLICY_LRU || policy > BM_POLICY_FREQ_STATIC) {
        bm::set_error("bm_cache_create: unknown eviction policy %d", policy);
        return BM_ECONFIG;
    }
    if (policy == BM_POLICY_FREQ_STATIC && !static_freq_host) {
        bm::set_error("freq_static policy needs profiling frequencies");
        return BM_ECONFIG;
    }
    if (expert_load_ms < 0 || hit_ms < 0 || prefetch_ms < 0 || expert_bytes <= 0) {
        bm::set_error("bm_cache_create: bad cost model");
        return BM_ECONFIG;
    }
    bm_cache *c = new bm_cache();
    c->load_ms = expert_load_ms;
    c->hit_ms = hit_ms;
    c->prefetch_ms = prefetch_ms;
    c->expert_bytes = expert_bytes;
    c->layers.resize(num_layers);
    for (int l = 0; l < num_layers; ++l) {
        Layer &L = c->layers[l];
        L.layer = l;
        L.E = num_experts;
        L.cap = capacity;
        L.policy = policy;
        L.mask.assign(num_experts, 0);
        L.last_use.assign(num_experts, 0);
        L.freq.assign(num_experts, 0.0);
        L.unused_prefetch.assign(num_experts, 0);
        L.init_lists(num_experts);
        if (static_freq_host) L.stat.assign(static_freq_host + (size_t)l * num_experts,
                                            static_freq_host + (size_t)(l + 1) * num_experts);
        // initial residents are touched in ascending id order (memtier.py:138-140)
        if (initial_host && capacity > 0) {
            std::vector<int> init;
            for (int i = 0; i < capacity; ++i) {
                int e = initial_host[(size_t)l * capacity + i];
                if (e >= 0) init.push_back(e);
            }
            std::sort(init.begin(), init.end());
            for (int e : init) {
                if (e >= num_experts || L.mask[e]) {
                    delete c;
                    bm::set_error("bm_cache_create: bad initial resident %d", e);
                    return BM_EINVAL;
                }
                L.mask[e] = 1;
                ++L.resident;
                L.touch(e);
            }
        }
    }
    *out = c;
    return BM_OK;
}

extern "C" void bm_cache_destroy(bm_cache *c) { delete c; }

static int check_layer(const bm_cache *c, int32_t layer) {
    if (!c || layer < 0 || layer >= (int)c->layers.size()) {
        bm::set_error("bm_cache: layer %d out of range", layer);
        return BM_EINVAL;
    }
    return BM_OK;
}

extern "C" int bm_cache_access(bm_cache *c, int32_t layer, int32_t expert, int32_t mode, int32_t token,
                               bm_event *ev_out_host) {
    if (int rc = check_layer(c, layer)) return rc;
    Layer &L = c->layers[layer];
    if (mode != 0 && mode != 1) {
        bm::set_error("unknown access mode %d", mode);
        return BM_EINVAL;
    }
    if (expert < 0 || expert >= L.E) {
        bm::set_error("expert id out of range");
        return BM_EINVAL;
    }
    bm_event ev = c->access(L, expert, mode == 1, token);
    if (ev_out_host) *ev_out_host = ev;
    return BM_OK;
}

extern "C" int bm_cache_apply_plan(bm_cache *c, int32_t layer, int64_t B, int64_t k, const int32_t *tokens_host,
                                   const int32_t *topk_host, const int32_t *executed_host, const uint8_t *kind_host,
                                   int64_t *out_host) {
    if (int rc = check_layer(c, layer)) return rc;
    Layer &L = c->layers[layer];
    int64_t executed_slots = 0, ondemand = 0, subs = 0, bytes = 0;
    for (int64_t b = 0; b < B; ++b) {
        const int tok = tokens_host ? tokens_host[b] : (int)b;
        for (int64_t s = 0; s < k; ++s) {
            const int orig = topk_host[b * k + s], ex = executed_host[b * k + s];
            const int kd = kind_host[b * k + s];
            if (orig < 0 || orig >= L.E || ex < 0 || ex >= L.E) {
                bm::set_error("plan references expert outside the layer");
                return BM_EINVAL;
            }
            if (kd == BM_KIND_DROPPED) {  // harness.py:367-369
                c->log(c->now, BM_EV_DROP, layer, tok, orig, 0, 0.0);
                continue;
            }
            ++executed_slots;
            if (kd == BM_KIND_SUBSTITUTED) {  // harness.py:371-373
                ++subs;
                c->access(L, orig, true, tok);
                // the stand-in was resident at snapshot time but an earlier
                // token of this batch may have evicted it: then it misses too
                bm_event ev = c->access(L, ex, false, tok);
                if (ev.kind == BM_EV_MISS_ONDEMAND) {
                    ++ondemand;
                    bytes += ev.bytes;
                }
            } else {
                bm_event ev = c->access(L, ex, false, tok);
                if (ev.kind == BM_EV_MISS_ONDEMAND) {
                    ++ondemand;
                    bytes += ev.bytes;
                }
            }
        }
    }
    if (out_host) {
        out_host[0] = executed_slots;
        out_host[1] = ondemand;
        out_host[2] = subs;
        out_host[3] = bytes;
    }
    return BM_OK;
}

extern "C" int bm_cache_prefetch(bm_cache *c, int32_t layer, const int32_t *experts_host, int64_t n) {
    if (int rc = check_layer(c, layer)) return rc;
    Layer &L = c->layers[layer];  // memtier.py:257-280
    for (int64_t i = 0; i < n; ++i) {
        const int e = experts_host[i];
        if (e < 0 || e >= L.E) {
            bm::set_error("expert id out of range");
            return BM_EINVAL;
        }
        if (L.mask[e]) continue;
        bool inflight = false;
        for (auto &p : L.pending) inflight |= (p.second == e);
        if (inflight) continue;
        const double done = c->acquire(c->now, c->prefetch_ms);
        L.pending.emplace_back(done, e);
        c->log(c->now, BM_EV_PREFETCH_ISSUE, L.layer, -1, e, 0, 0.0);
    }
    return BM_OK;
}

extern "C" int bm_cache_settle(bm_cache *c, int32_t layer) {
    if (int rc = check_layer(c, layer)) return rc;
    Layer &L = c->layers[layer];  // memtier.py:283-300
    std::vector<std::pair<double, int>> remaining;
    for (auto &p : L.pending) {
        if (p.first <= c->now) {
            const int v = L.insert(p.second, true);
            c->log(p.first, BM_EV_PREFETCH_COMPLETE, L.layer, -1, p.second, c->expert_bytes, 0.0);
            if (v >= 0) c->log(p.first, BM_EV_EVICT, L.layer, -1, v, 0, 0.0);
        } else {
            remaining.push_back(p);
        }
    }
    L.pending.swap(remaining);
    return BM_OK;
}

extern "C" int bm_cache_advance(bm_cache *c, double ms) {
    if (!c) return BM_EINVAL;
    if (ms < 0) {  // memtier.py:90-92
        bm::set_error("clock cannot move backwards");
        return BM_EINVARIANT;
    }
    c->now += ms;
    return BM_OK;
}

extern "C" int bm_cache_now(const bm_cache *c, double *now_host) {
    if (!c || !now_host) return BM_EINVAL;
    *now_host = c->now;
    return BM_OK;
}

extern "C" int bm_cache_snapshot(const bm_cache *c, int32_t layer, uint8_t *mask_host, uint32_t *bitmap_host) {
    if (int rc = check_layer(c, layer)) return rc;
    const Layer &L = c->layers[layer];
    if (mask_host) memcpy(mask_host, L.mask.data(), L.E);
    if (bitmap_host) {
        const int words = (L.E + 31) / 32;
        for (int w = 0; w < words; ++w) bitmap_host[w] = 0;
        for (int e = 0; e < L.E; ++e)
            if (L.mask[e]) bitmap_host[e >> 5] |= 1u << (e & 31);
    }
    return BM_OK;
}

extern "C" int bm_cache_predict(const bm_cache *c, int32_t layer, const int32_t *counts_host, int32_t *out_host,
                                int64_t *n_out_host) {
    if (int rc = check_layer(c, layer)) return rc;
    const Layer &L = c->layers[layer];  // harness.py:209-218
    std::vector<std::pair<int, int>> nz;
    for (int e = 0; e < L.E; ++e)
        if (counts_host[e] > 0) nz.emplace_back(-counts_host[e], e);
    int64_t n = 0;
    if (!nz.empty()) {
        const int m = std::max(0, L.cap - (int)nz.size());
        std::sort(nz.begin(), nz.end());
        for (int i = 0; i < m && i < (int)nz.size(); ++i) out_host[n++] = nz[i].second;
    }
    *n_out_host = n;
    return BM_OK;
}

extern "C" int64_t bm_cache_num_events(const bm_cache *c) { return c ? (int64_t)c->events.size() : 0; }

extern "C" int bm_cache_events(const bm_cache *c, int64_t start, int64_t n, bm_event *out_host) {
    if (!c || start < 0 || start + n > (int64_t)c->events.size()) {
        bm::set_error("bm_cache_events: range out of bounds");
        return BM_EINVAL;
    }
    if (n > 0) memcpy(out_host, c->events.data() + start, (size_t)n * sizeof(bm_event));
    return BM_OK;
}

extern "C" void bm_cache_clear_events(bm_cache *c) {
    if (c) c->events.clear();
}

extern "C" int bm_cache_layer_state(const bm_cache *c, int32_t layer, int64_t *last_use_host, double *freq_host,
                                    int64_t *scalars_host) {
    if (int rc = check_layer(c, layer)) return rc;
    const Layer &L = c->layers[layer];
    if (last_use_host) memcpy(last_use_host, L.last_use.data(), L.E * sizeof(int64_t));
    if (freq_host) memcpy(freq_host, L.freq.data(), L.E * sizeof(double));
    if (scalars_host) {
        int64_t unused = 0;
        for (int e = 0; e < L.E; ++e) unused += (L.unused_prefetch[e] && L.mask[e]) ? 1 : 0;
        scalars_host[0] = L.tick;
        scalars_host[1] = (int64_t)L.pending.size();
        scalars_host[2] = L.waste;
        scalars_host[3] = unused;
    }
    return BM_OK;
}

extern "C" int bm_cache_set_clock(bm_cache *c, double now, double free_at) {
    if (!c) return BM_EINVAL;
    c->now = now;
    c->free_at = free_at;
    return BM_OK;
}

extern "C" int bm_cache_get_clock(const bm_cache *c, double *now_host, double *free_at_host) {
    if (!c || !now_host || !free_at_host) return BM_EINVAL;
    *now_host = c->now;
    *free_at_host = c->free_at;
    return BM_OK;
}

extern "C" int bm_cache_set_costs(bm_cache *c, double expert_load_ms, double hit_ms, double prefetch_ms,
                                  int64_t expert_bytes) {
    if (!c || expert_load_ms < 0 || hit_ms < 0 || prefetch_ms < 0 || expert_bytes <= 0) {
        bm::set_error("bm_cache_set_costs: bad cost model");
        return BM_ECONFIG;
    }
    c->load_ms = expert_load_ms;
    c->hit_ms = hit_ms;
    c->prefetch_ms = prefetch_ms;
    c->expert_bytes = expert_bytes;
    return BM_OK;
}

extern "C" int bm_cache_insert(bm_cache *c, int32_t layer, int32_t expert, int32_t via_prefetch, int32_t *victim_host) {
    if (int rc = check_layer(c, layer)) return rc;
    Layer &L = c->layers[layer];
    if (expert < 0 || expert >= L.E) {
        bm::set_error("expert id out of range");
        return BM_EINVAL;
    }
    const int v = L.insert(expert, via_prefetch != 0);
    if (L.resident > L.cap) {  // memtier.py:193-194
        bm::set_error("residency exceeded capacity");
        return BM_EINVARIANT;
    }
    if (victim_host) *victim_host = v;
    return BM_OK;
}

extern "C" int bm_cache_pending(const bm_cache *c, int32_t layer, double *done_host, int32_t *expert_host,
                                int64_t cap) {
    if (int rc = check_layer(c, layer)) return rc;
    const Layer &L = c->layers[layer];
    for (int64_t i = 0; i < (int64_t)L.pending.size() && i < cap; ++i) {
        done_host[i] = L.pending[i].first;
        expert_host[i] = L.pending[i].second;
    }
    return BM_OK;
}
