// The paper's Random baseline (substitution.random_plan, substitution.py:227-248)
// as host code over numpy's own random stream, so the engine's Random arm makes
// the same draws as the reference's run_simulation(method="random")
// (harness.py:299-300, 358-359).
//
// The reference draws with np.random.Generator(PCG64).integers(0, n), n = the
// pool size. That is, for the record of what is replicated here:
//   - PCG64 = PCG XSL-RR 128/64: state <- state * M + inc (mod 2^128), then
//     output = rotr64(hi(state) ^ lo(state), state >> 122);
//   - next_uint32 hands out the low half of a 64-bit output and keeps the high
//     half for the next call (has_uint32 / uinteger in the bit generator state);
//   - integers(0, n) with n-1 = 0 returns 0 without a draw; otherwise Lemire's
//     nearly-divisionless bounded draw on 32-bit outputs (n <= 2^32):
//     m = u32 * n; reject while (m mod 2^32) < (2^32 - n) mod n; result m >> 32.
// Seeding (SeedSequence -> initial state) stays in numpy on the Python side;
// the caller passes the bit generator state in and gets the advanced state back.
#include <stdint.h>
#include <string.h>

#include "../../include/bmoe.h"

namespace bm {
void set_error(const char *fmt, ...);
}

namespace {

typedef unsigned __int128 u128;

struct Pcg64 {
    u128 state, inc;
    bool has32;
    uint32_t u32;

    uint64_t next64() {
        const u128 mult = ((u128)0x2360ED051FC65DA4ull << 64) | (u128)0x4385DF649FCCF645ull;
        state = state * mult + inc;
        const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
        const unsigned rot = (unsigned)(state >> 122);
        const uint64_t x = hi ^ lo;
        return (x >> rot) | (x << ((64u - rot) & 63u));
    }
    uint32_t next32() {
        if (has32) {
            has32 = false;
            return u32;
        }
        const uint64_t v = next64();
        has32 = true;
        u32 = (uint32_t)(v >> 32);
        return (uint32_t)v;
    }
    // Generator.integers(0, n), n >= 1, n <= 2^32
    uint64_t below(uint64_t n) {
        const uint64_t rng = n - 1;
        if (rng == 0) return 0;
        if (rng == 0xFFFFFFFFull) return next32();
        const uint32_t excl = (uint32_t)n;
        uint64_t m = (uint64_t)next32() * excl;
        uint32_t left = (uint32_t)m;
        if (left < excl) {
            const uint32_t threshold = (uint32_t)((UINT32_MAX - (uint32_t)rng) % excl);
            while (left < threshold) {
                m = (uint64_t)next32() * excl;
                left = (uint32_t)m;
            }
        }
        return m >> 32;
    }
};

Pcg64 load(const bm_pcg64 *s) {
    Pcg64 g;
    g.state = ((u128)s->state_hi << 64) | s->state_lo;
    g.inc = ((u128)s->inc_hi << 64) | s->inc_lo;
    g.has32 = s->has_uint32 != 0;
    g.u32 = s->uinteger;
    return g;
}

void store(const Pcg64 &g, bm_pcg64 *s) {
    s->state_hi = (uint64_t)(g.state >> 64);
    s->state_lo = (uint64_t)g.state;
    s->inc_hi = (uint64_t)(g.inc >> 64);
    s->inc_lo = (uint64_t)g.inc;
    s->has_uint32 = g.has32 ? 1 : 0;
    s->uinteger = g.u32;
}

}  // namespace

namespace bm {

// One batch of random plans in token order (the reference builds the plans of
// a batch-layer with one shared generator, harness.py:358-359). resident_bits:
// the residency snapshot as a u32 bitmap. Returns BM_OK or BM_EINVAL.
int random_plan_batch(const int32_t *topk, int64_t B, int64_t k, const uint32_t *resident_bits, int64_t E,
                      bm_pcg64 *rng, int32_t *executed, uint8_t *kind, int32_t *used) {
    if (E < 1 || E > 4096 || k < 1) {
        set_error("bm_random_plan: bad shape (E=%lld, k=%lld)", (long long)E, (long long)k);
        return BM_EINVAL;
    }
    Pcg64 g = load(rng);
    int32_t pool[4096];
    uint8_t assigned[4096];
    for (int64_t b = 0; b < B; ++b) {
        const int32_t *t = topk + b * k;
        memset(assigned, 0, (size_t)E);
        for (int64_t s = 0; s < k; ++s) {
            if (t[s] < 0 || t[s] >= E) {
                store(g, rng);
                set_error("bm_random_plan: expert id %d outside [0, %lld)", t[s], (long long)E);
                return BM_EINVAL;
            }
            assigned[t[s]] = 1;
        }
        int32_t u = 0;
        for (int64_t s = 0; s < k; ++s) {
            const int orig = t[s];
            int32_t *ex = executed + b * k + s;
            uint8_t *kd = kind + b * k + s;
            *ex = orig;
            if ((resident_bits[orig >> 5] >> (orig & 31)) & 1u) {
                *kd = BM_KIND_KEPT;
                continue;
            }
            // pool = flatnonzero(mask) minus the token's assigned set, ascending
            int n = 0;
            for (int e = 0; e < E; ++e)
                if (((resident_bits[e >> 5] >> (e & 31)) & 1u) && !assigned[e]) pool[n++] = e;
            if (n == 0) {
                *kd = BM_KIND_ONDEMAND;
                continue;
            }
            const int j = pool[g.below((uint64_t)n)];
            *ex = j;
            *kd = BM_KIND_SUBSTITUTED;
            assigned[j] = 1;
            ++u;
        }
        if (used) used[b] = u;
    }
    store(g, rng);
    return BM_OK;
}

}  // namespace bm

extern "C" int bm_random_plan(const int32_t *topk_host, int64_t B, int64_t k, const uint8_t *mask_host, int64_t E,
                              bm_pcg64 *rng_host, int32_t *executed_host, uint8_t *kind_host, int32_t *used_host) {
    if ((B > 0 && (!topk_host || !executed_host || !kind_host)) || !mask_host || !rng_host || B < 0) {
        bm::set_error("bm_random_plan: null argument");
        return BM_EINVAL;
    }
    if (E < 1 || E > 4096) {
        bm::set_error("bm_random_plan: E=%lld outside [1, 4096]", (long long)E);
        return BM_EINVAL;
    }
    uint32_t bits[128] = {};
    for (int64_t e = 0; e < E; ++e)
        if (mask_host[e]) bits[e >> 5] |= 1u << (e & 31);
    return bm::random_plan_batch(topk_host, B, k, bits, E, rng_host, executed_host, kind_host, used_host);
}

extern "C" int bm_pcg64_integers(bm_pcg64 *rng_host, int64_t n, int64_t count, int64_t *out_host) {
    if (!rng_host || (count > 0 && !out_host) || n < 1 || n > (int64_t)1 << 32 || count < 0) {
        bm::set_error("bm_pcg64_integers: bad arguments (n=%lld)", (long long)n);
        return BM_EINVAL;
    }
    Pcg64 g = load(rng_host);
    for (int64_t i = 0; i < count; ++i) out_host[i] = (int64_t)g.below((uint64_t)n);
    store(g, rng_host);
    return BM_OK;
}
