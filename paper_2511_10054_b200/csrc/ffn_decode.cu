// K4 decode: the bf16 grouped expert FFN for decode-width token tiles
// (n_tile <= 64) as ONE cooperative launch per call (see the kernel comment).
// Decode is weight-streaming: every executed expert's W1/W3/W2 must cross
// HBM once per layer-step while the token count per expert is tiny, so the
// weights are the M=128 operand ("swap-AB"), stored in HBM already in the
// UMMA-tiled, 128B-swizzled image (bm_pack_expert_bf16) so each pipeline
// stage is ONE contiguous bulk copy of KPS k-blocks of every matrix; one
// persistent CTA per SM walks an equal share of the (tile, k-step) space.
// Warp roles (256 threads): w0 producer (bulk copies), w1 MMA issuer (one
// thread; precomputed descriptors), w2 TMEM allocator, w4-7 epilogue.
#include "combine.cuh"
#include "ffn_common.cuh"

namespace bm {
namespace ffn {

// ------------------------------------------------ fused decode FFN (one launch)
// GEMM1 (W1|W3, or Win) -> SwiGLU / tanh -> H -> GEMM2 (W2, or Wout) ->
// y_perm in ONE persistent launch for decode-width tiles (n_tile <= 64):
//  * split (stream-K) tiles are reduced inside the kernel by the CTA that
//    owns their first k-steps (see fused_epilogue), summing in fixed CTA
//    order, so the result is bit-identical to the separate fixup kernel;
//  * one grid barrier separates the phases (H complete). The launch is
//    cooperative, so all CTAs (one per SM) are co-resident;
//  * while waiting at the barrier the producer already streams the first
//    stages of W2 (they do not depend on H) and completes each of those
//    stages with its H part once the barrier opens.
// The counters are self-cleaning (the reducer resets them), so the
// workspace is zeroed once, when it is allocated.

constexpr int kSmemFused = 216 * 1024;

struct Geom {
    uint32_t base, stage_bytes, bsz, b_off;  // b_off: B part offset inside a stage (max A bytes)
    int stages;
    uint32_t full0, empty0, tfull0, tempty0;
};

template <int NMAT, int KPS>
__device__ void fused_produce(const GemmParams &P, const Sched &s, const Geom &gm, int &stage, uint32_t &phase,
                              long long it0, long long it1, int spt, uint64_t pol,
                              const unsigned long long *gate, unsigned long long gate_target, int prefetch,
                              unsigned long long *gate_stamp = nullptr) {
    constexpr uint32_t kA = (uint32_t)(KPS * NMAT) * kATileBytes;
    const int mtiles = P.M / kBM;
    int cur = -1;
    const uint8_t *a_tile = nullptr, *b_tile = nullptr;
    uint32_t bbytes = 0;
    auto locate = [&](long long it, int &st) {
        const int tile = (int)(it / spt);
        st = (int)(it - (long long)tile * spt);
        if (tile != cur) {
            cur = tile;
            const TileInfo ti = decode_tile(s, tile, mtiles, P.n_tile);
            const int buf = P.buf_of_expert[ti.e];
            a_tile = P.arena + (long long)buf * P.buf_bytes + P.mat_off + (long long)ti.mtile * spt * kA;
            b_tile = P.b_planes + (long long)ti.row0 * 128;
            bbytes = (uint32_t)ti.n * 128u;
        }
    };
    auto issue_b = [&](int stg, int st) {
        const uint32_t sB = gm.base + (uint32_t)stg * gm.stage_bytes + gm.b_off;
        const uint32_t fb = gm.full0 + 8 * stg;
#pragma unroll
        for (int i = 0; i < KPS; ++i)
            ptx::bulk_load(sB + i * gm.bsz, b_tile + (long long)(st * KPS + i) * P.b_plane_bytes, bbytes, fb);
    };
    long long it = it0;
    if (gate && !prefetch) {
        while (ptx::ld_acquire_gpu_u64(gate) < gate_target) __nanosleep(32);
        if (gate_stamp) *gate_stamp = ptx::globaltimer();
        ptx::fence_proxy_async_global();
    } else if (gate) {
        // the weights do not depend on H: A parts of the first stages now ...
        const long long pre_end = min(it1, it0 + (long long)gm.stages);
        const int stage0 = stage;
        for (; it < pre_end; ++it) {
            int st;
            locate(it, st);
            ptx::mbar_wait(gm.empty0 + 8 * stage, phase ^ 1u);
            const uint32_t fb = gm.full0 + 8 * stage;
            ptx::mbar_expect_tx_only(fb, kA);
            ptx::bulk_load_hint(gm.base + (uint32_t)stage * gm.stage_bytes, a_tile + (long long)st * kA, kA, fb, pol);
            if (++stage == gm.stages) {
                stage = 0;
                phase ^= 1u;
            }
        }
        // ... then the H parts once every CTA has finished phase 1
        while (ptx::ld_acquire_gpu_u64(gate) < gate_target) __nanosleep(32);
        if (gate_stamp) *gate_stamp = ptx::globaltimer();
        ptx::fence_proxy_async_global();
        int stg = stage0;
        for (long long j = it0; j < pre_end; ++j) {
            int st;
            locate(j, st);
            ptx::mbar_expect_tx(gm.full0 + 8 * stg, (uint32_t)KPS * bbytes);  // the stage's arrive
            issue_b(stg, st);
            if (++stg == gm.stages) stg = 0;
        }
    }
    for (; it < it1; ++it) {
        int st;
        locate(it, st);
        ptx::mbar_wait(gm.empty0 + 8 * stage, phase ^ 1u);
        const uint32_t fb = gm.full0 + 8 * stage;
        ptx::mbar_expect_tx(fb, kA + (uint32_t)KPS * bbytes);
        ptx::bulk_load_hint(gm.base + (uint32_t)stage * gm.stage_bytes, a_tile + (long long)st * kA, kA, fb, pol);
        issue_b(stage, st);
        if (++stage == gm.stages) {
            stage = 0;
            phase ^= 1u;
        }
    }
}

// GEMM2 producer under per-expert H readiness: the A part (W2, independent of
// H) of up to `stages` iterations is issued ahead while the next stage's expert
// is not ready yet; a stage's H part goes out once h_ready[e] is complete.
template <int KPS>
__device__ void fused_produce_ready(const GemmParams &P, const Sched &s, const Geom &gm, int &stage, uint32_t &phase,
                                    long long it0, long long it1, int spt, uint64_t pol, const int *h_ready,
                                    int mtiles1, unsigned long long *gate_stamp) {
    constexpr uint32_t kA = (uint32_t)KPS * kATileBytes;
    const int mtiles = P.M / kBM;
    struct Cur {  // one cursor's tile cache (the tile decode and buffer lookup once per tile)
        int tile = -1, e = 0, need = 0;
        const uint8_t *a = nullptr, *b = nullptr;
        uint32_t bbytes = 0;
    };
    auto locate = [&](Cur &c, long long it, int &st) {
        const int tile = (int)(it / spt);
        st = (int)(it - (long long)tile * spt);
        if (tile != c.tile) {
            c.tile = tile;
            const TileInfo ti = decode_tile(s, tile, mtiles, P.n_tile);
            c.e = ti.e;
            c.need = mtiles1 * ti.nch;
            c.a = P.arena + (long long)P.buf_of_expert[ti.e] * P.buf_bytes + P.mat_off + (long long)ti.mtile * spt * kA;
            c.b = P.b_planes + (long long)ti.row0 * 128;
            c.bbytes = (uint32_t)ti.n * 128u;
        }
    };
    Cur ca, cb;
    long long ia = it0, ib = it0;  // next iteration whose A part / H part is issued
    int stage_a = stage;
    uint32_t phase_a = phase;
    int ready_e = -1;
    bool stamped = false;
    while (ib < it1) {
        int st;
        locate(cb, ib, st);
        bool rdy = cb.e == ready_e ||
                   ptx::ld_acquire_gpu(reinterpret_cast<const unsigned *>(h_ready + cb.e)) >= (unsigned)cb.need;
        if (!rdy && ia < it1 && ia - ib < gm.stages) {  // stream W2 ahead meanwhile
            int sta;
            locate(ca, ia, sta);
            ptx::mbar_wait(gm.empty0 + 8 * stage_a, phase_a ^ 1u);
            const uint32_t fb = gm.full0 + 8 * stage_a;
            ptx::mbar_expect_tx_only(fb, kA);
            ptx::bulk_load_hint(gm.base + (uint32_t)stage_a * gm.stage_bytes, ca.a + (long long)sta * kA, kA, fb, pol);
            if (++stage_a == gm.stages) {
                stage_a = 0;
                phase_a ^= 1u;
            }
            ++ia;
            continue;
        }
        while (!rdy) {
            __nanosleep(32);
            rdy = ptx::ld_acquire_gpu(reinterpret_cast<const unsigned *>(h_ready + cb.e)) >= (unsigned)cb.need;
        }
        if (cb.e != ready_e) ptx::fence_proxy_async_global();  // H (generic writes) -> bulk-copy reads
        ready_e = cb.e;
        if (gate_stamp && !stamped) {
            *gate_stamp = ptx::globaltimer();
            stamped = true;
        }
        const uint32_t fb = gm.full0 + 8 * stage;
        if (ia == ib) {  // A part not issued ahead: both parts now
            ptx::mbar_wait(gm.empty0 + 8 * stage, phase ^ 1u);
            ptx::mbar_expect_tx(fb, kA + (uint32_t)KPS * cb.bbytes);
            ptx::bulk_load_hint(gm.base + (uint32_t)stage * gm.stage_bytes, cb.a + (long long)st * kA, kA, fb, pol);
            if (++stage_a == gm.stages) {
                stage_a = 0;
                phase_a ^= 1u;
            }
            ++ia;
        } else {
            ptx::mbar_expect_tx(fb, (uint32_t)KPS * cb.bbytes);  // the stage's arrive
        }
        const uint32_t sB = gm.base + (uint32_t)stage * gm.stage_bytes + gm.b_off;
#pragma unroll
        for (int i = 0; i < KPS; ++i)
            ptx::bulk_load(sB + i * gm.bsz, cb.b + (long long)(st * KPS + i) * P.b_plane_bytes, cb.bbytes, fb);
        if (++stage == gm.stages) {
            stage = 0;
            phase ^= 1u;
        }
        ++ib;
    }
}

template <int NMAT, int KPS>
__device__ void fused_mma(const GemmParams &P, const Sched &s, const Geom &gm, int &stage, uint32_t &phase, int &acc,
                          uint32_t &acc_phase, long long it0, long long it1, int spt, uint32_t tmem_base,
                          unsigned long long *first_full = nullptr) {
    const int mtiles = P.M / kBM;
    const uint64_t desc0 = ptx::sw128_desc(gm.base);
    const uint64_t stage_d = gm.stage_bytes >> 4, bsz_d = gm.bsz >> 4, boff_d = gm.b_off >> 4;
    long long it = it0;
    while (it < it1) {
        const int tile = (int)(it / spt);
        const int st_end = (int)min((long long)spt, it1 - (long long)tile * spt);
        const TileInfo ti = decode_tile(s, tile, mtiles, P.n_tile);
        const uint32_t idesc = ptx::idesc_bf16_f32(kBM, (uint32_t)ti.n);
        ptx::mbar_wait(gm.tempty0 + 8 * acc, acc_phase ^ 1u);
        ptx::tc_fence_after();
        const uint32_t d0 = tmem_base + (uint32_t)acc * 256u;
        const uint32_t d1 = d0 + (uint32_t)P.n_tile;
        uint32_t accum = 0;
        for (int st = (int)(it - (long long)tile * spt); st < st_end; ++st, ++it) {
            ptx::mbar_wait(gm.full0 + 8 * stage, phase);
            ptx::tc_fence_after();
            if (first_full) {
                *first_full = ptx::globaltimer();
                first_full = nullptr;
            }
            const uint64_t a = desc0 + (uint64_t)stage * stage_d;
            const uint64_t b = a + boff_d;
#pragma unroll
            for (int i = 0; i < KPS; ++i) {
                const uint64_t bi = b + (uint64_t)i * bsz_d;
#pragma unroll
                for (int kk = 0; kk < kBK / 16; ++kk) {
                    ptx::mma_bf16(d0, a + (uint64_t)((i * NMAT) * (kATileBytes >> 4) + 2 * kk), bi + 2 * kk, idesc,
                                  accum);
                    if (NMAT == 2)
                        ptx::mma_bf16(d1, a + (uint64_t)((i * NMAT + 1) * (kATileBytes >> 4) + 2 * kk), bi + 2 * kk,
                                      idesc, accum);
                    accum = 1u;
                }
            }
            ptx::mma_commit(gm.empty0 + 8 * stage);
            if (++stage == gm.stages) {
                stage = 0;
                phase ^= 1u;
            }
        }
        ptx::mma_commit(gm.tfull0 + 8 * acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1u;
    }
}

// Split tiles: the CTA owning a tile's FIRST k-steps (c0) processes them at
// the end of its range, after every other contributor (c0+1..c1) has
// processed its share at the start of its own. So c0 reduces: it keeps its
// accumulator in TMEM, waits on the tile's arrival counter (normally already
// complete), adds the other slots in CTA order -- ((0 + own) + s_c0+1) + ...,
// the fixup kernel's order -- and finishes the tile. The others publish an
// fp32 partial slot and arrive. No partial write, fence or atomic sits on
// the reducer's critical path.
template <int NMAT>
__device__ void fused_epilogue(const GemmParams &P, const Sched &s, const Geom &gm, int *arrive, int &acc,
                               uint32_t &acc_phase, long long base, long long T, int G, int slot_off, int cta, int spt,
                               uint32_t tmem_base, int q, unsigned lane, int *h_ready = nullptr,
                               unsigned long long *tr = nullptr) {
    if (cta >= G) return;
    const int mtiles = P.M / kBM;
    const long long it0 = base + range_start(cta, T, G), it1 = base + range_start(cta + 1, T, G);
    const long long slot_elems = 2LL * P.n_tile * kBM;
    const int m_local = q * 32 + (int)lane;
    long long it = it0;
    while (it < it1) {
        const int tile = (int)(it / spt);
        const long long tile_end = (long long)(tile + 1) * spt;
        const bool whole = it == (long long)tile * spt && tile_end <= it1;
        const bool reducer = !whole && it == (long long)tile * spt;  // owns the first k-steps, not the last
        it = min(tile_end, it1);
        const TileInfo ti = decode_tile(s, tile, mtiles, P.n_tile);
        ptx::mbar_wait(gm.tfull0 + 8 * acc, acc_phase);
        ptx::tc_fence_after();
        if (tr && m_local == 0) tr[8] = ptx::globaltimer();  // last accumulator ready
        const uint32_t tbase = tmem_base + (uint32_t)acc * 256u + ((uint32_t)(q * 32) << 16);
        if (whole) {
            for (int c0 = 0; c0 < ti.n; c0 += 16) {
                float g[16], u[16];
                ptx::tmem_ld16(tbase + (uint32_t)c0, g);
                if (NMAT == 2) ptx::tmem_ld16(tbase + (uint32_t)(P.n_tile + c0), u);
                finish16<NMAT>(P, ti, c0, q, lane, g, u);
            }
        } else if (reducer) {
            const int c1 = cta_of((long long)(tile + 1) * spt - 1 - base, T, G);
            if (m_local == 0) {
                while (ptx::ld_acquire_gpu(reinterpret_cast<const unsigned *>(arrive + tile)) < (unsigned)(c1 - cta))
                    __nanosleep(32);
                arrive[tile] = 0;  // every contributor has arrived: reset for the next launch
                if (tr) tr[9] = ptx::globaltimer();
            }
            ptx::named_bar_sync(1, 128);
            for (int cc = 0; cc < ti.n; cc += 16) {
                float g[16], u[16], o[16];
                ptx::tmem_ld16(tbase + (uint32_t)cc, o);
#pragma unroll
                for (int j = 0; j < 16; ++j) g[j] = 0.f + o[j];
                if (NMAT == 2) {
                    ptx::tmem_ld16(tbase + (uint32_t)(P.n_tile + cc), o);
#pragma unroll
                    for (int j = 0; j < 16; ++j) u[j] = 0.f + o[j];
                }
                // the partials of kGrp contributors are loaded together (one L2 round trip),
                // then added in CTA order: the sum is the same as one slot at a time
                constexpr int kGrp = NMAT == 2 ? 2 : 4;
                for (int c0 = cta + 1; c0 <= c1; c0 += kGrp) {
                    float pg[kGrp][16], pu[kGrp][NMAT == 2 ? 16 : 1];
#pragma unroll
                    for (int x = 0; x < kGrp; ++x) {
                        if (c0 + x > c1) break;
                        const float *src = P.partials + ((long long)tile + c0 + x + slot_off) * slot_elems;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            pg[x][j] = __ldcg(src + (long long)(cc + j) * kBM + m_local);
                            if (NMAT == 2) pu[x][j] = __ldcg(src + (long long)(P.n_tile + cc + j) * kBM + m_local);
                        }
                    }
#pragma unroll
                    for (int x = 0; x < kGrp; ++x) {
                        if (c0 + x > c1) break;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            g[j] += pg[x][j];
                            if (NMAT == 2) u[j] += pu[x][j];
                        }
                    }
                }
                finish16<NMAT>(P, ti, cc, q, lane, g, u);
            }
        } else {
            float *dst = P.partials + ((long long)tile + cta + slot_off) * slot_elems;
#pragma unroll
            for (int m = 0; m < NMAT; ++m)
                for (int c0 = 0; c0 < ti.n; c0 += 16) {
                    float v[16];
                    ptx::tmem_ld16(tbase + (uint32_t)(m * P.n_tile + c0), v);
#pragma unroll
                    for (int j = 0; j < 16; ++j) dst[((long long)m * P.n_tile + c0 + j) * kBM + m_local] = v[j];
                }
        }
        ptx::tc_fence_before();
        __syncwarp();
        if (lane == 0) ptx::mbar_arrive(gm.tempty0 + 8 * acc);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1u;
        if (h_ready && (whole || reducer)) {  // this tile's H rows are written: publish them
            ptx::fence_proxy_async_global();
            __threadfence();
            ptx::named_bar_sync(1, 128);
            if (m_local == 0) atomicAdd(h_ready + ti.e, 1);
        }
        if (!whole && !reducer) {  // publish the partial, then arrive
            __threadfence();
            ptx::named_bar_sync(1, 128);
            if (m_local == 0) atomicAdd(arrive + tile, 1);
        }
    }
}

// The call's work as phases: with ng expert groups (contiguous in the
// schedule) the order is G1(0), G1(1), G2(0), G1(2), G2(1), ..., G2(ng-1), so
// each group's GEMM2 follows the NEXT group's GEMM1 and finds its H (per-
// expert readiness) already written instead of waiting at the end of the
// whole GEMM1 stream. Each phase is its own stream-K range over the CTAs
// (iterations [base, base + T)); its split-tile partial slots are offset by
// g * G so the overlapping phases of one GEMM never share a slot.
struct Phase {
    bool g2;
    int g, G, slot_off;
    long long base, T;
};
__device__ __forceinline__ Phase phase_at(int p, int ng, const Sched &s, int mtiles1, int mtiles2, int spt1,
                                          int spt2, int Gn, int min_iters) {
    Phase ph;
    if (p == 0) {
        ph.g2 = false;
        ph.g = 0;
    } else if (p == 2 * ng - 1) {
        ph.g2 = true;
        ph.g = ng - 1;
    } else {
        const int k = p - 1;
        ph.g2 = (k & 1) != 0;
        ph.g = ph.g2 ? (k - 1) / 2 : k / 2 + 1;
    }
    const int a0 = ph.g * s.n_act / ng, a1 = (ph.g + 1) * s.n_act / ng;
    const int mt = ph.g2 ? mtiles2 : mtiles1, spt = ph.g2 ? spt2 : spt1;
    ph.base = (long long)mt * s.chunk_prefix[a0] * spt;
    ph.T = (long long)mt * (s.chunk_prefix[a1] - s.chunk_prefix[a0]) * spt;
    // a tiny phase (a few small experts) on fewer CTAs, each with >= min_iters k-steps: every
    // CTA streams more, but no tile is split over many CTAs (a split reducer adds every
    // contributor's partial tile)
    ph.G = (int)min((long long)Gn, max(min(ph.T, 1LL), ph.T / max(1, min_iters)));  // default 2 (A/B: profiles/r2s_mi_ab.jsonl)
    ph.slot_off = ph.g * Gn;
    return ph;
}

template <int NMAT1, int KPS1, int KPS2>
__global__ void __launch_bounds__(kThreads, 1) ffn_fused_kernel(const __grid_constant__ FusedParams fp) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ Sched sched;
    __shared__ __align__(8) uint64_t bars[64];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    // phase trace (diagnostics): 0 entry, 1 setup done, 2 GEMM1 loads issued, 3 GEMM1 MMAs committed,
    // 4 GEMM1 epilogue done, 5 barrier seen by the producer, 6 GEMM2 epilogue done, 7 exit
    unsigned long long *tr = fp.trace ? fp.trace + (size_t)blockIdx.x * kTracePts : nullptr;
    if (tr && threadIdx.x == 0) tr[0] = ptx::globaltimer();
    if (fp.span && threadIdx.x == 0) atomicMin(fp.span, ptx::globaltimer());
    const GemmParams &P1 = fp.g[0];
    const GemmParams &P2 = fp.g[1];
    const int n_tile = P1.n_tile;
    // launched with programmatic stream serialization (fp.pdl): nothing below reads
    // what the preceding kernel writes before this wait
    if (fp.pdl && warp == 0) ptx::grid_dep_wait();
    // no barrier instance of this launch can complete before this CTA arrives,
    // so the count read here rounds down to the launch's base (see FusedParams);
    // issued ahead of the schedule's loads so the two round trips overlap
    unsigned long long bar0 = 0;
    if (threadIdx.x == 0) bar0 = *reinterpret_cast<volatile unsigned long long *>(fp.grid_bar);
    if (warp == 0) build_sched_warp(sched, P1.count, P1.offset, P1.E, n_tile);
    if (threadIdx.x == 0) bar0 = bar0 / (unsigned long long)gridDim.x * (unsigned long long)gridDim.x;
    // per-expert H readiness: this launch's counter array (see FusedParams)
    __shared__ int *h_ready_sh;
    if (fp.h_ready && threadIdx.x == 32) {  // warp 1 lane 0 (warp 0 builds the schedule)
        if (fp.pdl) ptx::grid_dep_wait();
        const unsigned long long n = *reinterpret_cast<volatile unsigned long long *>(fp.launch_count) /
                                     (unsigned long long)gridDim.x;
        h_ready_sh = fp.h_ready + (n & 1ull) * kMaxE;
        if (blockIdx.x == 0)  // the array launch n - 1 used is next launch's: clear it
            for (int e = 0; e < P1.E; ++e) fp.h_ready[((n + 1ull) & 1ull) * kMaxE + e] = 0;
    }

    constexpr uint32_t kA1 = (uint32_t)(KPS1 * NMAT1) * kATileBytes, kA2 = (uint32_t)KPS2 * kATileBytes;
    constexpr uint32_t kAmax = kA1 > kA2 ? kA1 : kA2;
    constexpr int kKmax = KPS1 > KPS2 ? KPS1 : KPS2;
    Geom gm;
    gm.base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    gm.bsz = ((uint32_t)n_tile * 128u + 1023u) & ~1023u;
    gm.b_off = kAmax;
    gm.stage_bytes = kAmax + (uint32_t)kKmax * gm.bsz;
    gm.stages = min(16, (int)((kSmemFused - 1024) / gm.stage_bytes));
    gm.full0 = ptx::smem_u32(&bars[0]);
    gm.empty0 = ptx::smem_u32(&bars[16]);
    gm.tfull0 = ptx::smem_u32(&bars[32]);
    gm.tempty0 = ptx::smem_u32(&bars[34]);

    if (warp == 1 && lane == 0) {
        for (int s = 0; s < gm.stages; ++s) {
            ptx::mbar_init(gm.full0 + 8 * s, 1);
            ptx::mbar_init(gm.empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(gm.tfull0 + 8 * a, 1);
            ptx::mbar_init(gm.tempty0 + 8 * a, 4);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc(ptx::smem_u32(&tmem_base_sh), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = tmem_base_sh;
    int *const h_ready = fp.h_ready ? h_ready_sh : nullptr;
    if (tr && threadIdx.x == 0) tr[1] = ptx::globaltimer();

    const int cta = blockIdx.x, Gn = gridDim.x;
    const int spt1 = P1.K / (kBK * KPS1), spt2 = P2.K / (kBK * KPS2);
    const int mtiles1 = P1.M / kBM, mtiles2 = P2.M / kBM;
    // expert groups (see phase_at): only with per-expert readiness, at most one per expert
    // and only while every GEMM1 phase keeps >= group_min_iters k-steps per CTA (short phases
    // split every tile across many CTAs: measured slower for calls of many small experts)
    const long long T1all = (long long)total_tiles(sched, mtiles1) * spt1;
    const int ng = h_ready ? max(1, (int)min((long long)min(fp.groups, sched.n_act),
                                             fp.group_min_iters > 0 ? T1all / ((long long)fp.group_min_iters * Gn)
                                                                    : (long long)kMaxGroups))
                           : 1;
    const int n_ph = 2 * ng;
    const int last_g1 = ng == 1 ? 0 : n_ph - 3;  // the phase index of G1(ng - 1)

    if (warp == 0 && lane == 0) {
        const uint64_t pol = ptx::policy_evict_first();  // weights stream through once
        int stage = 0;
        uint32_t phase = 0;
        for (int p = 0; p < n_ph; ++p) {
            const Phase ph = phase_at(p, ng, sched, mtiles1, mtiles2, spt1, spt2, Gn, fp.min_iters);
            if (cta < ph.G) {
                const long long i0 = ph.base + range_start(cta, ph.T, ph.G);
                const long long i1 = ph.base + range_start(cta + 1, ph.T, ph.G);
                if (!ph.g2)
                    fused_produce<NMAT1, KPS1>(P1, sched, gm, stage, phase, i0, i1, spt1, pol, nullptr, 0, 0);
                else if (h_ready)
                    fused_produce_ready<KPS2>(P2, sched, gm, stage, phase, i0, i1, spt2, pol, h_ready, mtiles1,
                                              tr && ph.g == 0 ? tr + 5 : nullptr);
                else
                    fused_produce<1, KPS2>(P2, sched, gm, stage, phase, i0, i1, spt2, pol, fp.grid_bar,
                                           bar0 + (unsigned long long)Gn, fp.prefetch_w2, tr ? tr + 5 : nullptr);
            }
            if (tr && p == last_g1) tr[2] = ptx::globaltimer();
        }
    } else if (warp == 1 && lane == 0) {
        int stage = 0, acc = 0;
        uint32_t phase = 0, acc_phase = 0;
        bool first_g2 = true;
        for (int p = 0; p < n_ph; ++p) {
            const Phase ph = phase_at(p, ng, sched, mtiles1, mtiles2, spt1, spt2, Gn, fp.min_iters);
            if (cta < ph.G) {
                const long long i0 = ph.base + range_start(cta, ph.T, ph.G);
                const long long i1 = ph.base + range_start(cta + 1, ph.T, ph.G);
                if (!ph.g2) {
                    fused_mma<NMAT1, KPS1>(P1, sched, gm, stage, phase, acc, acc_phase, i0, i1, spt1, tmem_base);
                } else {
                    fused_mma<1, KPS2>(P2, sched, gm, stage, phase, acc, acc_phase, i0, i1, spt2, tmem_base,
                                       tr && first_g2 ? tr + 10 : nullptr);
                    first_g2 = false;
                }
            }
            if (tr && p == last_g1) tr[3] = ptx::globaltimer();
        }
        if (tr) tr[11] = ptx::globaltimer();
    } else if (warp >= 4) {
        const int q = warp - 4;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int p = 0; p < n_ph; ++p) {
            const Phase ph = phase_at(p, ng, sched, mtiles1, mtiles2, spt1, spt2, Gn, fp.min_iters);
            if (!ph.g2)
                fused_epilogue<NMAT1>(P1, sched, gm, fp.arrive, acc, acc_phase, ph.base, ph.T, ph.G, ph.slot_off, cta,
                                      spt1, tmem_base, q, lane, h_ready, tr);
            else
                fused_epilogue<1>(P2, sched, gm, fp.arrive + fp.tile_cap, acc, acc_phase, ph.base, ph.T, ph.G,
                                  ph.slot_off, cta, spt2, tmem_base, q, lane);
            if (p == last_g1) {
                // all of this CTA's H is written: publish it (to the bulk-copy proxy too) and
                // arrive at barrier 1 (GEMM2 waits on it without per-expert readiness)
                if (tr && q == 0 && lane == 0) tr[4] = ptx::globaltimer();
                ptx::fence_proxy_async_global();
                __threadfence();
                ptx::named_bar_sync(1, 128);
                if (q == 0 && lane == 0) atomicAdd(fp.grid_bar, 1ull);
            }
        }
        if (tr && q == 0 && lane == 0) tr[6] = ptx::globaltimer();
    }
    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc(tmem_base, 512);
    if (fp.h_ready && threadIdx.x == 0) atomicAdd(fp.launch_count, 1ull);  // result unused: a reduction
    if (fp.cmb.B > 0) {
        // K5 (gate-weighted combine + layer_update, in place on h) once every
        // CTA's y tiles are written: a second grid barrier, then token b on CTA
        // b (mod G) with all 256 threads -- combine_kernel's own code and thread
        // count, so h is bit-identical to the separate launch.
        __shared__ CombineShared<float> csh;
        __threadfence();
        __syncthreads();
        if (threadIdx.x == 0) {
            // barrier 2 counts only after barrier 1 has completed, or a fast CTA's second
            // arrival could stand in for a slow CTA's first
            while (ptx::ld_acquire_gpu_u64(fp.grid_bar) < bar0 + (unsigned long long)Gn) __nanosleep(32);
            atomicAdd(fp.grid_bar, 1ull);
            while (ptx::ld_acquire_gpu_u64(fp.grid_bar) < bar0 + 2ull * (unsigned long long)Gn) __nanosleep(32);
        }
        __syncthreads();
        float *hbuf = reinterpret_cast<float *>(smem_raw);
        for (int b = cta; b < fp.cmb.B; b += Gn)
            combine_token<float, 4, true>(b, P2.y_perm, fp.cmb.slot_row, fp.cmb.probs, fp.cmb.kind, fp.cmb.k, P2.M,
                                          fp.cmb.h, fp.cmb.scale, fp.cmb.h, hbuf, csh);
    }
    if (tr && threadIdx.x == 0) tr[7] = ptx::globaltimer();
    if (fp.span) {
        __syncthreads();  // the combine's last stores of this CTA are issued
        if (threadIdx.x == 0) atomicMax(fp.span + 1, ptx::globaltimer());
    }
}

template <int NMAT1, int KPS1, int KPS2>
int launch_fused(const FusedParams &fp, int G, cudaStream_t s) {
    static bool attr = false;
    auto kern = ffn_fused_kernel<NMAT1, KPS1, KPS2>;
    if (!attr) {
        BM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemFused));
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)G);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemFused;
    cfg.stream = s;
    // the grid barrier needs every CTA resident: a cooperative launch guarantees it
    // (BMOE_COOP=0: a plain launch, resident in practice at one CTA per SM);
    // fp.pdl: programmatic stream serialization, so the launch and the prologue
    // (barrier init, TMEM allocation) overlap the preceding kernel
    static const int coop = getenv("BMOE_COOP") ? atoi(getenv("BMOE_COOP")) : 1;
    cudaLaunchAttribute at[2];
    int na = 0;
    if (coop) {
        at[na].id = cudaLaunchAttributeCooperative;
        at[na++].val.cooperative = 1;
    }
    if (fp.pdl) {
        at[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        at[na++].val.programmaticStreamSerializationAllowed = 1;
    }
    cfg.attrs = at;
    cfg.numAttrs = na;
    BM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, fp));
    return BM_OK;
}

template <int NMAT1>
int launch_fused_k(const FusedParams &fp, int kps1, int kps2, int G, cudaStream_t s) {
    if (kps1 == 2) {
        if (kps2 == 4) return launch_fused<NMAT1, 2, 4>(fp, G, s);
        if (kps2 == 2) return launch_fused<NMAT1, 2, 2>(fp, G, s);
        return launch_fused<NMAT1, 2, 1>(fp, G, s);
    }
    if (kps2 == 4) return launch_fused<NMAT1, 1, 4>(fp, G, s);
    if (kps2 == 2) return launch_fused<NMAT1, 1, 2>(fp, G, s);
    return launch_fused<NMAT1, 1, 1>(fp, G, s);
}

// fused-kernel k-blocks per stage: GEMM1 KPS1 in {2,1}, GEMM2 KPS2 in {4,2,1},
// the largest dividing K/64 whose combined stage leaves >= 3 stages
// (>= 2 for the widest tiles) in kSmemFused.
void fused_kps(int nmat1, long long d, long long f, long long n_tile, int *k1, int *k2) {
    const long long bsz = ((n_tile * 128 + 1023) / 1024) * 1024;
    int best1 = 1, best2 = 1;
    // tuning / A-B overrides: BMOE_KPS sets both (as for the unfused GEMMs), BMOE_KPS1/2 each
    int e1 = 0, e2 = 0;
    if (const char *ev = getenv("BMOE_KPS")) e1 = e2 = atoi(ev);
    if (const char *ev = getenv("BMOE_KPS1")) e1 = atoi(ev);
    if (const char *ev = getenv("BMOE_KPS2")) e2 = atoi(ev);
    if ((e1 == 1 || e1 == 2) && (e2 == 1 || e2 == 2 || e2 == 4) && (d / kBK) % e1 == 0 && (f / kBK) % e2 == 0) {
        const long long stage = std::max((long long)e1 * nmat1, (long long)e2) * kATileBytes + std::max(e1, e2) * bsz;
        if ((kSmemFused - 1024) / stage >= 2) {
            *k1 = e1;
            *k2 = e2;
            return;
        }
    }
    for (int a : {2, 1}) {
        if ((d / kBK) % a) continue;
        for (int b : {4, 2, 1}) {
            if ((f / kBK) % b) continue;
            const long long amax = std::max((long long)a * nmat1, (long long)b) * kATileBytes;
            const long long stage = amax + std::max(a, b) * bsz;
            const int want = n_tile <= 32 ? 3 : 2;
            if ((kSmemFused - 1024) / stage >= want) {
                *k1 = a;
                *k2 = b;
                return;
            }
        }
    }
    *k1 = best1;
    *k2 = best2;
}


int launch_fused_dispatch(const FusedParams &fp, int nmat1, int kps1, int kps2, int G, cudaStream_t s) {
    return nmat1 == 2 ? launch_fused_k<2>(fp, kps1, kps2, G, s) : launch_fused_k<1>(fp, kps1, kps2, G, s);
}

}  // namespace ffn
}  // namespace bm
