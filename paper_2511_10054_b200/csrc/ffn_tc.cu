// bf16 grouped expert FFN on 5th-gen tensor cores (sm_100a).
//
// Decode is weight-streaming: every executed expert's W1/W3/W2 must cross
// HBM once per layer-step while the token count per expert is tiny. So the
// weights are the M=128 operand ("swap-AB"), stored in HBM already in the
// UMMA-tiled, 128B-swizzled image (bm_pack_expert_bf16) so each pipeline
// stage is ONE contiguous bulk copy (TMA engine, UBLKCP) of KPS k-blocks of
// every matrix; the permuted tokens are the N operand (16..n_tile columns,
// moved the same way from a pre-swizzled image written by gather_sw128 /
// the GEMM1 fixup); accumulators live in TMEM. One persistent CTA per SM
// walks an equal share of the global (tile, k-step) iteration space
// ("stream-K"), so HBM traffic is balanced over all 148 SMs however many
// experts a step executes. Split tiles are reduced deterministically (fixed
// CTA order, no atomics) by a fixup kernel that also applies SwiGLU / tanh
// and writes GEMM2's B operand in the same swizzled image.
//
// Warp roles (256 threads): w0 producer (bulk copies), w1 MMA issuer (one
// thread; descriptors are precomputed per stage and advanced by compile-time
// offsets — at decode N the MMA *issue* rate, not the math, bounds the weight
// stream), w2 TMEM allocator, w3 idle, w4-7 epilogue (TMEM lane quadrants).
//
// Reference semantics: Expert.__call__ / forward_batch (model.py:85-99,
// 318-340); SwiGLU is the Mixtral/Qwen3/DSV2 expert (no reference oracle).
#include <cuda.h>
#include <cuda_bf16.h>
#include <math.h>
#include <stdlib.h>

#include <algorithm>
#include <mutex>
#include <vector>

#include "common.cuh"
#include "ptx.cuh"

namespace bm {
namespace {

constexpr int kThreads = 256;
constexpr int kBM = 128;                    // weight rows per tile (UMMA M)
constexpr int kBK = 64;                     // K per k-block (one 128-byte swizzle row)
constexpr int kATileBytes = kBM * kBK * 2;  // 16 KB
constexpr int kMaxE = 256;
constexpr int kSmemBudget = 220 * 1024;     // dynamic; static smem (schedule, barriers) comes on top

struct Sched {
    // device-side schedule, identical in every kernel that needs it: the
    // active experts in ascending id order with their row counts, first
    // permuted row and token chunks; expert a's tiles are
    // [mtiles*chunk_prefix[a], mtiles*chunk_prefix[a+1]), m-tile major.
    int n_act;
    int act_e[kMaxE];
    int act_cnt[kMaxE];
    int act_off[kMaxE];
    int act_nch[kMaxE];
    int chunk_prefix[kMaxE + 1];
};

struct GemmParams {
    const int32_t *count;
    const int32_t *offset;
    const int32_t *buf_of_expert;
    int E, M, K, nmat, n_tile, kps;
    const uint8_t *arena;     // expert buffers in the UMMA-tiled layout
    long long buf_bytes;      // bytes per buffer
    long long mat_off;        // byte offset of this GEMM's weight region inside a buffer
    const uint8_t *b_planes;  // [K/64][r_max][128 B]
    long long b_plane_bytes;
    float *partials;          // slot (tile + cta): nmat * n_tile * 128 floats
    int num_ctas;             // launched grid (persistent)
    int mode;                 // epilogue: 0 SwiGLU -> H, 1 tanh -> H, 2 plain -> y_perm
    int fuse;                 // finish wholly-owned tiles in the GEMM epilogue (decode-width tiles)
    int dp;                   // data-parallel tiles (prefill): CTA c owns whole tiles c, c+G, ... (see SegIter)
    int probe;                // diagnostics only (BMOE_PROBE): 1 = skip the MMAs (operand-feed bound), 2 = skip loads
    uint8_t *h_planes;        // GEMM1 output: bf16 SW128 planes [M/64][h_rmax][64]
    int h_rmax;
    float *y_perm;            // GEMM2 output: fp32 [r_max][M]
    long long arena_bytes;    // whole weights arena (the CTA-pair kernel's tensor map spans it)
};

__device__ __forceinline__ int chunks_of(int c, int n_tile) { return (((c + 15) & ~15) + n_tile - 1) / n_tile; }

// Built by warp 0 (the other threads must not touch `s` before the
// following __syncthreads): each lane owns E/32 consecutive experts, so the
// count loads are issued in parallel, and one warp scan places them.
__device__ void build_sched_warp(Sched &s, const int32_t *count, const int32_t *offset, int E, int n_tile) {
    constexpr int kPer = kMaxE / 32;
    const int lane = (int)lane_id();
    const int per = (E + 31) / 32;
    int c[kPer];
    int nact = 0, nch = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {
        const int e = lane * per + i;
        c[i] = (i < per && e < E) ? count[e] : 0;
    }
#pragma unroll
    for (int i = 0; i < kPer; ++i)
        if (c[i] > 0) {
            ++nact;
            nch += chunks_of(c[i], n_tile);
        }
    int a = nact, ch = nch;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int ya = __shfl_up_sync(0xffffffffu, a, o), yc = __shfl_up_sync(0xffffffffu, ch, o);
        if (lane >= o) {
            a += ya;
            ch += yc;
        }
    }
    int ia = a - nact, ic = ch - nch;
#pragma unroll
    for (int i = 0; i < kPer; ++i)
        if (c[i] > 0) {
            const int e = lane * per + i, nc = chunks_of(c[i], n_tile);
            s.act_e[ia] = e;
            s.act_cnt[ia] = c[i];
            s.act_off[ia] = offset[e];
            s.act_nch[ia] = nc;
            s.chunk_prefix[ia] = ic;
            ic += nc;
            ++ia;
        }
    if (lane == 31) {
        s.n_act = a;
        s.chunk_prefix[a] = ch;
    }
}

__device__ __forceinline__ int total_tiles(const Sched &s, int mtiles) { return s.chunk_prefix[s.n_act] * mtiles; }

struct TileInfo {
    int e, mtile, chunk, n;  // n = columns (tokens, padded to 16) of this tile
    int row0;                // first permuted row of the chunk
};

__device__ __forceinline__ TileInfo decode_tile(const Sched &s, int t, int mtiles, int n_tile) {
    int lo = 0, hi = s.n_act - 1;
    while (lo < hi) {  // last a with mtiles * chunk_prefix[a] <= t
        int mid = (lo + hi + 1) >> 1;
        if (s.chunk_prefix[mid] * mtiles <= t) lo = mid; else hi = mid - 1;
    }
    TileInfo ti;
    ti.e = s.act_e[lo];
    const int local = t - s.chunk_prefix[lo] * mtiles;
    const int nch = s.act_nch[lo];
    ti.mtile = local / nch;
    ti.chunk = local % nch;
    const int npad = (s.act_cnt[lo] + 15) & ~15;
    ti.n = min(n_tile, npad - ti.chunk * n_tile);
    ti.row0 = s.act_off[lo] + ti.chunk * n_tile;
    return ti;
}

__device__ __forceinline__ long long range_start(int c, long long T, int G) { return (long long)c * T / G; }


// A CTA's work as segments (tile, k-steps [st0, st1)).
//  stream-K (decode): one contiguous range [it0, it1) of the (tile, k-step)
//    space, so every SM streams an equal share of the weights;
//  data-parallel (prefill, dp): whole tiles cta, cta+G, ... Tiles are
//    m-tile major / token-chunk minor, so the CTAs running at the same time
//    work on the chunks of the same weight m-tiles and read each weight
//    block from DRAM once (the other chunks hit L2), and every tile is
//    finished in the GEMM's own epilogue (no partials, no fixup kernel).
struct SegIter {
    bool dp;
    int cta, G, ntiles, spt, seg;
    long long it, it1;
    __device__ SegIter(bool dp_, int cta_, int G_, int ntiles_, int spt_, long long it0_, long long it1_)
        : dp(dp_), cta(cta_), G(G_), ntiles(ntiles_), spt(spt_), seg(0), it(it0_), it1(it1_) {}
    __device__ __forceinline__ bool next(int &tile, int &st0, int &st1) {
        if (dp) {
            tile = cta + (seg++) * G;
            st0 = 0;
            st1 = spt;
            return tile < ntiles;
        }
        if (it >= it1) return false;
        tile = (int)(it / spt);
        st0 = (int)(it - (long long)tile * spt);
        st1 = (int)min((long long)spt, it1 - (long long)tile * spt);
        it = (long long)tile * spt + st1;
        return true;
    }
};


// Expert activation in the bf16 epilogues (its output is rounded to bf16):
// SwiGLU silu(g)*u with ex2.approx / rcp.approx, tanh with tanh.approx —
// a few instructions instead of ~40 for expf + IEEE division, which made the
// wide prefill epilogue ALU-bound. Every bf16 path (fused, fixup, prefill)
// uses this one function, so they stay bitwise comparable.
template <int NMAT>
__device__ __forceinline__ float expert_act(float g, float u) {
    if (NMAT == 2) return __fdividef(g, 1.0f + __expf(-g)) * u;
    float t;
    asm("tanh.approx.f32 %0, %1;" : "=f"(t) : "f"(g));
    return t;
}

// Finish columns [c0, c0+16) of a tile for this thread's weight row m =
// mtile*128 + q*32 + lane (g: gate/only accumulator, u: SwiGLU up):
// mode 2 -> y_perm fp32 (32 lanes write 128 consecutive bytes per column);
// else the activation -> bf16 SW128 H planes, lanes packing pairs to bf16x2
// and gathering 8 m's (one 16-byte swizzle chunk) per 128-bit store.
template <int NMAT>
__device__ __forceinline__ void finish16(const GemmParams &p, const TileInfo &ti, int c0, int q, unsigned lane,
                                         const float (&g)[16], const float (&u)[16]) {
    if (p.mode == 2) {
        const int m = ti.mtile * kBM + q * 32 + (int)lane;
#pragma unroll
        for (int j = 0; j < 16; ++j) p.y_perm[(long long)(ti.row0 + c0 + j) * p.M + m] = g[j];
        return;
    }
    const int mg = ti.mtile * kBM + q * 32 + ((int)lane & ~7);  // group's first m
    const int plane = mg >> 6, chunk = (mg & 63) >> 3;
    const int gbase = (int)lane & ~7;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const float hv = expert_act<NMAT>(g[j], u[j]);
        const float ov = __shfl_xor_sync(0xffffffffu, hv, 1);
        const __nv_bfloat162 pr2 = (lane & 1) ? __floats2bfloat162_rn(ov, hv) : __floats2bfloat162_rn(hv, ov);
        const uint32_t w = *reinterpret_cast<const uint32_t *>(&pr2);
        uint4 v4;
        v4.x = __shfl_sync(0xffffffffu, w, gbase + 0);
        v4.y = __shfl_sync(0xffffffffu, w, gbase + 2);
        v4.z = __shfl_sync(0xffffffffu, w, gbase + 4);
        v4.w = __shfl_sync(0xffffffffu, w, gbase + 6);
        if (((int)lane & 7) == (j & 7)) {
            const int row = ti.row0 + c0 + j;
            uint4 *dstp = reinterpret_cast<uint4 *>(p.h_planes) +
                          (((long long)plane * p.h_rmax + row) * 8 + (chunk ^ (row & 7)));
            *dstp = v4;
        }
    }
}

template <int NMAT, int KPS>
__global__ void __launch_bounds__(kThreads, 1) ffn_gemm_kernel(GemmParams p) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ Sched sched;
    __shared__ __align__(8) uint64_t bars[64];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const int mtiles = p.M / kBM;
    const int steps_per_tile = p.K / (kBK * KPS);  // pipeline steps per tile

    if (warp == 0) build_sched_warp(sched, p.count, p.offset, p.E, p.n_tile);
    __syncthreads();
    const int ntiles = total_tiles(sched, mtiles);
    const long long T = (long long)ntiles * steps_per_tile;
    const int G = (int)min((long long)p.num_ctas, p.dp ? (long long)ntiles : T);
    const int cta = (int)blockIdx.x;
    if (cta >= G) return;  // uniform for the whole CTA
    const long long it0 = range_start(cta, T, G), it1 = range_start(cta + 1, T, G);
    const SegIter seg0(p.dp, cta, G, ntiles, steps_per_tile, it0, it1);

    // smem: stages of [A: KPS x NMAT x 16 KB | B: KPS x bsz], 1024-aligned
    constexpr uint32_t kAStage = (uint32_t)(KPS * NMAT) * kATileBytes;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t bsz = ((uint32_t)p.n_tile * 128u + 1023u) & ~1023u;
    const uint32_t stage_bytes = kAStage + (uint32_t)KPS * bsz;
    const int stages = min(16, (int)((kSmemBudget - 1024) / stage_bytes));
    // TMEM: accumulator stage [NMAT][n_tile] fp32 columns, double-buffered when it fits
    const int acc_stages = (2 * NMAT * p.n_tile <= 512) ? 2 : 1;
    const uint32_t acc_cols = acc_stages == 2 ? 256u : 512u;

    const uint32_t full0 = ptx::smem_u32(&bars[0]);     // [stages]
    const uint32_t empty0 = ptx::smem_u32(&bars[16]);   // [stages]
    const uint32_t tfull0 = ptx::smem_u32(&bars[32]);   // [2]
    const uint32_t tempty0 = ptx::smem_u32(&bars[34]);  // [2]

    if (warp == 1 && lane == 0) {
        for (int s = 0; s < stages; ++s) {
            ptx::mbar_init(full0 + 8 * s, 1);
            ptx::mbar_init(empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(tfull0 + 8 * a, 1);
            ptx::mbar_init(tempty0 + 8 * a, 4);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc(ptx::smem_u32(&tmem_base_sh), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem_base = tmem_base_sh;

    if (warp == 0 && lane == 0) {
        // ===================== producer =====================
        const uint64_t pol = ptx::policy_evict_first();  // decode: weights stream through once
        int stage = 0;
        uint32_t phase = 0;
        SegIter w = seg0;
        int tile, st_beg, st_end;
        while (w.next(tile, st_beg, st_end)) {
            const TileInfo ti = decode_tile(sched, tile, mtiles, p.n_tile);
            const int buf = p.buf_of_expert[ti.e];
            // the m-tile's blocks are contiguous along k: [mt][kb][NMAT][16 KB]
            const uint8_t *a_src = p.arena + (long long)buf * p.buf_bytes + p.mat_off +
                                   (long long)ti.mtile * steps_per_tile * kAStage;
            const uint8_t *b_src = p.b_planes + (long long)ti.row0 * 128;
            const uint32_t bbytes = (uint32_t)ti.n * 128u;
            for (int st = st_beg; st < st_end; ++st) {
                ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1u);
                const uint32_t sA = base + (uint32_t)stage * stage_bytes;
                const uint32_t sB = sA + kAStage;
                const uint32_t fb = full0 + 8 * stage;
                if (p.probe == 2) {  // diagnostics: no data movement, only the barrier protocol
                    ptx::mbar_arrive(fb);
                } else {
                ptx::mbar_expect_tx(fb, kAStage + (uint32_t)KPS * bbytes);
                if (p.dp) {  // the CTAs on the m-tile's other chunks read the same block: keep it in L2
                    ptx::bulk_load(sA, a_src + (long long)st * kAStage, kAStage, fb);
                } else {
                    ptx::bulk_load_hint(sA, a_src + (long long)st * kAStage, kAStage, fb, pol);
                }
#pragma unroll
                for (int i = 0; i < KPS; ++i)
                    ptx::bulk_load(sB + i * bsz, b_src + (long long)(st * KPS + i) * p.b_plane_bytes, bbytes, fb);
                }
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
    } else if (warp == 1 && lane == 0) {
        // ===================== MMA issuer (single thread) =====================
        // Descriptor start addresses advance in 16-byte units: k-subblock kk
        // (+32 B) -> +2, matrix/k-block (+16 KB) -> +1024, B k-block -> +bsz/16.
        const uint64_t desc0 = ptx::sw128_desc(base);
        const uint64_t stage_d = stage_bytes >> 4, bsz_d = bsz >> 4;
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        SegIter w = seg0;
        int tile, st_beg, st_end;
        while (w.next(tile, st_beg, st_end)) {
            const TileInfo ti = decode_tile(sched, tile, mtiles, p.n_tile);
            const uint32_t idesc = ptx::idesc_bf16_f32(kBM, (uint32_t)ti.n);
            ptx::mbar_wait(tempty0 + 8 * acc, acc_phase ^ 1u);
            ptx::tc_fence_after();
            const uint32_t d0 = tmem_base + (uint32_t)acc * acc_cols;
            const uint32_t d1 = d0 + (uint32_t)p.n_tile;
            uint32_t accum = 0;
            for (int st = st_beg; st < st_end; ++st) {
                ptx::mbar_wait(full0 + 8 * stage, phase);
                ptx::tc_fence_after();
                const uint64_t a = desc0 + (uint64_t)stage * stage_d;
                const uint64_t b = a + (kAStage >> 4);
                if (p.probe != 1) {
#pragma unroll
                    for (int i = 0; i < KPS; ++i) {
                        const uint64_t bi = b + (uint64_t)i * bsz_d;
#pragma unroll
                        for (int kk = 0; kk < kBK / 16; ++kk) {
                            ptx::mma_bf16(d0, a + (uint64_t)((i * NMAT) * (kATileBytes >> 4) + 2 * kk), bi + 2 * kk,
                                          idesc, accum);
                            if (NMAT == 2)
                                ptx::mma_bf16(d1, a + (uint64_t)((i * NMAT + 1) * (kATileBytes >> 4) + 2 * kk),
                                              bi + 2 * kk, idesc, accum);
                            accum = 1u;
                        }
                    }
                }
                ptx::mma_commit(empty0 + 8 * stage);  // frees the smem stage when these MMAs finish
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            ptx::mma_commit(tfull0 + 8 * acc);  // accumulator ready for the epilogue
            if (acc_stages == 2) {
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1u;
            } else {
                acc_phase ^= 1u;
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue: TMEM -> fp32 partial slot =====================
        const int q = warp - 4;  // TMEM lane quadrant
        const int m_local = q * 32 + (int)lane;
        int acc = 0;
        uint32_t acc_phase = 0;
        SegIter w = seg0;
        int tile, st_beg, st_end;
        while (w.next(tile, st_beg, st_end)) {
            const TileInfo ti = decode_tile(sched, tile, mtiles, p.n_tile);
            // this CTA owns the whole tile: finish it here (activation / output),
            // otherwise park an fp32 partial for the deterministic fixup
            const bool whole = p.fuse && st_beg == 0 && st_end == steps_per_tile;
            ptx::mbar_wait(tfull0 + 8 * acc, acc_phase);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem_base + (uint32_t)acc * acc_cols + ((uint32_t)(q * 32) << 16);
            if (whole) {
                for (int c0 = 0; c0 < ti.n; c0 += 16) {
                    float g[16], u[16];
                    ptx::tmem_ld16(tbase + (uint32_t)c0, g);
                    if (NMAT == 2) ptx::tmem_ld16(tbase + (uint32_t)(p.n_tile + c0), u);
                    finish16<NMAT>(p, ti, c0, q, lane, g, u);
                }
            } else {
                const long long slot = (long long)tile + cta;
                float *dst = p.partials + slot * (long long)NMAT * p.n_tile * kBM;
#pragma unroll
                for (int m = 0; m < NMAT; ++m) {
                    for (int c0 = 0; c0 < ti.n; c0 += 16) {
                        float v[16];
                        ptx::tmem_ld16(tbase + (uint32_t)(m * p.n_tile + c0), v);
#pragma unroll
                        for (int j = 0; j < 16; ++j) dst[((long long)m * p.n_tile + c0 + j) * kBM + m_local] = v[j];
                    }
                }
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(tempty0 + 8 * acc);
            if (acc_stages == 2) {
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1u;
            } else {
                acc_phase ^= 1u;
            }
        }
    }
    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc(tmem_base, 512);
}

// ------------------------------------------------ prefill GEMM on CTA pairs
// cta_group::2 tcgen05 MMAs (M = 256): the two CTAs of a cluster hold the two
// weight m-tiles of an m-tile pair, each loads ITS 128 weight rows and HALF of
// the token chunk (N/2 rows), and the leader CTA issues M=256 MMAs that read
// both CTAs' shared memory and write both CTAs' TMEM. Per MAC every SM then
// moves and reads fewer operand bytes through shared memory than the
// single-CTA tile, whose bulk-copy writes plus tensor-core reads saturate the
// SM's shared-memory bandwidth (profiles/README.md). Each CTA finishes its own
// m-tile in its own epilogue (SwiGLU -> H, or y), exactly as the single-CTA
// kernel does, so the outputs are bitwise identical.
// Both CTAs load with cta_group::2 tensor-map copies that complete on the
// LEADER's full[s] barrier, so the leader's MMA sees both halves land
// without a relay; the two byte-image tensor maps (weights arena, token
// planes) are [rows][128 B] views of the pre-swizzled images.
//   full[s]  : leader only, both CTAs' bytes (leader expects them)
//   empty[s] : both CTAs, released by the leader's multicast commit
//   tfull[a] : both CTAs, leader's multicast commit
//   tempty[a]: leader only, 4 local + 4 remote epilogue-warp arrivals
struct PairMaps {
    CUtensorMap a;  // weights arena, uint8 [rows][128], box 128 x 256 rows
    CUtensorMap b;  // token planes, uint8 [K/64 * r_max][128], box 128 x n_tile/2 rows
};

template <int NMAT, int KPS>
__global__ void __launch_bounds__(kThreads, 1) ffn_gemm_2sm_kernel(GemmParams p, const __grid_constant__ PairMaps tm) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ Sched sched;
    __shared__ __align__(8) uint64_t bars[64];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const int rank = (int)ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int mpairs = p.M / (2 * kBM);
    const int spt = p.K / (kBK * KPS);

    if (warp == 0) build_sched_warp(sched, p.count, p.offset, p.E, p.n_tile);
    __syncthreads();
    const int units = total_tiles(sched, mpairs);  // (expert, m-tile pair, token chunk)
    const int G = min(p.num_ctas / 2, units);
    const int pair = (int)(blockIdx.x >> 1);
    if (pair >= G) return;  // uniform for both CTAs of the pair

    constexpr uint32_t kAStage = (uint32_t)(KPS * NMAT) * kATileBytes;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t bbox = (uint32_t)(p.n_tile / 2) * 128u;  // bytes of one B box (a k-block of the token half)
    const uint32_t bhalf = (bbox + 1023u) & ~1023u;
    const uint32_t stage_bytes = kAStage + (uint32_t)KPS * bhalf;
    const int stages = min(16, (int)((kSmemBudget - 1024) / stage_bytes));
    const int acc_stages = (2 * NMAT * p.n_tile <= 512) ? 2 : 1;
    const uint32_t acc_cols = acc_stages == 2 ? 256u : 512u;

    const uint32_t full0 = ptx::smem_u32(&bars[0]);     // [stages] (leader)
    const uint32_t empty0 = ptx::smem_u32(&bars[16]);   // [stages]
    const uint32_t tfull0 = ptx::smem_u32(&bars[48]);   // [2]
    const uint32_t tempty0 = ptx::smem_u32(&bars[50]);  // [2] (leader)

    if (warp == 1 && lane == 0) {
        for (int s = 0; s < stages; ++s) {
            ptx::mbar_init(full0 + 8 * s, 1);
            ptx::mbar_init(empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(tfull0 + 8 * a, 1);
            ptx::mbar_init(tempty0 + 8 * a, 8);
        }
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc_pair(ptx::smem_u32(&tmem_base_sh), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = tmem_base_sh;

    if (warp == 0 && lane == 0) {
        // ===================== producer (both CTAs): own weight m-tile + own half of the tokens
        ptx::prefetch_tmap(&tm.a);
        ptx::prefetch_tmap(&tm.b);
        const uint32_t full_leader = leader ? full0 : ptx::mapa(full0, 0);
        const int b_rows = (int)(p.b_plane_bytes / 128);  // rows per k-block plane
        int stage = 0;
        uint32_t phase = 0;
        for (int u = pair; u < units; u += G) {
            const TileInfo ti = decode_tile(sched, u, mpairs, p.n_tile);
            const int mt = 2 * ti.mtile + rank;
            const int buf = p.buf_of_expert[ti.e];
            const long long a_row0 = ((long long)buf * p.buf_bytes + p.mat_off + (long long)mt * spt * kAStage) / 128;
            const int b_row0 = ti.row0 + rank * (ti.n / 2);
            for (int st = 0; st < spt; ++st) {
                ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1u);
                const uint32_t sA = base + (uint32_t)stage * stage_bytes;
                const uint32_t sB = sA + kAStage;
                const uint32_t fb = full_leader + 8 * stage;
                if (leader) ptx::mbar_expect_tx(full0 + 8 * stage, 2u * (kAStage + (uint32_t)KPS * bbox));
                const long long ar = a_row0 + (long long)st * (kAStage / 128);
#pragma unroll
                for (int j = 0; j < (int)(kAStage / 32768); ++j)
                    ptx::tma_load_2d_pair(sA + (uint32_t)j * 32768u, &tm.a, fb, 0, (int32_t)(ar + 256 * j));
#pragma unroll
                for (int i = 0; i < KPS; ++i)
                    ptx::tma_load_2d_pair(sB + (uint32_t)i * bhalf, &tm.b, fb, 0, (st * KPS + i) * b_rows + b_row0);
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
        for (int i = 0; i < stages; ++i) {  // every stage released: no multicast commit still in flight to us
            ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1u);
            if (++stage == stages) {
                stage = 0;
                phase ^= 1u;
            }
        }
    } else if (warp == 1 && lane == 0 && leader) {
        // ===================== leader: M=256 pair MMAs
        const uint64_t desc0 = ptx::sw128_desc(base);
        const uint64_t stage_d = stage_bytes >> 4, bh_d = bhalf >> 4;
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = pair; u < units; u += G) {
            const TileInfo ti = decode_tile(sched, u, mpairs, p.n_tile);
            const uint32_t idesc = ptx::idesc_bf16_f32(2 * kBM, (uint32_t)ti.n);
            ptx::mbar_wait_cluster(tempty0 + 8 * acc, acc_phase ^ 1u);
            ptx::tc_fence_after();
            const uint32_t d0 = tmem_base + (uint32_t)acc * acc_cols;
            const uint32_t d1 = d0 + (uint32_t)p.n_tile;
            uint32_t accum = 0;
            for (int st = 0; st < spt; ++st) {
                ptx::mbar_wait_cluster(full0 + 8 * stage, phase);
                ptx::tc_fence_after();
                const uint64_t a = desc0 + (uint64_t)stage * stage_d;
                const uint64_t b = a + (kAStage >> 4);
#pragma unroll
                for (int i = 0; i < KPS; ++i) {
                    const uint64_t bi = b + (uint64_t)i * bh_d;
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        ptx::mma_bf16_pair(d0, a + (uint64_t)((i * NMAT) * (kATileBytes >> 4) + 2 * kk), bi + 2 * kk,
                                           idesc, accum);
                        if (NMAT == 2)
                            ptx::mma_bf16_pair(d1, a + (uint64_t)((i * NMAT + 1) * (kATileBytes >> 4) + 2 * kk),
                                               bi + 2 * kk, idesc, accum);
                        accum = 1u;
                    }
                }
                ptx::mma_commit_pair(empty0 + 8 * stage, 0x3);  // both CTAs' stage is free once these finish
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            ptx::mma_commit_pair(tfull0 + 8 * acc, 0x3);  // both CTAs' accumulators are ready
            if (acc_stages == 2) {
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1u;
            } else {
                acc_phase ^= 1u;
            }
        }
    } else if (warp >= 4) {
        // ===================== epilogue (both CTAs): own m-tile, all tokens of the chunk
        const int q = warp - 4;
        const uint32_t tempty_leader = leader ? tempty0 : ptx::mapa(tempty0, 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = pair; u < units; u += G) {
            TileInfo ti = decode_tile(sched, u, mpairs, p.n_tile);
            ti.mtile = 2 * ti.mtile + rank;
            ptx::mbar_wait_cluster(tfull0 + 8 * acc, acc_phase);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem_base + (uint32_t)acc * acc_cols + ((uint32_t)(q * 32) << 16);
            for (int c0 = 0; c0 < ti.n; c0 += 16) {
                float g[16], uu[16];
                ptx::tmem_ld16(tbase + (uint32_t)c0, g);
                if (NMAT == 2) ptx::tmem_ld16(tbase + (uint32_t)(p.n_tile + c0), uu);
                finish16<NMAT>(p, ti, c0, q, lane, g, uu);
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader)
                    ptx::mbar_arrive(tempty0 + 8 * acc);
                else
                    ptx::mbar_arrive_cluster(tempty_leader + 8 * acc);
            }
            if (acc_stages == 2) {
                acc ^= 1;
                if (acc == 0) acc_phase ^= 1u;
            } else {
                acc_phase ^= 1u;
            }
        }
    }
    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();  // neither CTA frees TMEM / leaves while the pair still works
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc_pair(tmem_base, 512);
}

// ------------------------------------------------ prefill GEMM1 (SwiGLU) on CTA pairs, W1 | W3 split
// The pair's M = 256 rows are W1's and W3's rows of ONE m-tile: the leader
// CTA holds the W1 block, the peer the W3 block, each with half of a
// 256-token chunk, so each CTA's TMEM keeps one 256-column accumulator (double
// buffered) and per MAC every SM moves the same operand bytes as GEMM2's pair
// tiles. SwiGLU needs g (leader) and u (peer) side by side: each CTA sends the
// accumulator columns its peer finishes (leader: g of the upper token half,
// peer: u of the lower half) into the peer's shared memory (DSMEM stores),
// then finishes its own token half — the same activation and bf16 rounding
// as every other path, so H is bitwise identical.
//   xfull : my receive buffer holds this tile's columns (4 remote warp arrivals)
//   xfree : my PEER's receive buffer may be overwritten (4 remote arrivals)
template <int KPS>
__global__ void __launch_bounds__(kThreads, 1) ffn_gemm1_split_kernel(GemmParams p, const __grid_constant__ PairMaps tm) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ Sched sched;
    __shared__ __align__(8) uint64_t bars[64];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const int rank = (int)ptx::cluster_ctarank();
    const bool leader = rank == 0;
    const int mtiles = p.M / kBM;
    const int kblocks = p.K / kBK;
    const int spt = kblocks / KPS;

    if (warp == 0) build_sched_warp(sched, p.count, p.offset, p.E, p.n_tile);
    __syncthreads();
    const int units = total_tiles(sched, mtiles);  // (expert, m-tile, token chunk)
    const int G = min(p.num_ctas / 2, units);
    const int pair = (int)(blockIdx.x >> 1);
    if (pair >= G) return;

    constexpr uint32_t kAStage = (uint32_t)KPS * kATileBytes;  // own matrix only
    constexpr int kXCols = 64;                                 // columns per exchange round
    constexpr uint32_t kXStride = kXCols * 4 + 16;             // receive-buffer row (padded: conflict-free)
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    const uint32_t bbox = (uint32_t)(p.n_tile / 2) * 128u;
    const uint32_t bhalf = (bbox + 1023u) & ~1023u;
    const uint32_t stage_bytes = kAStage + (uint32_t)KPS * bhalf;
    const uint32_t xbuf_bytes = 128u * kXStride;  // 128 rows x kXCols fp32 (+ padding)
    const int stages = min(16, (int)((kSmemBudget - 1024 - xbuf_bytes) / stage_bytes));
    const uint32_t xbuf = base + (uint32_t)stages * stage_bytes;
    const uint32_t acc_cols = 256u;  // one accumulator of <= 256 token columns, double buffered

    const uint32_t full0 = ptx::smem_u32(&bars[0]);     // [stages] (leader)
    const uint32_t empty0 = ptx::smem_u32(&bars[16]);   // [stages]
    const uint32_t tfull0 = ptx::smem_u32(&bars[48]);   // [2]
    const uint32_t tempty0 = ptx::smem_u32(&bars[50]);  // [2] (leader)
    const uint32_t xfull = ptx::smem_u32(&bars[52]);
    const uint32_t xfree = ptx::smem_u32(&bars[53]);

    if (warp == 1 && lane == 0) {
        for (int s = 0; s < stages; ++s) {
            ptx::mbar_init(full0 + 8 * s, 1);
            ptx::mbar_init(empty0 + 8 * s, 1);
        }
        for (int a = 0; a < 2; ++a) {
            ptx::mbar_init(tfull0 + 8 * a, 1);
            ptx::mbar_init(tempty0 + 8 * a, 8);
        }
        ptx::mbar_init(xfull, 4);
        ptx::mbar_init(xfree, 4);
        ptx::fence_barrier_init();
    }
    if (warp == 2) ptx::tmem_alloc_pair(ptx::smem_u32(&tmem_base_sh), 512);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    const uint32_t tmem_base = tmem_base_sh;

    if (warp == 0 && lane == 0) {
        // ===================== producer (both CTAs): own matrix's weight blocks + own token half
        ptx::prefetch_tmap(&tm.a);
        ptx::prefetch_tmap(&tm.b);
        const uint32_t full_leader = leader ? full0 : ptx::mapa(full0, 0);
        const int b_rows = (int)(p.b_plane_bytes / 128);
        int stage = 0;
        uint32_t phase = 0;
        for (int u = pair; u < units; u += G) {
            const TileInfo ti = decode_tile(sched, u, mtiles, p.n_tile);
            const int buf = p.buf_of_expert[ti.e];
            // block (mt, kb, mat) of the UMMA-tiled expert: ((mt*K/64 + kb)*2 + mat) * 16 KB
            const long long blk0 = ((long long)buf * p.buf_bytes + p.mat_off) / kATileBytes +
                                   ((long long)ti.mtile * kblocks) * 2 + rank;
            const int b_row0 = ti.row0 + rank * (ti.n / 2);
            for (int st = 0; st < spt; ++st) {
                ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1u);
                const uint32_t sA = base + (uint32_t)stage * stage_bytes;
                const uint32_t sB = sA + kAStage;
                const uint32_t fb = full_leader + 8 * stage;
                if (leader) ptx::mbar_expect_tx(full0 + 8 * stage, 2u * (kAStage + (uint32_t)KPS * bbox));
#pragma unroll
                for (int i = 0; i < KPS; ++i) {
                    const long long blk = blk0 + 2LL * (st * KPS + i);
                    ptx::tma_load_2d_pair(sA + (uint32_t)i * kATileBytes, &tm.a, fb, 0, (int32_t)(blk * 128));
                    ptx::tma_load_2d_pair(sB + (uint32_t)i * bhalf, &tm.b, fb, 0, (st * KPS + i) * b_rows + b_row0);
                }
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
        }
        for (int i = 0; i < stages; ++i) {
            ptx::mbar_wait(empty0 + 8 * stage, phase ^ 1u);
            if (++stage == stages) {
                stage = 0;
                phase ^= 1u;
            }
        }
    } else if (warp == 1 && lane == 0 && leader) {
        // ===================== leader: M=256 pair MMAs ([W1 ; W3] rows x 256 tokens)
        const uint64_t desc0 = ptx::sw128_desc(base);
        const uint64_t stage_d = stage_bytes >> 4, bh_d = bhalf >> 4;
        int stage = 0;
        uint32_t phase = 0;
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = pair; u < units; u += G) {
            const TileInfo ti = decode_tile(sched, u, mtiles, p.n_tile);
            const uint32_t idesc = ptx::idesc_bf16_f32(2 * kBM, (uint32_t)ti.n);
            ptx::mbar_wait_cluster(tempty0 + 8 * acc, acc_phase ^ 1u);
            ptx::tc_fence_after();
            const uint32_t d0 = tmem_base + (uint32_t)acc * acc_cols;
            uint32_t accum = 0;
            for (int st = 0; st < spt; ++st) {
                ptx::mbar_wait_cluster(full0 + 8 * stage, phase);
                ptx::tc_fence_after();
                const uint64_t a = desc0 + (uint64_t)stage * stage_d;
                const uint64_t b = a + (kAStage >> 4);
#pragma unroll
                for (int i = 0; i < KPS; ++i) {
                    const uint64_t ai = a + (uint64_t)i * (kATileBytes >> 4), bi = b + (uint64_t)i * bh_d;
#pragma unroll
                    for (int kk = 0; kk < kBK / 16; ++kk) {
                        ptx::mma_bf16_pair(d0, ai + 2 * kk, bi + 2 * kk, idesc, accum);
                        accum = 1u;
                    }
                }
                ptx::mma_commit_pair(empty0 + 8 * stage, 0x3);
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1u;
                }
            }
            ptx::mma_commit_pair(tfull0 + 8 * acc, 0x3);
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1u;
        }
    } else if (warp >= 4) {
        // ===================== epilogue: exchange half the accumulator, SwiGLU on own token half
        const int q = warp - 4;
        const int m_local = q * 32 + (int)lane;
        const int peer = rank ^ 1;
        const uint32_t tempty_leader = leader ? tempty0 : ptx::mapa(tempty0, 0);
        const uint32_t peer_xbuf = ptx::mapa(xbuf, (uint32_t)peer);
        const uint32_t peer_xfull = ptx::mapa(xfull, (uint32_t)peer);
        const uint32_t peer_xfree = ptx::mapa(xfree, (uint32_t)peer);
        int acc = 0;
        uint32_t acc_phase = 0, xph = 0;
        for (int u = pair; u < units; u += G) {
            const TileInfo ti = decode_tile(sched, u, mtiles, p.n_tile);
            const int csplit = ((ti.n / 2) + 15) & ~15;  // leader finishes [0, csplit), peer [csplit, n)
            const int mine0 = leader ? 0 : csplit, mine1 = leader ? csplit : ti.n;
            const int send0 = leader ? csplit : 0, send1 = leader ? ti.n : csplit;
            ptx::mbar_wait_cluster(tfull0 + 8 * acc, acc_phase);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem_base + (uint32_t)acc * acc_cols + ((uint32_t)(q * 32) << 16);
            // in rounds of kXCols columns (both halves have <= 128 columns: two rounds, always
            // executed so the two CTAs' handshakes pair up):
            for (int rd = 0; rd < 128 / kXCols; ++rd) {
                // 1. my accumulator columns the peer finishes -> its receive buffer
                const int s0 = send0 + rd * kXCols, s1 = min(send1, s0 + kXCols);
                ptx::mbar_wait_cluster(xfree, xph ^ 1u);
                for (int c0 = s0; c0 < s1; c0 += 16) {
                    float v[16];
                    ptx::tmem_ld16(tbase + (uint32_t)c0, v);
                    const uint32_t dst = peer_xbuf + (uint32_t)m_local * kXStride + (uint32_t)(c0 - s0) * 4u;
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        ptx::st_cluster_v4(dst + 4u * j, v[j], v[j + 1], v[j + 2], v[j + 3]);
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster(peer_xfull);
                // 2. my token half: own accumulator + the peer's columns from my receive buffer
                const int m0 = mine0 + rd * kXCols, m1 = min(mine1, m0 + kXCols);
                ptx::mbar_wait_cluster(xfull, xph);
                for (int c0 = m0; c0 < m1; c0 += 16) {
                    float own[16], oth[16];
                    ptx::tmem_ld16(tbase + (uint32_t)c0, own);
                    const uint32_t src = xbuf + (uint32_t)m_local * kXStride + (uint32_t)(c0 - m0) * 4u;
#pragma unroll
                    for (int j = 0; j < 16; j += 4)
                        ptx::ld_shared_v4(src + 4u * j, oth[j], oth[j + 1], oth[j + 2], oth[j + 3]);
                    if (leader)
                        finish16<2>(p, ti, c0, q, lane, own, oth);
                    else
                        finish16<2>(p, ti, c0, q, lane, oth, own);
                }
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive_cluster(peer_xfree);  // my receive buffer is consumed
                xph ^= 1u;
            }
            ptx::tc_fence_before();
            __syncwarp();
            if (lane == 0) {
                if (leader)
                    ptx::mbar_arrive(tempty0 + 8 * acc);
                else
                    ptx::mbar_arrive_cluster(tempty_leader + 8 * acc);
            }
            acc ^= 1;
            if (acc == 0) acc_phase ^= 1u;
        }
    }
    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::cluster_sync();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc_pair(tmem_base, 512);
}

// ---------------------------------------------------------------- fixups
__device__ __forceinline__ int cta_of(long long i, long long T, int G) {
    return (int)(((i + 1) * (long long)G - 1) / T);
}

// mode 0: SwiGLU (nmat 2) / 1: tanh (nmat 1) -> H as bf16 SW128 planes
// mode 2: plain (nmat 1) -> y_perm fp32 [r_max][M]
__global__ void __launch_bounds__(kBM) ffn_fixup_kernel(GemmParams p, int mode, uint4 *h_planes, int h_rmax,
                                                        float *y_perm) {
    __shared__ Sched sched;
    const int mtiles = p.M / kBM;
    const int steps_per_tile = p.K / (kBK * p.kps);  // must match ffn_gemm_kernel's iteration space
    if (threadIdx.x < 32) build_sched_warp(sched, p.count, p.offset, p.E, p.n_tile);
    __syncthreads();
    const int ntiles = total_tiles(sched, mtiles);
    const long long T = (long long)ntiles * steps_per_tile;
    const int G = (int)min((long long)p.num_ctas, T);
    const int m_local = threadIdx.x;
    for (int tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
        const TileInfo ti = decode_tile(sched, tile, mtiles, p.n_tile);
        const int c0 = cta_of((long long)tile * steps_per_tile, T, G);
        const int c1 = cta_of((long long)(tile + 1) * steps_per_tile - 1, T, G);
        if (p.fuse && c0 == c1) continue;  // one CTA owned it: its epilogue already wrote the result
        const long long slot_elems = (long long)p.nmat * p.n_tile * kBM;
        const int m = ti.mtile * kBM + m_local;
        for (int n = 0; n < ti.n; ++n) {
            float g = 0.f, u = 0.f;
            for (int c = c0; c <= c1; ++c) {
                const float *src = p.partials + ((long long)tile + c) * slot_elems;
                g += src[(long long)n * kBM + m_local];
                if (p.nmat == 2) u += src[((long long)p.n_tile + n) * kBM + m_local];
            }
            const int row = ti.row0 + n;
            if (mode == 2) {
                y_perm[(long long)row * p.M + m] = g;
            } else {
                const float h = mode == 0 ? expert_act<2>(g, u) : expert_act<1>(g, 0.f);
                // bf16 SW128 image: plane m/64, chunk (m%64)/8 at position chunk ^ (row & 7)
                __nv_bfloat16 *hp = reinterpret_cast<__nv_bfloat16 *>(h_planes);
                const int plane = m >> 6, chunk = (m & 63) >> 3;
                const long long idx = ((long long)plane * h_rmax + row) * 64 + ((chunk ^ (row & 7)) << 3) + (m & 7);
                hp[idx] = __float2bfloat16_rn(h);
            }
        }
    }
}

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
struct FusedParams {
    GemmParams g[2];
    int *arrive;         // [2][tile_cap] split-tile arrival counters
    int tile_cap;
    unsigned *grid_bar;  // [0] arrivals, [1] generation
    int prefetch_w2;     // stream W2's first stages before the barrier opens
};

constexpr int kSmemFused = 216 * 1024;

struct Geom {
    uint32_t base, stage_bytes, bsz, b_off;  // b_off: B part offset inside a stage (max A bytes)
    int stages;
    uint32_t full0, empty0, tfull0, tempty0;
};

template <int NMAT, int KPS>
__device__ void fused_produce(const GemmParams &P, const Sched &s, const Geom &gm, int &stage, uint32_t &phase,
                              long long it0, long long it1, int spt, uint64_t pol, const unsigned *gate,
                              unsigned gen0, int prefetch) {
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
        while (ptx::ld_acquire_gpu(gate) == gen0) __nanosleep(64);
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
        while (ptx::ld_acquire_gpu(gate) == gen0) __nanosleep(64);
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

template <int NMAT, int KPS>
__device__ void fused_mma(const GemmParams &P, const Sched &s, const Geom &gm, int &stage, uint32_t &phase, int &acc,
                          uint32_t &acc_phase, long long it0, long long it1, int spt, uint32_t tmem_base) {
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
                               uint32_t &acc_phase, long long T, int G, int cta, int spt, uint32_t tmem_base, int q,
                               unsigned lane) {
    if (cta >= G) return;
    const int mtiles = P.M / kBM;
    const long long it0 = range_start(cta, T, G), it1 = range_start(cta + 1, T, G);
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
        const uint32_t tbase = tmem_base + (uint32_t)acc * 256u + ((uint32_t)(q * 32) << 16);
        if (whole) {
            for (int c0 = 0; c0 < ti.n; c0 += 16) {
                float g[16], u[16];
                ptx::tmem_ld16(tbase + (uint32_t)c0, g);
                if (NMAT == 2) ptx::tmem_ld16(tbase + (uint32_t)(P.n_tile + c0), u);
                finish16<NMAT>(P, ti, c0, q, lane, g, u);
            }
        } else if (reducer) {
            const int c1 = cta_of((long long)(tile + 1) * spt - 1, T, G);
            if (m_local == 0) {
                while (ptx::ld_acquire_gpu(reinterpret_cast<const unsigned *>(arrive + tile)) < (unsigned)(c1 - cta))
                    __nanosleep(32);
                arrive[tile] = 0;  // every contributor has arrived: reset for the next launch
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
                for (int c = cta + 1; c <= c1; ++c) {
                    const float *src = P.partials + ((long long)tile + c) * slot_elems;
#pragma unroll
                    for (int j = 0; j < 16; ++j) {
                        g[j] += __ldcg(src + (long long)(cc + j) * kBM + m_local);
                        if (NMAT == 2) u[j] += __ldcg(src + (long long)(P.n_tile + cc + j) * kBM + m_local);
                    }
                }
                finish16<NMAT>(P, ti, cc, q, lane, g, u);
            }
        } else {
            float *dst = P.partials + ((long long)tile + cta) * slot_elems;
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
        if (!whole && !reducer) {  // publish the partial, then arrive
            __threadfence();
            ptx::named_bar_sync(1, 128);
            if (m_local == 0) atomicAdd(arrive + tile, 1);
        }
    }
}

template <int NMAT1, int KPS1, int KPS2>
__global__ void __launch_bounds__(kThreads, 1) ffn_fused_kernel(const __grid_constant__ FusedParams fp) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ Sched sched;
    __shared__ __align__(8) uint64_t bars[64];
    __shared__ uint32_t tmem_base_sh;

    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const GemmParams &P1 = fp.g[0];
    const GemmParams &P2 = fp.g[1];
    const int n_tile = P1.n_tile;
    if (warp == 0) build_sched_warp(sched, P1.count, P1.offset, P1.E, n_tile);
    // the barrier generation cannot advance before this CTA arrives, so
    // reading it here (before the __syncthreads) is race-free
    unsigned gen0 = 0;
    if (threadIdx.x == 0) gen0 = *reinterpret_cast<volatile unsigned *>(fp.grid_bar + 1);

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

    const int cta = blockIdx.x, Gn = gridDim.x;
    const int spt1 = P1.K / (kBK * KPS1), spt2 = P2.K / (kBK * KPS2);
    const long long T1 = (long long)total_tiles(sched, P1.M / kBM) * spt1;
    const long long T2 = (long long)total_tiles(sched, P2.M / kBM) * spt2;
    const int G1 = (int)min((long long)Gn, T1), G2 = (int)min((long long)Gn, T2);

    if (warp == 0 && lane == 0) {
        const uint64_t pol = ptx::policy_evict_first();  // weights stream through once
        int stage = 0;
        uint32_t phase = 0;
        if (cta < G1)
            fused_produce<NMAT1, KPS1>(P1, sched, gm, stage, phase, range_start(cta, T1, G1),
                                       range_start(cta + 1, T1, G1), spt1, pol, nullptr, 0, 0);
        if (cta < G2)
            fused_produce<1, KPS2>(P2, sched, gm, stage, phase, range_start(cta, T2, G2), range_start(cta + 1, T2, G2),
                                   spt2, pol, fp.grid_bar + 1, gen0, fp.prefetch_w2);
    } else if (warp == 1 && lane == 0) {
        int stage = 0, acc = 0;
        uint32_t phase = 0, acc_phase = 0;
        if (cta < G1)
            fused_mma<NMAT1, KPS1>(P1, sched, gm, stage, phase, acc, acc_phase, range_start(cta, T1, G1),
                                   range_start(cta + 1, T1, G1), spt1, tmem_base);
        if (cta < G2)
            fused_mma<1, KPS2>(P2, sched, gm, stage, phase, acc, acc_phase, range_start(cta, T2, G2),
                               range_start(cta + 1, T2, G2), spt2, tmem_base);
    } else if (warp >= 4) {
        const int q = warp - 4;
        int acc = 0;
        uint32_t acc_phase = 0;
        fused_epilogue<NMAT1>(P1, sched, gm, fp.arrive, acc, acc_phase, T1, G1, cta, spt1, tmem_base, q, lane);
        // H of this CTA is written: publish it (to the bulk-copy proxy too) and arrive
        ptx::fence_proxy_async_global();
        __threadfence();
        ptx::named_bar_sync(1, 128);
        if (q == 0 && lane == 0) {
            const unsigned prev = atomicAdd(fp.grid_bar, 1u);
            if (prev == (unsigned)Gn - 1u) {
                fp.grid_bar[0] = 0u;
                __threadfence();
                atomicAdd(fp.grid_bar + 1, 1u);
            }
        }
        fused_epilogue<1>(P2, sched, gm, fp.arrive + fp.tile_cap, acc, acc_phase, T2, G2, cta, spt2, tmem_base, q,
                          lane);
    }
    __syncwarp();
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == 2) ptx::tmem_dealloc(tmem_base, 512);
}

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

// kernel timing (for the bench's roofline), off by default
struct Timing {
    bool enabled = false;
    std::vector<cudaEvent_t> ev;  // 4 per call: before/after GEMM1, before/after GEMM2
    std::mutex mu;
} g_timing;

int record_event(cudaStream_t s) {
    cudaEvent_t e;
    BM_CUDA_TRY(cudaEventCreate(&e));
    BM_CUDA_TRY(cudaEventRecord(e, s));
    g_timing.ev.push_back(e);
    return BM_OK;
}

typedef void (*GemmFn)(GemmParams);

template <int NMAT, int KPS>
int launch_gemm(const GemmParams &g, int G, cudaStream_t s) {
    static bool attr = false;
    auto kern = ffn_gemm_kernel<NMAT, KPS>;
    if (!attr) {
        BM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
        attr = true;
    }
    kern<<<G, kThreads, kSmemBudget, s>>>(g);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

int launch_gemm_1sm(const GemmParams &g, int G, cudaStream_t s) {
    if (g.nmat == 2) {
        if (g.kps == 1) return launch_gemm<2, 1>(g, G, s);
        if (g.kps == 2) return launch_gemm<2, 2>(g, G, s);
        return launch_gemm<2, 4>(g, G, s);
    }
    if (g.kps == 1) return launch_gemm<1, 1>(g, G, s);
    if (g.kps == 2) return launch_gemm<1, 2>(g, G, s);
    return launch_gemm<1, 4>(g, G, s);
}

// cuTensorMapEncodeTiled through the runtime's driver entry point (no -lcuda):
// a uint8 [rows][128] view of a pre-swizzled byte image, box 128 x box_rows
typedef CUresult (*EncodeTiledFn)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *, const cuuint64_t *,
                                  const cuuint64_t *, const cuuint32_t *, const cuuint32_t *, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int encode_rows(CUtensorMap *m, const void *base, unsigned long long rows, unsigned box_rows) {
    static EncodeTiledFn fn = nullptr;
    if (!fn) {
        cudaDriverEntryPointQueryResult q;
        void *f = nullptr;
        BM_CUDA_TRY(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q));
        BM_REQUIRE(f && q == cudaDriverEntryPointSuccess, BM_ECUDA, "cuTensorMapEncodeTiled unavailable");
        fn = reinterpret_cast<EncodeTiledFn>(f);
    }
    const cuuint64_t dims[2] = {128, (cuuint64_t)rows};
    const cuuint64_t strides[1] = {128};
    const cuuint32_t box[2] = {128, (cuuint32_t)box_rows};
    const cuuint32_t es[2] = {1, 1};
    const CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void *>(base), dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    BM_REQUIRE(r == CUDA_SUCCESS, BM_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return BM_OK;
}

// NMAT 0: GEMM1 with W1 | W3 split over the pair (ffn_gemm1_split_kernel)
template <int NMAT, int KPS>
int launch_gemm_2sm(const GemmParams &g, int G, cudaStream_t s) {
    static bool attr = false;
    auto kern = NMAT == 0 ? ffn_gemm1_split_kernel<KPS> : ffn_gemm_2sm_kernel<NMAT == 0 ? 1 : NMAT, KPS>;
    if (!attr) {
        BM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
        attr = true;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = kSmemBudget;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    static int max_clusters = 0;  // persistent pairs: only co-resident clusters
    if (!max_clusters) {
        cfg.gridDim = dim3((unsigned)(G & ~1));
        BM_CUDA_TRY(cudaOccupancyMaxActiveClusters(&max_clusters, kern, &cfg));
        if (max_clusters < 1) max_clusters = 1;
    }
    GemmParams gp = g;
    gp.num_ctas = 2 * std::min(G / 2, max_clusters);
    cfg.gridDim = dim3((unsigned)gp.num_ctas);
    PairMaps maps;
    if (int rc = encode_rows(&maps.a, g.arena, (unsigned long long)(g.arena_bytes / 128), NMAT == 0 ? 128 : 256))
        return rc;
    if (int rc = encode_rows(&maps.b, g.b_planes, (unsigned long long)(g.K / kBK) * (g.b_plane_bytes / 128),
                             (unsigned)(g.n_tile / 2)))
        return rc;
    BM_CUDA_TRY(cudaLaunchKernelEx(&cfg, kern, gp, maps));
    BM_LAUNCH_CHECK();
    return BM_OK;
}

// k-blocks per stage of the CTA-pair GEMM: the largest of {2, 1} dividing
// K/64 that leaves >= 3 stages (BMOE_KPS_2SM overrides)
int kps_2sm(int nmat, long long K, long long n_tile) {
    const long long bhalf = ((n_tile / 2) * 128 + 1023) / 1024 * 1024;
    if (const char *ev = getenv("BMOE_KPS_2SM"))  // tuning override (must divide K/64 and fit twice)
        if (atoi(ev) == 1 || (atoi(ev) == 2 && (K / kBK) % 2 == 0)) return atoi(ev);
    int kps = 2;
    while (kps > 1 && ((K / kBK) % kps || (kSmemBudget - 1024) / (kps * (nmat * kATileBytes + bhalf)) < 3)) kps >>= 1;
    return kps;
}

// Data-parallel (prefill) GEMMs on CTA pairs (cta_group::2, M = 256) at
// 256-token tiles, one accumulator per CTA (double-buffered TMEM):
//  * GEMM2 (and a tanh GEMM1): the pair's rows are two weight m-tiles
//    (even m-tile count): Mixtral 4096 x 2 0.93 -> 0.73 ms;
//  * SwiGLU GEMM1: the pair's rows are W1 and W3 of one m-tile
//    (ffn_gemm1_split_kernel, accumulator halves exchanged through DSMEM).
// BMOE_2SM=0: single CTAs; 2: SwiGLU GEMM1 as two m-tiles x (W1, W3) instead
// (two accumulators per CTA at 128 tokens; measured slower).
int two_sm_mode() {
    const char *ev = getenv("BMOE_2SM");
    return ev ? atoi(ev) : 1;
}
bool use_2sm(const GemmParams &g) {
    const int mode = two_sm_mode();
    if (!g.dp || mode == 0 || g.n_tile < 32 || g.n_tile % 32) return false;
    // W1 | W3 split pair: its accumulator exchange costs a few us per tile, paid
    // back only by long tiles (Mixtral K=4096: 1.66 -> 1.51 ms; Qwen3 K=2048:
    // 0.45 -> 0.56 ms, so shorter K keeps single CTAs)
    if (g.nmat == 2 && mode == 1) return g.K >= 4096;
    return (g.nmat == 1 || mode == 2) && (g.M / kBM) % 2 == 0;
}

int launch_gemm_2sm_dispatch(const GemmParams &g, int G, cudaStream_t s) {
    if (g.nmat == 2 && two_sm_mode() == 1) return g.kps == 1 ? launch_gemm_2sm<0, 1>(g, G, s) : launch_gemm_2sm<0, 2>(g, G, s);
    if (g.nmat == 2) return g.kps == 1 ? launch_gemm_2sm<2, 1>(g, G, s) : launch_gemm_2sm<2, 2>(g, G, s);
    return g.kps == 1 ? launch_gemm_2sm<1, 1>(g, G, s) : launch_gemm_2sm<1, 2>(g, G, s);
}

int launch_gemm_dispatch(const GemmParams &g, int G, cudaStream_t s) {
    if (use_2sm(g)) {
        GemmParams g2 = g;
        if (g.nmat == 2 && two_sm_mode() == 1) {  // W1 | W3 split: 256-token tiles, one matrix per CTA
            g2.n_tile = 256;
            if (const char *ev = getenv("BMOE_NT1")) g2.n_tile = atoi(ev);
            g2.kps = 1;  // 4 stages of 32 KB beside the 66 KB receive buffer
        } else {
            g2.kps = kps_2sm(g.nmat, g.K, g.n_tile);
        }
        return launch_gemm_2sm_dispatch(g2, G, s);
    }
    return launch_gemm_1sm(g, G, s);
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
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;  // the grid barrier needs every CTA resident
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
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

// k-blocks per pipeline stage: the largest of {4,2,1} dividing K/64 whose
// stage fits twice in shared memory (BMOE_KPS overrides for tuning).
int kps_for(int nmat, long long K, long long n_tile) {
    int kps = 4;
    if (const char *ev = getenv("BMOE_KPS")) kps = atoi(ev);
    const long long per_kb = (long long)nmat * kATileBytes + ((n_tile * 128 + 1023) / 1024) * 1024;
    while (kps > 1 && ((K / kBK) % kps || kps * per_kb > (kSmemBudget - 1024) / 2)) kps >>= 1;
    return kps < 1 ? 1 : (kps > 4 ? 4 : kps);
}

}  // namespace
}  // namespace bm

using namespace bm;

namespace bm {
namespace {
// workspace: [fp32 partial slots | bf16 SW128 H planes | split-tile arrival
// counters (2 phases) + grid barrier]; the counters must start at zero.
struct WsLayout {
    long long partial_bytes, h_off, h_bytes, ctr_off, tile_cap, total;
};
WsLayout ws_layout(long long E, long long d, long long f, long long r_max, long long n_tile) {
    WsLayout w;
    const long long M = std::max(d, f);
    w.tile_cap = max_tiles(E, M, r_max, n_tile);
    const long long slots = w.tile_cap + sm_count() + 1;
    w.partial_bytes = ((slots * 2 * n_tile * kBM * 4 + 1023) / 1024) * 1024;
    w.h_off = w.partial_bytes;
    w.h_bytes = (((f / 64) * r_max * 128 + 1023) / 1024) * 1024;
    w.ctr_off = w.h_off + w.h_bytes;
    w.total = w.ctr_off + (2 * w.tile_cap + 2) * 4;
    return w;
}
}  // namespace
}  // namespace bm

extern "C" int64_t bm_expert_ffn_bf16_workspace(int64_t E, int64_t d, int64_t f, int64_t r_max, int64_t n_tile) {
    return ws_layout(E, d, f, r_max, n_tile).total;
}

extern "C" int bm_expert_ffn_bf16(const void *x_perm, const int32_t *expert_count, const int32_t *expert_offset,
                                  int64_t E, int64_t d, int64_t f, int32_t act, const void *w_arena, int64_t n_bufs,
                                  const int32_t *buf_of_expert, int64_t r_max, int64_t n_tile, void *workspace,
                                  int64_t workspace_bytes, float *y_perm, bm_stream_t stream) {
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
    float *partials = static_cast<float *>(workspace);
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
    if (fused) {
        int k1 = 1, k2 = 1;
        fused_kps(nmat1, d, f, n_tile, &k1, &k2);
        g1.kps = k1;
        g2.kps = k2;
        g1.fuse = g2.fuse = 1;
        g1.dp = g2.dp = 0;
        int pre = 1;
        if (const char *ev = getenv("BMOE_PREFETCH_W2")) pre = atoi(ev);
        FusedParams fp{{g1, g2}, counters, (int)wl.tile_cap, reinterpret_cast<unsigned *>(counters + 2 * wl.tile_cap),
                       pre};
        // timing record: [start, end] of the one kernel, then an empty GEMM2 interval
        if (timing && record_event(s)) return BM_ECUDA;
        const int rc = nmat1 == 2 ? launch_fused_k<2>(fp, k1, k2, G, s) : launch_fused_k<1>(fp, k1, k2, G, s);
        if (rc) return rc;
        if (timing) {
            if (record_event(s)) return BM_ECUDA;
            g_timing.ev.push_back(nullptr);  // no second kernel: GEMM2 interval reported as 0
            g_timing.ev.push_back(nullptr);
        }
        return BM_OK;
    }
    if (timing && record_event(s)) return BM_ECUDA;
    if (int rc = launch_gemm_dispatch(g1, G, s)) return rc;
    if (timing && record_event(s)) return BM_ECUDA;
    if (dp) {  // every tile was finished by its GEMM epilogue
        // GEMM2 (one accumulator per tile) keeps a double-buffered 256-token
        // tile on CTA pairs: wider tiles halve its per-MAC operand traffic
        if (n_tile >= 128 && use_2sm(g2)) {
            const char *ev = getenv("BMOE_NT2");
            g2.n_tile = ev ? atoi(ev) : 256;
        }
        if (timing && record_event(s)) return BM_ECUDA;
        if (int rc = launch_gemm_dispatch(g2, G, s)) return rc;
        if (timing && record_event(s)) return BM_ECUDA;
        return BM_OK;
    }
    const int fix_blocks = 4 * G;
    ffn_fixup_kernel<<<fix_blocks, kBM, 0, s>>>(g1, act == BM_ACT_SWIGLU ? 0 : 1, reinterpret_cast<uint4 *>(h_planes),
                                                (int)r_max, nullptr);
    BM_LAUNCH_CHECK();
    if (timing && record_event(s)) return BM_ECUDA;
    if (int rc = launch_gemm_dispatch(g2, G, s)) return rc;
    if (timing && record_event(s)) return BM_ECUDA;
    ffn_fixup_kernel<<<fix_blocks, kBM, 0, s>>>(g2, 2, nullptr, 0, y_perm);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_set_kernel_timing(int32_t enable) {
    std::lock_guard<std::mutex> lk(g_timing.mu);
    for (cudaEvent_t e : g_timing.ev)
        if (e) cudaEventDestroy(e);
    g_timing.ev.clear();
    g_timing.enabled = enable != 0;
    return BM_OK;
}

extern "C" int bm_kernel_timing_enabled(void) { return g_timing.enabled ? 1 : 0; }

// Two floats per bm_expert_ffn_bf16 call since timing was enabled: GEMM1
// and GEMM2 kernel durations in ms (CUDA events on the launching stream).
extern "C" int64_t bm_kernel_times(float *out_host, int64_t cap) {
    std::lock_guard<std::mutex> lk(g_timing.mu);
    int64_t n = 0;
    for (size_t i = 0; i + 3 < g_timing.ev.size() && n + 2 <= cap; i += 4) {
        const bool one = g_timing.ev[i + 2] == nullptr;  // fused decode call: one kernel
        if (cudaEventSynchronize(g_timing.ev[one ? i + 1 : i + 3]) != cudaSuccess) return -1;
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, g_timing.ev[i], g_timing.ev[i + 1]);
        if (!one) cudaEventElapsedTime(&b, g_timing.ev[i + 2], g_timing.ev[i + 3]);
        out_host[n++] = a;
        out_host[n++] = b;
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
