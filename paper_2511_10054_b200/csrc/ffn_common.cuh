// Shared pieces of the bf16 grouped expert FFN (K4) on 5th-gen tensor cores
// (sm_100a): tile geometry, the device-side expert schedule, tile decoding,
// the stream-K / data-parallel work iterator, the expert activation and the
// tile epilogue, plus the launch entry points each kernel family exports.
//   ffn_decode.cu  : decode width (n_tile <= 64), one cooperative launch per call
//   ffn_prefill.cu : prefill width, data-parallel tiles, single CTAs and CTA pairs
//   ffn_tc.cu      : the C-ABI (bm_expert_ffn_bf16 dispatch, packing, workspace, timing)
// Not part of the ABI.
#pragma once

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
namespace ffn {

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
inline __device__ void build_sched_warp(Sched &s, const int32_t *count, const int32_t *offset, int E, int n_tile) {
    constexpr int kPer = kMaxE / 32;
    const int lane = (int)lane_id();
    const int per = (E + 31) / 32;
    int c[kPer], o[kPer];
    int nact = 0, nch = 0;
#pragma unroll
    for (int i = 0; i < kPer; ++i) {  // counts and offsets in one round of loads
        const int e = lane * per + i;
        const bool in = i < per && e < E;
        c[i] = in ? count[e] : 0;
        o[i] = in ? offset[e] : 0;
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
            s.act_off[ia] = o[i];
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
    int nch;                 // token chunks of expert e
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
    ti.nch = nch;
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

// gate-weighted combine + layer_update fused behind the FFN (B = 0: none):
// h[b] = rmsnorm(h[b] + scale * sum_s probs[b,s] * y_perm[slot_row[b,s]])
struct CombineArgs {
    const int32_t *slot_row;
    const float *probs;
    const uint8_t *kind;
    float *h;
    float scale;
    int B, k;
};

struct FusedParams {
    GemmParams g[2];
    int *arrive;         // [2][tile_cap] split-tile arrival counters
    int tile_cap;
    // grid barrier: a monotonic 64-bit arrival count. Every launch's barriers take
    // G arrivals each, so at a CTA's entry floor(count / G) * G is the base of this
    // launch (no instance of this launch can complete before the CTA arrives), and
    // barrier n of the launch has passed once the count reaches base + n * G.
    unsigned long long *grid_bar;
    int prefetch_w2;     // stream W2's first stages before the barrier opens
    unsigned long long *trace;  // diagnostics (BMOE_FFN_TRACE): kTracePts globaltimer stamps per CTA, else null
    CombineArgs cmb;            // K5 after a second grid barrier, in the same launch
    int pdl;                    // launched with programmatic stream serialization (griddepcontrol.wait first)
    // per-expert H readiness (null: GEMM2 waits for the whole of GEMM1 at the grid barrier):
    // h_ready[p][e] counts expert e's finished GEMM1 tiles; a GEMM2 stage of expert e loads its
    // H part once all mtiles1 * nch(e) of them are in. Two arrays alternate by launch parity
    // (launch n = floor(launch_count / G), every CTA adds 1 on exit, fire and forget): launch
    // n counts in h_ready[n & 1] and clears h_ready[(n + 1) & 1], which launch n - 1 used.
    int *h_ready;
    unsigned long long *launch_count;
    unsigned long long *span;  // kernel timing: [min entry, max exit] globaltimer of this launch, else null
    int groups;                // expert groups whose GEMM1 / GEMM2 phases interleave (needs h_ready; <= kMaxGroups)
    int group_min_iters;       // ... while each GEMM1 phase keeps this many k-steps per CTA (0: no limit)
    int min_iters;             // k-steps per CTA below which a phase runs on fewer CTAs (1: all CTAs)
};
constexpr int kMaxGroups = 4;
constexpr int kTracePts = 12;

// CTA that processes stream-K iteration i of T over G CTAs
__device__ __forceinline__ int cta_of(long long i, long long T, int G) {
    return (int)(((i + 1) * (long long)G - 1) / T);
}

// ---------------------------------------------------------- cross-file entry points
// prefill (ffn_prefill.cu)
int launch_gemm_dispatch(const GemmParams &g, int G, cudaStream_t s);  // one GEMM of a call
bool use_2sm(const GemmParams &g);                                      // CTA-pair kernels for this GEMM?
int kps_for(int nmat, long long K, long long n_tile);                   // k-blocks per pipeline stage
int launch_fixup(const GemmParams &g, int mode, uint4 *h_planes, int h_rmax, float *y_perm, int blocks,
                 cudaStream_t s);                                       // stream-K split-tile reduction
// kernel timing of FFN calls inside captured graphs (ffn_tc.cu; the engine's timing pass)
void *ffn_timing_take_capture();      // the timed calls recorded during the capture just ended
void ffn_timing_replayed(void *group);  // that graph was launched
int ffn_timing_harvest();             // read the replayed groups (their launches completed)
void ffn_timing_release(void *group);
// decode (ffn_decode.cu)
void fused_kps(int nmat1, long long d, long long f, long long n_tile, int *k1, int *k2);
int launch_fused_dispatch(const FusedParams &fp, int nmat1, int kps1, int kps2, int G, cudaStream_t s);

}  // namespace ffn
}  // namespace bm
