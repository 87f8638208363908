// K4 prefill: bf16 grouped expert GEMMs for wide token tiles (n_tile > 64),
// plus the stream-K GEMM + fixup pair that the decode kernel's A/B switch
// (BMOE_FUSED=0) and BMOE_DP=0 fall back to.
//  * ffn_gemm_kernel: single-CTA tcgen05 tiles (M=128 weight rows x N tokens),
//    stream-K (decode switch) or data-parallel (prefill) work;
//  * ffn_gemm_2sm_kernel / ffn_gemm1_split_kernel: CTA pairs (cta_group::2,
//    M = 256) for the data-parallel prefill GEMMs;
//  * ffn_fixup_kernel: deterministic reduction of stream-K split tiles.
// Reference semantics: Expert.__call__ / forward_batch (model.py:85-99,
// 318-340); SwiGLU is the Mixtral/Qwen3/DSV2 expert (no reference oracle).
#include "ffn_common.cuh"

namespace bm {
namespace ffn {

// Token-major SwiGLU finish: g / u hold W1 / W3 rows [c0, c0+16) of m-tile
// `mtile` for token `row`; SwiGLU -> bf16 -> the two 16-byte chunks of H.
__device__ __forceinline__ void finish_tm16(const GemmParams &p, int mtile, int row, int c0, const float (&g)[16],
                                            const float (&u)[16]) {
    uint32_t w[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const __nv_bfloat162 pr =
            __floats2bfloat162_rn(expert_act<2>(g[2 * j], u[2 * j]), expert_act<2>(g[2 * j + 1], u[2 * j + 1]));
        w[j] = *reinterpret_cast<const uint32_t *>(&pr);
    }
    const int f0 = mtile * kBM + c0, plane = f0 >> 6, chunk = (f0 & 63) >> 3;
    uint4 *dst = reinterpret_cast<uint4 *>(p.h_planes) + ((long long)plane * p.h_rmax + row) * 8;
    dst[chunk ^ (row & 7)] = make_uint4(w[0], w[1], w[2], w[3]);
    dst[(chunk + 1) ^ (row & 7)] = make_uint4(w[4], w[5], w[6], w[7]);
}

// TM (token-major SwiGLU GEMM1, data-parallel 128-token tiles): the MMA takes
// the tokens as A (M = 128) and the m-tile's W1 and W3 blocks, which lie back
// to back in the stage, as ONE B operand (N = 256), instead of two MMAs with
// the weights as A. Per k-block the tensor core then reads 48 KB of operands
// instead of 64 KB (tokens once, not once per matrix), which is what bounds
// these tiles (shared-memory bandwidth, profiles/README.md). The accumulator
// is [token lane][W1 | W3 column], so a lane finishes 16 consecutive f of its
// token with two 16-byte H stores, no shuffles.
template <int NMAT, int KPS, bool TM = false>
__global__ void __launch_bounds__(kThreads, 1) ffn_gemm_kernel(GemmParams p) {
    static_assert(!TM || NMAT == 2, "token-major tiles are the SwiGLU GEMM1");
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
            const uint32_t idesc = TM ? ptx::idesc_bf16_f32(kBM, 2 * kBM) : ptx::idesc_bf16_f32(kBM, (uint32_t)ti.n);
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
                if (TM && p.probe != 1) {  // A = the token rows, B = [W1 ; W3] (256 rows)
#pragma unroll
                    for (int i = 0; i < KPS; ++i) {
#pragma unroll
                        for (int kk = 0; kk < kBK / 16; ++kk) {
                            ptx::mma_bf16(d0, b + (uint64_t)i * bsz_d + 2 * kk,
                                          a + (uint64_t)((i * NMAT) * (kATileBytes >> 4) + 2 * kk), idesc, accum);
                            accum = 1u;
                        }
                    }
                } else if (p.probe != 1) {
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
            if (TM) {  // lane = token row m_local of the tile; columns [0,128) W1, [128,256) W3
                const int row = ti.row0 + m_local;
                for (int c0 = 0; c0 < kBM; c0 += 16) {
                    float g[16], u[16];
                    ptx::tmem_ld16(tbase + (uint32_t)c0, g);
                    ptx::tmem_ld16(tbase + (uint32_t)(kBM + c0), u);
                    if (m_local < ti.n) finish_tm16(p, ti.mtile, row, c0, g, u);
                }
            } else if (whole) {
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
// TMP (token-major pair, BMOE_TM=2): the same loads, with the operands' roles
// swapped: A = the pair's 256 tokens (each CTA's token half = its 128 rows of
// A), B = [W1 ; W3] as N = 256 split along N (W1 block in the leader, W3 in
// the peer). Each CTA's TMEM then holds its own tokens x (W1 | W3) and
// finishes SwiGLU locally: no DSMEM exchange.
template <int KPS, bool TMP = false>
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
            const uint32_t idesc = TMP ? ptx::idesc_bf16_f32(2 * kBM, 2 * kBM) : ptx::idesc_bf16_f32(2 * kBM, (uint32_t)ti.n);
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
                        if (TMP)
                            ptx::mma_bf16_pair(d0, bi + 2 * kk, ai + 2 * kk, idesc, accum);
                        else
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
    } else if (TMP && warp >= 4) {
        // ===================== epilogue (token-major): own tokens x (W1 | W3), SwiGLU in place
        const int q = warp - 4;
        const int m_local = q * 32 + (int)lane;
        const uint32_t tempty_leader = leader ? tempty0 : ptx::mapa(tempty0, 0);
        int acc = 0;
        uint32_t acc_phase = 0;
        for (int u = pair; u < units; u += G) {
            const TileInfo ti = decode_tile(sched, u, mtiles, p.n_tile);
            const int h0 = ti.n / 2;  // the producers' split: leader tokens [0, h0), peer [h0, n)
            const int mine = leader ? h0 : ti.n - h0;
            const int row = ti.row0 + (leader ? 0 : h0) + m_local;
            ptx::mbar_wait_cluster(tfull0 + 8 * acc, acc_phase);
            ptx::tc_fence_after();
            const uint32_t tbase = tmem_base + (uint32_t)acc * acc_cols + ((uint32_t)(q * 32) << 16);
            for (int c0 = 0; c0 < kBM; c0 += 16) {
                float g[16], uu[16];
                ptx::tmem_ld16(tbase + (uint32_t)c0, g);
                ptx::tmem_ld16(tbase + (uint32_t)(kBM + c0), uu);
                if (m_local < mine) finish_tm16(p, ti.mtile, row, c0, g, uu);
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

template <int NMAT, int KPS, bool TM = false>
int launch_gemm(const GemmParams &g, int G, cudaStream_t s) {
    static bool attr = false;
    auto kern = ffn_gemm_kernel<NMAT, KPS, TM>;
    if (!attr) {
        BM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBudget));
        attr = true;
    }
    kern<<<G, kThreads, kSmemBudget, s>>>(g);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

// token-major SwiGLU GEMM1 tiles (BMOE_TM, read per call; default on): data-parallel
// 128-token tiles finished in their own epilogue
int tm_mode();
bool use_tm(const GemmParams &g) {
    return tm_mode() != 0 && g.nmat == 2 && g.mode == 0 && g.dp && g.fuse && g.n_tile == 128 &&
           g.probe == 0;
}

int launch_gemm_1sm(const GemmParams &g, int G, cudaStream_t s) {
    if (use_tm(g)) {
        if (g.kps == 1) return launch_gemm<2, 1, true>(g, G, s);
        if (g.kps == 2) return launch_gemm<2, 2, true>(g, G, s);
        return launch_gemm<2, 4, true>(g, G, s);
    }
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
    auto kern = NMAT == 0    ? ffn_gemm1_split_kernel<KPS>
                : NMAT == -1 ? ffn_gemm1_split_kernel<KPS, true>
                             : ffn_gemm_2sm_kernel<NMAT <= 0 ? 1 : NMAT, KPS>;
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
    if (int rc = encode_rows(&maps.a, g.arena, (unsigned long long)(g.arena_bytes / 128), NMAT <= 0 ? 128 : 256))
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
// BMOE_TM (read per call): 0 weight-major GEMM1 tiles everywhere, 1 token-major single-CTA
// tiles, 2 token-major CTA pairs (ffn_gemm1_split_kernel<KPS, true>) at any K, 3 (default)
// pairs once the call averages >= 256 rows per expert, else single CTAs: the 256-token pair
// tiles half-fill at fewer rows (Qwen3 2048 x 8, 128 rows / expert: 0.173 vs 0.168 ms single;
// 8192 x 8: 0.394 vs 0.432 ms; profiles/r2s_prefill_tmp.jsonl)
int tm_mode() {
    const char *ev = getenv("BMOE_TM");
    return ev ? atoi(ev) : 3;
}
bool tm_pair(const GemmParams &g) {
    const int m = tm_mode();
    return (m == 2 || (m == 3 && (long long)g.h_rmax >= 256LL * g.E)) && g.nmat == 2 && g.mode == 0 && g.dp &&
           g.fuse;
}

bool use_2sm(const GemmParams &g) {
    const int mode = two_sm_mode();
    if (!g.dp || mode == 0 || g.n_tile < 32 || g.n_tile % 32) return false;
    // W1 | W3 split pair: its accumulator exchange costs a few us per tile, paid
    // back only by long tiles (Mixtral K=4096: 1.66 -> 1.51 ms; Qwen3 K=2048:
    // 0.45 -> 0.56 ms, so shorter K keeps single CTAs)
    if (g.nmat == 2 && mode == 1) return g.K >= 4096 || tm_pair(g);
    return (g.nmat == 1 || mode == 2) && (g.M / kBM) % 2 == 0;
}

int launch_gemm_2sm_dispatch(const GemmParams &g, int G, cudaStream_t s) {
    if (g.nmat == 2 && two_sm_mode() == 1 && tm_pair(g))
        return g.kps == 1 ? launch_gemm_2sm<-1, 1>(g, G, s) : launch_gemm_2sm<-1, 2>(g, G, s);
    if (g.nmat == 2 && two_sm_mode() == 1) return g.kps == 1 ? launch_gemm_2sm<0, 1>(g, G, s) : launch_gemm_2sm<0, 2>(g, G, s);
    if (g.nmat == 2) return g.kps == 1 ? launch_gemm_2sm<2, 1>(g, G, s) : launch_gemm_2sm<2, 2>(g, G, s);
    return g.kps == 1 ? launch_gemm_2sm<1, 1>(g, G, s) : launch_gemm_2sm<1, 2>(g, G, s);
}

int launch_gemm_dispatch(const GemmParams &g, int G, cudaStream_t s) {
    if (use_2sm(g)) {
        GemmParams g2 = g;
        if (g.nmat == 2 && two_sm_mode() == 1) {  // W1 | W3 split: 256-token tiles, one matrix per CTA
            g2.n_tile = 256;
            if (const char *ev = getenv("BMOE_NT1"); ev && !tm_pair(g)) g2.n_tile = atoi(ev);  // token-major: 2 x 128 rows
            g2.kps = 1;  // 5 stages of 32 KB beside the 35 KB receive buffer
            if (const char *kv = getenv("BMOE_KPS_SPLIT")) g2.kps = (atoi(kv) == 2 && (g.K / kBK) % 2 == 0) ? 2 : 1;
        } else {
            g2.kps = kps_2sm(g.nmat, g.K, g.n_tile);
        }
        return launch_gemm_2sm_dispatch(g2, G, s);
    }
    return launch_gemm_1sm(g, G, s);
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


int launch_fixup(const GemmParams &g, int mode, uint4 *h_planes, int h_rmax, float *y_perm, int blocks,
                 cudaStream_t s) {
    ffn_fixup_kernel<<<blocks, kBM, 0, s>>>(g, mode, h_planes, h_rmax, y_perm);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

}  // namespace ffn
}  // namespace bm
