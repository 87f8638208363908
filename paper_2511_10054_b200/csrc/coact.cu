// K6 co-activation counting (shared-memory-privatised triangular counters)
// and K7 buddy ranking (one warp per pivot, bit-exact f64 in numpy order).
// Reference: profiler.observe / conditional_row (profiler.py:67-119),
// buddies.cft_prefix / build_table (buddies.py:79-129).
#include <algorithm>

#include "common.cuh"
#include "numpy_order.cuh"
#include "ptx.cuh"

namespace bm {
namespace {

constexpr int kCountThreads = 512;
constexpr int kMaxE = 256;
constexpr int kMaxK = 32;

// packed upper triangle incl. diagonal: (i <= j) -> i*E - i*(i-1)/2 + (j-i)
__device__ __forceinline__ int tri(int i, int j, int E) { return i * E - ((i * (i - 1)) >> 1) + (j - i); }

// One thread per token. With k >= 2 and k distinct ids per token (the
// reference rejects duplicates, profiler.py:76-80) every token holding expert
// i adds exactly k-1 to row i of the pair matrix, so the diagonal is derived
// at flush time as rowsum/(k-1) instead of being counted: 28 instead of 36
// shared atomics per token at k=8 (the kernel is bound by the shared-memory
// atomic pipe, not by the trace read).
template <int KC>
__global__ void __launch_bounds__(kCountThreads) coact_count_kernel(const int32_t *__restrict__ topk, long long N,
                                                                    int k_rt, int E, long long per_block,
                                                                    unsigned long long *__restrict__ counts,
                                                                    unsigned long long *__restrict__ pairs,
                                                                    int *__restrict__ invalid) {
    extern __shared__ uint32_t tcount[];  // E*(E+1)/2
    const int k = KC > 0 ? KC : k_rt;
    const bool derive_diag = k >= 2;
    const int ntri = E * (E + 1) / 2;
    for (int i = threadIdx.x; i < ntri; i += blockDim.x) tcount[i] = 0;
    __syncthreads();
    const long long t0 = (long long)blockIdx.x * per_block;
    const long long t1 = min(N, t0 + per_block);
    if constexpr (KC == 8) {
        // The eight ids are sorted first (a 19-comparator network on unsigned values, so
        // negative ids sort last like out-of-range ones): range and duplicate checks become
        // one compare on the largest id and seven on neighbours, and every pair (x < y) is
        // already ordered, so its cell is rowbase(id_x) + id_y with the seven row bases
        // computed once -- one add per pair instead of a min, max and triangle index.
        for (long long t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
            const int4 *p = reinterpret_cast<const int4 *>(topk + t * 8);
            int4 a = __ldg(p), b = __ldg(p + 1);
            unsigned id[8] = {(unsigned)a.x, (unsigned)a.y, (unsigned)a.z, (unsigned)a.w,
                              (unsigned)b.x, (unsigned)b.y, (unsigned)b.z, (unsigned)b.w};
            auto cx = [&](int u, int v) {
                const unsigned lo = min(id[u], id[v]), hi = max(id[u], id[v]);
                id[u] = lo;
                id[v] = hi;
            };
            // Batcher odd-even merge sort, n = 8
            cx(0, 1); cx(2, 3); cx(4, 5); cx(6, 7);
            cx(0, 2); cx(1, 3); cx(4, 6); cx(5, 7);
            cx(1, 2); cx(5, 6);
            cx(0, 4); cx(1, 5); cx(2, 6); cx(3, 7);
            cx(2, 4); cx(3, 5);
            cx(1, 2); cx(3, 4); cx(5, 6);
            // profiler.py:76-80: ids in range and distinct, else the row is rejected
            bool bad = id[7] >= (unsigned)E;
#pragma unroll
            for (int x = 0; x < 7; ++x) bad |= id[x] == id[x + 1];
            if (bad) {
                atomicAdd(invalid, 1);
                continue;
            }
#pragma unroll
            for (int x = 0; x < 7; ++x) {
                const int i = (int)id[x];
                const int base = i * E - ((i * (i - 1)) >> 1) - i;  // tri(i, j, E) = base + j
#pragma unroll
                for (int y = x + 1; y < 8; ++y) atomicAdd(&tcount[base + (int)id[y]], 1u);
            }
        }
    } else {
        for (long long t = t0 + threadIdx.x; t < t1; t += blockDim.x) {
            int id[kMaxK];
            bool bad = false;
            for (int x = 0; x < k; ++x) {
                id[x] = __ldg(topk + t * k + x);
                bad |= (unsigned)id[x] >= (unsigned)E;
                for (int y = 0; y < x; ++y) bad |= id[x] == id[y];
            }
            if (bad) {
                atomicAdd(invalid, 1);
                continue;
            }
            for (int x = 0; x < k; ++x) {
                if (!derive_diag) atomicAdd(&tcount[tri(id[x], id[x], E)], 1u);
                for (int y = x + 1; y < k; ++y) {
                    int i = min(id[x], id[y]), j = max(id[x], id[y]);
                    atomicAdd(&tcount[tri(i, j, E)], 1u);
                }
            }
        }
    }
    __syncthreads();
    if (derive_diag) {  // diagonal cell := (sum of row i off the diagonal) / (k-1)
        for (int i = threadIdx.x; i < E; i += blockDim.x) {
            unsigned long long s = 0;
            for (int j = 0; j < i; ++j) s += tcount[tri(j, i, E)];
            for (int j = i + 1; j < E; ++j) s += tcount[tri(i, j, E)];
            tcount[tri(i, i, E)] = (uint32_t)(s / (unsigned long long)(k - 1));
        }
        __syncthreads();
    }
    // flush: diagonal -> counts, off-diagonal -> both mirror cells
    for (int i = 0; i < E; ++i) {
        const int base = tri(i, i, E);
        for (int j = i + threadIdx.x; j < E; j += blockDim.x) {
            const uint32_t v = tcount[base + (j - i)];
            if (!v) continue;
            if (j == i) {
                atomicAdd(&counts[i], (unsigned long long)v);
            } else {
                atomicAdd(&pairs[(size_t)i * E + j], (unsigned long long)v);
                atomicAdd(&pairs[(size_t)j * E + i], (unsigned long long)v);
            }
        }
    }
}

// K6 on the tensor cores (E <= 128): the co-activation matrix is X^T X over
// the trace's one-hot rows, X[t][e] = 1 if token t routed to expert e. A
// stage holds 256 tokens as two 128-token K blocks of X^T in the UMMA
// K-major, 128B-swizzled layout (expert e's row: one byte per token), built
// in shared memory by 256 builder threads (one token each: zero the stage,
// then one byte store per id); one thread issues tcgen05.mma kind::i8 with
// A = B = that block (D[i][j] += sum_t X[t][i] X[t][j], u8 x u8 -> s32 in
// TMEM, exact), so the diagonal is the per-expert count and the rest the
// pair counts, both symmetric halves. Rows with an out-of-range or repeated
// id are rejected like observe() does (profiler.py:76-80). At the end each
// CTA adds its 128 x 128 accumulator to the u64 counters.
constexpr int kTcBuild = 256;                // builder threads = tokens per stage
constexpr int kTcThreads = kTcBuild + 32;    // + the MMA warp
constexpr int kTcStages = 3;
constexpr uint32_t kTcSub = 128 * 128;       // one 128-token K block: 128 expert rows x 128 B
constexpr uint32_t kTcStage = 2 * kTcSub;    // 256 tokens
constexpr size_t kTcSmem = (size_t)kTcStages * kTcStage + 1024;
constexpr int kTcMaxK = 16;  // ids per token on the tensor-core path

template <int KC>
__global__ void __launch_bounds__(kTcThreads) coact_tc_kernel(const int32_t *__restrict__ topk, long long N, int k_rt,
                                                              int E, long long per_block,
                                                              unsigned long long *__restrict__ counts,
                                                              unsigned long long *__restrict__ pairs,
                                                              int *__restrict__ invalid) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[2 * kTcStages + 1];
    __shared__ uint32_t tmem_sh;
    const int tid = threadIdx.x, warp = tid >> 5;
    const unsigned lane = lane_id();
    const int k = KC > 0 ? KC : k_rt;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - ptx::smem_u32(smem_raw));
    const uint32_t full0 = ptx::smem_u32(&bars[0]), empty0 = ptx::smem_u32(&bars[kTcStages]),
                   done = ptx::smem_u32(&bars[2 * kTcStages]);
    const long long t0 = (long long)blockIdx.x * per_block, t1 = min(N, t0 + per_block);
    const long long nchunks = t1 > t0 ? (t1 - t0 + kTcBuild - 1) / kTcBuild : 0;
    if (tid == 0) {
        for (int s = 0; s < kTcStages; ++s) {
            ptx::mbar_init(full0 + 8 * s, kTcBuild);
            ptx::mbar_init(empty0 + 8 * s, 1);
        }
        ptx::mbar_init(done, 1);
        ptx::fence_barrier_init();
    }
    if (warp == kTcBuild / 32) ptx::tmem_alloc(ptx::smem_u32(&tmem_sh), 128);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_sh;
    if (warp < kTcBuild / 32) {
        // A builder thread owns one token column (sub, tl) of every stage. Each stage is zeroed
        // once; afterwards the thread clears only the bytes it set in that stage last time
        // (prev), so no barrier separates clearing from setting. The next chunk's ids are
        // loaded while the current one is built.
        constexpr int KM = KC > 0 ? KC : kTcMaxK;
        const int sub = tid >> 7, tl = tid & 127;
        const uint32_t col = (uint32_t)(tl & 15), chunk16 = (uint32_t)(tl >> 4);
        int bad = 0;
        int nxt[KM];
        bool nxt_ok = false;
        auto load_ids = [&](long long c, int (&id)[KM], bool &ok) {
            const long long t = t0 + c * kTcBuild + tid;
            ok = c < nchunks && t < t1;
            if (!ok) return;
            if constexpr (KC == 8) {
                const int4 *p = reinterpret_cast<const int4 *>(topk + t * 8);
                const int4 a = __ldg(p), b = __ldg(p + 1);
                id[0] = a.x; id[1] = a.y; id[2] = a.z; id[3] = a.w;
                id[4] = b.x; id[5] = b.y; id[6] = b.z; id[7] = b.w;
            } else {
#pragma unroll
                for (int x = 0; x < KM; ++x)
                    if (x < k) id[x] = __ldg(topk + t * k + x);
            }
        };
        load_ids(0, nxt, nxt_ok);
        // zero every stage once (all builders), then build
        {
            uint4 *z = reinterpret_cast<uint4 *>(base_ptr);
            for (int m = tid; m < (int)(kTcStages * kTcStage / 16); m += kTcBuild) z[m] = make_uint4(0, 0, 0, 0);
            ptx::named_bar_sync(1, kTcBuild);
        }
        int prev[kTcStages][KM];
        int prev_n[kTcStages] = {0, 0, 0};
        for (long long c0 = 0; c0 < nchunks; c0 += kTcStages) {
#pragma unroll
            for (int s = 0; s < kTcStages; ++s) {
                const long long c = c0 + s;
                if (c >= nchunks) break;
                const uint32_t ph = (uint32_t)((c / kTcStages) & 1);
                int id[KM];
                bool ok = nxt_ok;
#pragma unroll
                for (int x = 0; x < KM; ++x) id[x] = nxt[x];
                load_ids(c + 1, nxt, nxt_ok);  // in flight while this chunk is built
                if (ok) {
                    bool badrow = false;
#pragma unroll
                    for (int x = 0; x < KM; ++x) {
                        if (x >= k) break;
                        badrow |= (unsigned)id[x] >= (unsigned)E;
#pragma unroll
                        for (int y = 0; y < x; ++y) badrow |= id[x] == id[y];
                    }
                    if (badrow) {
                        ++bad;
                        ok = false;
                    }
                }
                ptx::mbar_wait(empty0 + 8 * s, ph ^ 1u);  // the MMAs that read this stage are done
                uint8_t *blk = base_ptr + (size_t)s * kTcStage + (size_t)sub * kTcSub;
#pragma unroll
                for (int x = 0; x < KM; ++x) {
                    if (x >= prev_n[s]) break;
                    const uint32_t e = (uint32_t)prev[s][x];
                    blk[e * 128u + (((chunk16 ^ (e & 7u)) << 4) | col)] = 0;
                }
                prev_n[s] = ok ? k : 0;
                if (ok) {
#pragma unroll
                    for (int x = 0; x < KM; ++x) {
                        if (x >= k) break;
                        const uint32_t e = (uint32_t)id[x];
                        prev[s][x] = id[x];
                        blk[e * 128u + (((chunk16 ^ (e & 7u)) << 4) | col)] = 1;
                    }
                }
                ptx::fence_proxy_async_shared();
                ptx::mbar_arrive(full0 + 8 * s);
            }
        }
        if (bad) atomicAdd(invalid, bad);
    } else if (lane == 0) {  // the MMA issuer
        const uint32_t idesc = ptx::idesc_u8_s32(128, 128);
        for (long long c = 0; c < nchunks; ++c) {
            const int s = (int)(c % kTcStages);
            const uint32_t ph = (uint32_t)((c / kTcStages) & 1);
            ptx::mbar_wait(full0 + 8 * s, ph);
            ptx::tc_fence_after();
#pragma unroll
            for (int sb = 0; sb < 2; ++sb) {
                const uint64_t d = ptx::sw128_desc(base + (uint32_t)s * kTcStage + (uint32_t)sb * kTcSub);
#pragma unroll
                for (int kk = 0; kk < 4; ++kk)  // K = 32 tokens per MMA: 32 bytes along the row
                    ptx::mma_i8(tmem, d + 2 * kk, d + 2 * kk, idesc, (c | sb | kk) != 0 ? 1u : 0u);
            }
            ptx::mma_commit(empty0 + 8 * s);
        }
        if (nchunks > 0) ptx::mma_commit(done);
    }
    // epilogue: warp w < 4 reads TMEM lanes 32w.. (rows i) x 128 columns (j)
    if (warp < 4 && nchunks > 0) {
        ptx::mbar_wait(done, 0);
        ptx::tc_fence_after();
        const int i = warp * 32 + (int)lane;
        for (int c0 = 0; c0 < 128; c0 += 16) {
            float v[16];
            ptx::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
            if (i >= E) continue;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int col = c0 + j;
                const unsigned long long n = (unsigned long long)__float_as_uint(v[j]);
                if (col >= E || n == 0) continue;
                if (col == i)
                    atomicAdd(&counts[i], n);
                else
                    atomicAdd(&pairs[(size_t)i * E + col], n);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == kTcBuild / 32) ptx::tmem_dealloc(tmem, 128);
}

// K6 on the FP4 tensor cores (E <= 128): the same X^T X, with the one-hot
// entries as packed e2m1 1.0 (a nibble per token: half the operand bytes of
// the u8 path, whose shared-memory traffic bound it) and block scales fixed
// at 1.0 in TMEM; f32 accumulation is exact while a CTA's counts stay below
// 2^24 (the launcher caps tokens per CTA). A builder warp owns one 16 KB
// stage of 256 tokens (expert rows of 128 B, 128B-swizzled, K-major): lane l
// takes tokens 8l..8l+7 = 32-bit word l of every row; the warp zeroes the
// stage with 16-byte stores, then each lane ORs a nibble per (token, id)
// into its own words. The MMA thread issues 4 kind::mxf4 MMAs (K = 64) per
// stage, A = B = the stage. Token order inside a row is irrelevant (the
// product sums over it), only the row = expert mapping matters.
constexpr int kF4Warps = 12;                       // builder warps = stages
constexpr int kF4Threads = (kF4Warps + 1) * 32;    // + the MMA warp
constexpr uint32_t kF4Stage = 128 * 128;           // 256 tokens x 128 expert rows, 4 bits each
constexpr size_t kF4Smem = (size_t)kF4Warps * kF4Stage + 1024;
constexpr long long kF4MaxPerBlock = 1LL << 23;    // f32-exact counts per CTA

// Transposed build (TB: the builder warps of BMOE_COACT_TB_MASK): lane = token. A lane turns
// its token's ids into a 128-bit expert mask in registers (rejecting the row
// when the mask's popcount is not k or a bit lies at or above E: exactly the
// out-of-range / duplicate test of profiler.py:76-80), the warp transposes
// each 32x32 bit block of (token, expert) with five xor-shuffle butterflies,
// and lane b then holds, for expert 32j + b, the bit set of its 32 tokens:
// one 16-byte chunk of that expert's row (word q, nibble n of the chunk <-
// token 4n + q, as e2m1 1.0). The warp writes whole chunks with 16-byte
// stores, 32 rows x one chunk per instruction: conflict-free under the 128B
// swizzle, no zero fill and no shared-memory atomics.
__device__ __forceinline__ uint32_t bit_transpose32(uint32_t x, unsigned lane) {
    // the two byte-granular stages are one PRMT each: lower lane [x0 x1 y0 y1] / [x0 y0 x2 y2],
    // upper lane [y2 y3 x2 x3] / [y1 x1 y3 x3] (y = the partner's word)
    uint32_t y = __shfl_xor_sync(0xffffffffu, x, 16);
    x = __byte_perm(x, y, (lane & 16u) ? 0x3276u : 0x5410u);
    y = __shfl_xor_sync(0xffffffffu, x, 8);
    x = __byte_perm(x, y, (lane & 8u) ? 0x3715u : 0x6240u);
#pragma unroll
    for (int s = 4; s >= 1; s >>= 1) {
        const uint32_t m = s == 4 ? 0x0F0F0F0Fu : s == 2 ? 0x33333333u : 0x55555555u;  // bits whose index has bit s clear
        const bool up = (lane & (unsigned)s) != 0;
        const uint32_t keep = up ? ~m : m;
        y = __shfl_xor_sync(0xffffffffu, x, s);
        // lower lane takes (y << s) & ~m, upper lane (y >> s) & m: both a rotation of y
        // (the wrapped bits fall outside the half taken)
        x = (x & keep) | (__funnelshift_l(y, y, up ? 32 - s : s) & ~keep);
    }
    return x;
}

template <int KC, bool TB>
__global__ void __launch_bounds__(kF4Threads) coact_fp4_kernel(const int32_t *__restrict__ topk, long long N, int k_rt,
                                                               int E, long long per_block,
                                                               unsigned long long *__restrict__ counts,
                                                               unsigned long long *__restrict__ pairs,
                                                               int *__restrict__ invalid, uint32_t tb_mask) {
    extern __shared__ uint8_t smem_raw[];
    __shared__ __align__(8) uint64_t bars[2 * kF4Warps + 1];
    __shared__ uint32_t tmem_sh;
    const int tid = threadIdx.x, warp = tid >> 5;
    const unsigned lane = lane_id();
    const int k = KC > 0 ? KC : k_rt;
    const uint32_t base = (ptx::smem_u32(smem_raw) + 1023u) & ~1023u;
    uint8_t *base_ptr = smem_raw + (base - ptx::smem_u32(smem_raw));
    const uint32_t full0 = ptx::smem_u32(&bars[0]), empty0 = ptx::smem_u32(&bars[kF4Warps]),
                   done = ptx::smem_u32(&bars[2 * kF4Warps]);
    const long long t0 = (long long)blockIdx.x * per_block, t1 = min(N, t0 + per_block);
    const long long nchunks = t1 > t0 ? (t1 - t0 + 255) / 256 : 0;
    if (tid == 0) {
        for (int s = 0; s < kF4Warps; ++s) {
            ptx::mbar_init(full0 + 8 * s, 1);
            ptx::mbar_init(empty0 + 8 * s, 1);
        }
        ptx::mbar_init(done, 1);
        ptx::fence_barrier_init();
    }
    // TMEM: accumulator columns [0, 128), block scales (all 1.0 = ue8m0 127) in [128, 144)
    if (warp == kF4Warps) ptx::tmem_alloc(ptx::smem_u32(&tmem_sh), 256);
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    const uint32_t tmem = tmem_sh;
    if (warp < 4) {
        ptx::tmem_fill8(tmem + ((uint32_t)(warp * 32) << 16) + 128u, 0x7F7F7F7Fu);
        ptx::tmem_fill8(tmem + ((uint32_t)(warp * 32) << 16) + 136u, 0x7F7F7F7Fu);
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp < kF4Warps) {
        constexpr int KM = KC > 0 ? KC : kTcMaxK;
        uint8_t *stage = base_ptr + (size_t)warp * kF4Stage;
        // lane's word in row e: 128B swizzle of 16-byte chunk (lane/4) by (e & 7)
        const uint32_t wcol = ((lane & 3u) << 2), wchunk = lane >> 2;
        int bad = 0;
        if (TB && ((tb_mask >> warp) & 1u)) {
            uint32_t okw[4];  // expert bits below E, per 32-expert word
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int n = min(max(E - 32 * j, 0), 32);
                okw[j] = n == 32 ? ~0u : ((1u << n) - 1u);
            }
            // k = 8: lane holds the ids of token tc0 + 32 g + lane for g = 0..7; group g of the
            // next stage is loaded as soon as group g of this one is turned into its mask
            constexpr int KP = KC == 8 ? 8 : 1;
            int4 ia[KP], ib[KP];
            auto load8 = [&](long long c, int g, int4 &a, int4 &b) {
                const long long t = t0 + c * 256 + 32 * g + (long long)lane;
                a = make_int4(-1, -1, -1, -1);
                b = a;
                if (c < nchunks && t < t1) {
                    const int4 *p = reinterpret_cast<const int4 *>(topk + t * 8);
                    a = __ldg(p);
                    b = __ldg(p + 1);
                }
            };
            if constexpr (KC == 8) {
#pragma unroll
                for (int g = 0; g < 8; ++g) load8(warp, g, ia[g], ib[g]);
            }
            for (long long c = warp, u = 0; c < nchunks; c += kF4Warps, ++u) {
                const long long tc0 = t0 + c * 256;
                ptx::mbar_wait(empty0 + 8 * warp, (uint32_t)(u & 1) ^ 1u);  // the MMAs that read the stage are done
#pragma unroll
                for (int g = 0; g < 8; ++g) {
                    const long long t = tc0 + 32 * g + (long long)lane;
                    // 128-bit expert mask as four words: bit (e - 32 j) of word j; shl clamps, so
                    // an id outside [0, 128) (negative ones wrap to huge) sets no bit
                    uint32_t w[4] = {0u, 0u, 0u, 0u};
#pragma unroll
                    for (int x = 0; x < KM; ++x) {
                        if (x >= k) break;
                        int v;
                        if constexpr (KC == 8) {
                            const int4 &q = x < 4 ? ia[g] : ib[g];
                            const int r = x & 3;
                            v = r == 0 ? q.x : r == 1 ? q.y : r == 2 ? q.z : q.w;
                        } else {
                            v = t < t1 ? __ldg(topk + t * k + x) : -1;
                        }
                        const uint32_t e = (uint32_t)v;
#pragma unroll
                        for (int j = 0; j < 4; ++j) w[j] |= ptx::shl_clamp(1u, e - 32u * (uint32_t)j);
                    }
                    if constexpr (KC == 8) load8(c + kF4Warps, g, ia[g], ib[g]);
                    const bool live = t < t1;
                    const bool ok = __popc(w[0]) + __popc(w[1]) + __popc(w[2]) + __popc(w[3]) == k &&
                                    ((w[0] & ~okw[0]) | (w[1] & ~okw[1]) | (w[2] & ~okw[2]) | (w[3] & ~okw[3])) == 0u;
                    if (live && !ok) ++bad;
#pragma unroll
                    for (int j = 0; j < 4; ++j) {
                        const uint32_t col = bit_transpose32(ok ? w[j] : 0u, lane);  // bit t: token 32g + t has expert 32j + lane
                        const uint32_t e = 32u * (uint32_t)j + lane;
                        // e2m1 1.0 (0b0010): the shifts are multiplies (FMA pipe), only the four
                        // masks use the integer ALU, which this build is bound by
                        const uint4 q = make_uint4((col * 2u) & 0x22222222u, col & 0x22222222u,
                                                   __umulhi(col, 0x80000000u) & 0x22222222u,
                                                   __umulhi(col, 0x40000000u) & 0x22222222u);
                        *reinterpret_cast<uint4 *>(stage + e * 128u + (((uint32_t)g ^ (e & 7u)) << 4)) = q;
                    }
                }
                ptx::fence_proxy_async_shared();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(full0 + 8 * warp);
            }
        } else
        for (long long c = warp, u = 0; c < nchunks; c += kF4Warps, ++u) {
            if constexpr (KC == 8) {
                // coalesced: lane l loads 16-byte piece i*32 + l of the chunk's ids, i.e. half
                // (l & 1) of token 16i + l/2; the partner lane holds the other half. Token
                // 16i + m goes to word m + 16 (i & 1), nibble i / 2 of its expert rows.
                const long long tc0 = t0 + c * 256;
                const int4 *p = reinterpret_cast<const int4 *>(topk + tc0 * 8);
                int4 v[16];
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const long long t = tc0 + 16 * i + (lane >> 1);
                    v[i] = t < t1 ? __ldg(p + i * 32 + lane) : make_int4(0, 0, 0, 0);
                }
                uint32_t okm = 0;
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    const long long t = tc0 + 16 * i + (lane >> 1);
                    int o[4];
                    o[0] = __shfl_xor_sync(0xffffffffu, v[i].x, 1);
                    o[1] = __shfl_xor_sync(0xffffffffu, v[i].y, 1);
                    o[2] = __shfl_xor_sync(0xffffffffu, v[i].z, 1);
                    o[3] = __shfl_xor_sync(0xffffffffu, v[i].w, 1);
                    if (t >= t1) continue;
                    const int a[8] = {v[i].x, v[i].y, v[i].z, v[i].w, o[0], o[1], o[2], o[3]};
                    bool badrow = false;
#pragma unroll
                    for (int x = 0; x < 8; ++x) {
                        badrow |= (unsigned)a[x] >= (unsigned)E;
#pragma unroll
                        for (int y = 0; y < x; ++y) badrow |= a[x] == a[y];
                    }
                    if (badrow) bad += (lane & 1) == 0;
                    else okm |= 1u << i;
                }
                ptx::mbar_wait(empty0 + 8 * warp, (uint32_t)(u & 1) ^ 1u);
                uint4 *z = reinterpret_cast<uint4 *>(stage);
#pragma unroll 8
                for (int m = (int)lane; m < (int)(kF4Stage / 16); m += 32) z[m] = make_uint4(0, 0, 0, 0);
                __syncwarp();
#pragma unroll
                for (int i = 0; i < 16; ++i) {
                    if (!((okm >> i) & 1u)) continue;
                    const uint32_t w = (lane >> 1) + 16u * (uint32_t)(i & 1), bit = 2u << (4 * (i >> 1));
                    const int ids[4] = {v[i].x, v[i].y, v[i].z, v[i].w};
#pragma unroll
                    for (int x = 0; x < 4; ++x) {
                        const uint32_t e = (uint32_t)ids[x];
                        atomicOr(reinterpret_cast<uint32_t *>(stage + e * 128u + ((((w >> 2) ^ (e & 7u)) << 4) |
                                                                                  ((w & 3u) << 2))),
                                 bit);  // e2m1 1.0
                    }
                }
                ptx::fence_proxy_async_shared();
                __syncwarp();
                if (lane == 0) ptx::mbar_arrive(full0 + 8 * warp);
                continue;
            }
            const long long tb = t0 + c * 256 + 8 * (long long)lane;
            int id[8][KM];
            uint32_t okm = 0;
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                const long long t = tb + j;
                if (t >= t1) break;
                if constexpr (KC == 8) {
                    const int4 *p = reinterpret_cast<const int4 *>(topk + t * 8);
                    const int4 a = __ldg(p), b = __ldg(p + 1);
                    id[j][0] = a.x; id[j][1] = a.y; id[j][2] = a.z; id[j][3] = a.w;
                    id[j][4] = b.x; id[j][5] = b.y; id[j][6] = b.z; id[j][7] = b.w;
                } else {
#pragma unroll
                    for (int x = 0; x < KM; ++x)
                        if (x < k) id[j][x] = __ldg(topk + t * k + x);
                }
                bool badrow = false;
#pragma unroll
                for (int x = 0; x < KM; ++x) {
                    if (x >= k) break;
                    badrow |= (unsigned)id[j][x] >= (unsigned)E;
#pragma unroll
                    for (int y = 0; y < x; ++y) badrow |= id[j][x] == id[j][y];
                }
                if (badrow) ++bad;
                else okm |= 1u << j;
            }
            ptx::mbar_wait(empty0 + 8 * warp, (uint32_t)(u & 1) ^ 1u);  // the MMAs that read the stage are done
            uint4 *z = reinterpret_cast<uint4 *>(stage);
#pragma unroll 8
            for (int m = (int)lane; m < (int)(kF4Stage / 16); m += 32) z[m] = make_uint4(0, 0, 0, 0);
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
                if (!((okm >> j) & 1u)) continue;
#pragma unroll
                for (int x = 0; x < KM; ++x) {
                    if (x >= k) break;
                    const uint32_t e = (uint32_t)id[j][x];
                    atomicOr(reinterpret_cast<uint32_t *>(stage + e * 128u + (((wchunk ^ (e & 7u)) << 4) | wcol)),
                             2u << (4 * j));  // e2m1 1.0
                }
            }
            ptx::fence_proxy_async_shared();
            __syncwarp();
            if (lane == 0) ptx::mbar_arrive(full0 + 8 * warp);
        }
        bad += __shfl_xor_sync(0xffffffffu, bad, 16);
        bad += __shfl_xor_sync(0xffffffffu, bad, 8);
        bad += __shfl_xor_sync(0xffffffffu, bad, 4);
        bad += __shfl_xor_sync(0xffffffffu, bad, 2);
        bad += __shfl_xor_sync(0xffffffffu, bad, 1);
        if (lane == 0 && bad) atomicAdd(invalid, bad);
    } else if (lane == 0) {  // the MMA issuer
        const uint32_t idesc = ptx::idesc_mxf4(128, 128);
        for (long long c = 0; c < nchunks; ++c) {
            const int s = (int)(c % kF4Warps);
            ptx::mbar_wait(full0 + 8 * s, (uint32_t)((c / kF4Warps) & 1));
            ptx::tc_fence_after();
            const uint64_t d = ptx::sw128_desc(base + (uint32_t)s * kF4Stage);
#pragma unroll
            for (int kk = 0; kk < 4; ++kk)  // K = 64 tokens per MMA: 32 bytes along the row
                ptx::mma_mxf4(tmem, d + 2 * kk, d + 2 * kk, idesc, tmem + 128u, tmem + 136u, (c | kk) != 0 ? 1u : 0u);
            ptx::mma_commit(empty0 + 8 * s);
        }
        if (nchunks > 0) ptx::mma_commit(done);
    }
    // epilogue: warp w < 4 reads TMEM lanes 32w.. (rows i) x 128 columns (j); counts are exact f32
    if (warp < 4 && nchunks > 0) {
        ptx::mbar_wait(done, 0);
        ptx::tc_fence_after();
        const int i = warp * 32 + (int)lane;
        for (int c0 = 0; c0 < 128; c0 += 16) {
            float v[16];
            ptx::tmem_ld16(tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0, v);
            if (i >= E) continue;
#pragma unroll
            for (int j = 0; j < 16; ++j) {
                const int col = c0 + j;
                const unsigned long long n = (unsigned long long)v[j];
                if (col >= E || n == 0) continue;
                if (col == i)
                    atomicAdd(&counts[i], n);
                else
                    atomicAdd(&pairs[(size_t)i * E + col], n);
            }
        }
    }
    ptx::tc_fence_before();
    __syncthreads();
    ptx::tc_fence_after();
    if (warp == kF4Warps) ptx::tmem_dealloc(tmem, 256);
}

__global__ void coact_weighted_kernel(const int32_t *__restrict__ topk, const float *__restrict__ probs, long long N,
                                      int k, int E, double w, double *__restrict__ pw) {
    const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= N) return;
    for (int x = 0; x < k; ++x) {
        const int i = topk[t * k + x];
        const double pa = probs[t * k + x];
        for (int y = x + 1; y < k; ++y) {
            const int j = topk[t * k + y];
            const double m = w * fmin(pa, (double)probs[t * k + y]);
            atomicAdd(&pw[(size_t)i * E + j], m);
            atomicAdd(&pw[(size_t)j * E + i], m);
        }
    }
}

// x + 1.0 applied n times with f64 rounding after every step, in O(#binades):
// inside a binade [2^m, 2^(m+1)) with m >= 0 adding 1.0 is exact until the
// result would reach 2^(m+1); only the crossing step rounds.
__device__ double add_ones_sequential(double x, unsigned long long n) {
    while (n > 0) {
        if (x >= 1.0 && x < 9007199254740992.0) {  // 2^53
            int ex;
            frexp(x, &ex);                      // x in [2^(ex-1), 2^ex)
            const double U = ldexp(1.0, ex);
            const double dd = dsub(U, x);       // exact
            unsigned long long j = (unsigned long long)ceil(dd) - 1ULL;  // steps keeping x + j < U
            if (j > n) j = n;
            x = dadd(x, (double)j);              // exact
            n -= j;
            if (n == 0) break;
        }
        x = dadd(x, 1.0);  // the one rounded step (or x < 1 / x >= 2^53)
        --n;
        if (x >= 9007199254740992.0) {
            // beyond 2^53 adding 1.0 rounds to even each step: x stays put
            // when its ulp is 2 and x + 1 ties to x. Fall back to stepping.
            while (n > 0) {
                double y = dadd(x, 1.0);
                if (y == x) { n = 0; break; }
                x = y;
                --n;
            }
        }
    }
    return x;
}

// Reference accumulation order per cell (profiler.py:81-95): the warm-up
// tokens (global index < warmup_steps) come first and each adds w, then
// every later token adds 1.0 — all sequentially in f64. w == 0 tokens are
// skipped (:83-84). Exact for any w, not only dyadic ones.
__global__ void counts_to_f64_kernel(const unsigned long long *warm, const unsigned long long *main_, long long n,
                                     double w, double *out) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= n) return;
    double x = 0.0;
    if (warm && w != 0.0) {
        const unsigned long long c = warm[i];
        for (unsigned long long t = 0; t < c; ++t) x = dadd(x, w);
    }
    out[i] = add_ones_sequential(x, main_[i]);
}

constexpr int kRankWarps = 4;
constexpr int kRankMaxE = 1024;

// rows_are_q: M already holds conditional rows q (cft_prefix on a given row);
// q_out / degenerate_out (optional) export profiler.conditional_row.
__global__ void __launch_bounds__(kRankWarps * 32) buddy_rank_kernel(const double *__restrict__ M, int E, double eps,
                                                                      double thr, int k_max, int32_t *ids,
                                                                      double *weights, int32_t *lens, int rows_are_q,
                                                                      double *q_out, uint8_t *degenerate_out, int R) {
    __shared__ double q[kRankWarps][kRankMaxE];
    __shared__ int order[kRankWarps][kRankMaxE];
    const int warp = threadIdx.x >> 5;
    const unsigned lane = lane_id();
    const int p = blockIdx.x * kRankWarps + warp;
    if (p >= R) return;
    double *qw = q[warp];
    int *ow = order[warp];
    // conditional_row (profiler.py:113-119): row + eps, diagonal forced to 0
    for (int j = lane; j < E; j += 32)
        qw[j] = rows_are_q ? M[(size_t)p * E + j] : ((j == p) ? 0.0 : dadd(M[(size_t)p * E + j], eps));
    __syncwarp();
    double total = 0.0;
    if (lane == 0) total = pairwise_sum(qw, E);
    total = __shfl_sync(0xffffffffu, total, 0);
    int32_t *oid = ids ? ids + (size_t)p * k_max : nullptr;
    double *ow_w = weights ? weights + (size_t)p * k_max : nullptr;
    if (degenerate_out && lane == 0) degenerate_out[p] = !(total > 0.0);
    if (!(total > 0.0)) {  // degenerate pivot -> empty list (buddies.py:118-123)
        for (int r = lane; r < k_max && oid; r += 32) {
            oid[r] = -1;
            ow_w[r] = 0.0;
        }
        if (q_out)
            for (int j = lane; j < E; j += 32) q_out[(size_t)p * E + j] = 0.0;
        if (lane == 0 && lens) lens[p] = 0;
        return;
    }
    if (!rows_are_q)
        for (int j = lane; j < E; j += 32) qw[j] = ddiv(qw[j], total);
    __syncwarp();
    if (q_out)
        for (int j = lane; j < E; j += 32) q_out[(size_t)p * E + j] = qw[j];
    if (!lens) return;  // conditional rows only
    // stable argsort(-q): rank = #(strictly larger) + #(equal with lower id)
    int nnz = 0;
    for (int j = lane; j < E; j += 32) {
        const double v = qw[j];
        int rank = 0;
        for (int i = 0; i < E; ++i) {
            const double u = qw[i];
            rank += (u > v || (u == v && i < j)) ? 1 : 0;
        }
        ow[rank] = j;
        nnz += (v != 0.0) ? 1 : 0;
    }
    for (int off = 16; off > 0; off >>= 1) nnz += __shfl_xor_sync(0xffffffffu, nnz, off);
    __syncwarp();
    // cft_prefix (buddies.py:86-95): sequential cumsum, first index >= alpha - tol
    int t = nnz;
    if (lane == 0) {
        double cum = 0.0;
        for (int r = 0; r < nnz; ++r) {
            cum = dadd(cum, qw[ow[r]]);
            if (cum >= thr) {
                t = r + 1;
                break;
            }
        }
    }
    t = __shfl_sync(0xffffffffu, t, 0);
    const int n = min(t, k_max);
    for (int r = lane; r < k_max; r += 32) {
        if (r < n) {
            oid[r] = ow[r];
            ow_w[r] = qw[ow[r]];
        } else {
            oid[r] = -1;
            ow_w[r] = 0.0;
        }
    }
    if (lane == 0) lens[p] = n;
}

}  // namespace
}  // namespace bm

using namespace bm;

extern "C" int bm_coact_count(const int32_t *topk, int64_t N, int64_t k, int64_t E, unsigned long long *counts,
                              unsigned long long *pairs, int32_t *invalid_rows, bm_stream_t stream) {
    BM_REQUIRE(N >= 0 && k >= 1 && k <= kMaxK && E >= 1 && E <= kMaxE && k <= E, BM_EINVAL,
               "bm_coact_count: bad shape N=%lld k=%lld E=%lld", (long long)N, (long long)k, (long long)E);
    BM_REQUIRE(counts && pairs && invalid_rows && (topk || N == 0), BM_EINVAL, "bm_coact_count: null pointer");
    if (N == 0) return BM_OK;
    // path (BMOE_COACT_TC, read per call: tests and benches switch it): 2 (default, E <= 128, k <= 16)
    // the kind::mxf4 tensor-core kernel, 0.84 / 0.99 ms on the 64M-token uniform / Zipf traces;
    // 0 the shared-memory atomics kernel (0.89 / 1.01 ms; any E); 1 the kind::i8 tensor-core
    // kernel (1.28 ms, bound by shared-memory traffic) -- DESIGN §7
    const char *tc_ev = getenv("BMOE_COACT_TC");
    const int tc_env = tc_ev ? atoi(tc_ev) : 2;
    if (tc_env == 2 && E <= 128 && k <= kTcMaxK && (k != 8 || (reinterpret_cast<uintptr_t>(topk) & 15) == 0)) {
        // builder warps (bit i = warp i) that build their one-hot tiles by register bit transposes
        // (BMOE_COACT_TB_MASK, default none: every warp ORs nibbles into shared memory). Measured on
        // the 64M-token trace (profiles/r2s_coact_mix.jsonl): ORs 0.84-0.87 ms (shared-memory bound),
        // transposes 0.95 ms (integer-ALU bound), mixes 1.47-1.65 ms (the transposes' shuffles queue
        // behind the ORs' bank-conflicted ATOMS on the same MIO pipe) -- DESIGN §7
        const char *mk = getenv("BMOE_COACT_TB_MASK");
        const uint32_t tb_mask = mk ? (uint32_t)strtoul(mk, nullptr, 0) & ((1u << kF4Warps) - 1u) : 0u;
        auto fk = tb_mask ? (k == 8 ? coact_fp4_kernel<8, true> : coact_fp4_kernel<0, true>)
                          : (k == 8 ? coact_fp4_kernel<8, false> : coact_fp4_kernel<0, false>);
        static bool fattr = false;
        if (!fattr) {
            for (auto f : {coact_fp4_kernel<8, true>, coact_fp4_kernel<0, true>, coact_fp4_kernel<8, false>,
                           coact_fp4_kernel<0, false>})
                BM_CUDA_TRY(cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kF4Smem));
            fattr = true;
        }
        long long blocks = (long long)sm_count();
        const long long need = (N + 4LL * 256 * kF4Warps - 1) / (4LL * 256 * kF4Warps);  // >= 4 stages per warp
        blocks = std::max(1LL, std::min(blocks, need));
        blocks = std::max(blocks, (N + kF4MaxPerBlock - 1) / kF4MaxPerBlock);
        const long long per_block = (N + blocks - 1) / blocks;
        fk<<<(unsigned)blocks, kF4Threads, kF4Smem, as_stream(stream)>>>(topk, N, (int)k, (int)E, per_block, counts,
                                                                         pairs, invalid_rows, tb_mask);
        BM_LAUNCH_CHECK();
        return BM_OK;
    }
    if (tc_env == 1 && E <= 128 && k <= kTcMaxK && (k != 8 || (reinterpret_cast<uintptr_t>(topk) & 15) == 0)) {
        auto tk = k == 8 ? coact_tc_kernel<8> : coact_tc_kernel<0>;
        static bool attr = false;
        if (!attr) {
            BM_CUDA_TRY(cudaFuncSetAttribute(coact_tc_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kTcSmem));
            BM_CUDA_TRY(cudaFuncSetAttribute(coact_tc_kernel<0>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)kTcSmem));
            attr = true;
        }
        int per_sm = 1;
        BM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tk, kTcThreads, kTcSmem));
        long long blocks = (long long)sm_count() * std::max(1, std::min(per_sm, 2));
        const long long need = (N + 4LL * kTcBuild - 1) / (4LL * kTcBuild);  // >= 4 stages per CTA
        blocks = std::max(1LL, std::min(blocks, need));
        const long long per_block = (N + blocks - 1) / blocks;
        tk<<<(unsigned)blocks, kTcThreads, kTcSmem, as_stream(stream)>>>(topk, N, (int)k, (int)E, per_block, counts,
                                                                         pairs, invalid_rows);
        BM_LAUNCH_CHECK();
        return BM_OK;
    }
    const size_t smem = (size_t)E * (E + 1) / 2 * sizeof(uint32_t);
    auto kern = k == 8 ? coact_count_kernel<8> : coact_count_kernel<0>;
    BM_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    int per_sm = 1;
    BM_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kCountThreads, smem));
    if (per_sm < 1) per_sm = 1;
    long long blocks = (long long)sm_count() * per_sm;
    // at least ~4 tokens per thread per block so the flush amortises
    long long min_per_block = 4LL * kCountThreads;
    long long need = (N + min_per_block - 1) / min_per_block;
    if (need < blocks) blocks = need;
    if (blocks < 1) blocks = 1;
    long long per_block = (N + blocks - 1) / blocks;
    if (k == 8 && (reinterpret_cast<uintptr_t>(topk) & 15) != 0) {
        BM_REQUIRE(false, BM_EINVAL, "bm_coact_count: k=8 trace must be 16-byte aligned");
    }
    kern<<<(unsigned)blocks, kCountThreads, smem, as_stream(stream)>>>(topk, N, (int)k, (int)E, per_block, counts,
                                                                       pairs, invalid_rows);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_coact_weighted(const int32_t *topk, const float *probs, int64_t N, int64_t k, int64_t E, double w,
                                 double *pair_weights, bm_stream_t stream) {
    BM_REQUIRE(N >= 0 && k >= 1 && E >= 1 && pair_weights && (N == 0 || (topk && probs)), BM_EINVAL,
               "bm_coact_weighted: bad args");
    if (N == 0 || w == 0.0) return BM_OK;
    coact_weighted_kernel<<<(unsigned)((N + 255) / 256), 256, 0, as_stream(stream)>>>(topk, probs, N, (int)k, (int)E,
                                                                                      w, pair_weights);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_counts_to_f64(const unsigned long long *warm, const unsigned long long *main_, int64_t n,
                                double w_warm, double *out, bm_stream_t stream) {
    BM_REQUIRE(main_ && out && n >= 0, BM_EINVAL, "bm_counts_to_f64: bad args");
    if (n == 0) return BM_OK;
    counts_to_f64_kernel<<<(unsigned)((n + 255) / 256), 256, 0, as_stream(stream)>>>(warm, main_, n, w_warm, out);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_buddy_rank(const double *pair_matrix, int64_t E, double eps, double alpha, int64_t k_max,
                             int32_t *ids, double *weights, int32_t *lens, bm_stream_t stream) {
    BM_REQUIRE(E >= 1 && E <= kRankMaxE, BM_EINVAL, "bm_buddy_rank: E=%lld out of range", (long long)E);
    BM_REQUIRE(alpha > 0.0 && alpha <= 1.0, BM_EINVAL, "alpha must be in (0, 1]");
    BM_REQUIRE(k_max >= 1, BM_EINVAL, "k_max must be >= 1");
    BM_REQUIRE(eps >= 0.0, BM_EINVAL, "laplace_eps must be nonnegative");
    BM_REQUIRE(pair_matrix && ids && weights && lens, BM_EINVAL, "bm_buddy_rank: null pointer");
    const double thr = alpha - 1e-9;  // buddies.py:25,94
    buddy_rank_kernel<<<(unsigned)((E + kRankWarps - 1) / kRankWarps), kRankWarps * 32, 0, as_stream(stream)>>>(
        pair_matrix, (int)E, eps, thr, (int)k_max, ids, weights, lens, 0, nullptr, nullptr, (int)E);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_conditional_rows(const double *pair_matrix, int64_t E, double eps, double *q_out,
                                   uint8_t *degenerate_out, bm_stream_t stream) {
    BM_REQUIRE(E >= 1 && E <= kRankMaxE && pair_matrix && q_out, BM_EINVAL, "bm_conditional_rows: bad args");
    BM_REQUIRE(eps >= 0.0, BM_EINVAL, "laplace_eps must be nonnegative");
    buddy_rank_kernel<<<(unsigned)((E + kRankWarps - 1) / kRankWarps), kRankWarps * 32, 0, as_stream(stream)>>>(
        pair_matrix, (int)E, eps, 0.0, 1, nullptr, nullptr, nullptr, 0, q_out, degenerate_out, (int)E);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_cft_prefix(const double *q_rows, int64_t R, int64_t E, double alpha, int32_t *t_out,
                             int32_t *order_out, uint8_t *degenerate_out, bm_stream_t stream) {
    BM_REQUIRE(R >= 0 && E >= 1 && E <= kRankMaxE && q_rows && t_out && order_out, BM_EINVAL,
               "bm_cft_prefix: bad args");
    BM_REQUIRE(alpha > 0.0 && alpha <= 1.0, BM_EINVAL, "alpha must be in (0, 1]");
    if (R == 0) return BM_OK;
    // k_max = E: the list length is min(t, nnz) exactly as cft_prefix returns it
    double *wscratch = nullptr;
    BM_CUDA_TRY(cudaMallocAsync(&wscratch, (size_t)R * E * sizeof(double), as_stream(stream)));
    buddy_rank_kernel<<<(unsigned)((R + kRankWarps - 1) / kRankWarps), kRankWarps * 32, 0, as_stream(stream)>>>(
        q_rows, (int)E, 0.0, alpha - 1e-9, (int)E, order_out, wscratch, t_out, 1, nullptr, degenerate_out, (int)R);
    BM_LAUNCH_CHECK();
    BM_CUDA_TRY(cudaFreeAsync(wscratch, as_stream(stream)));
    return BM_OK;
}
