// Exponent-coded expert transfer ("fetch codec"). New blobs use piece format
// v3 (xfer_v3.cuh: a per-piece Huffman code of the exponent, ~10.7 bits per
// value); format v2 below stays decodable and selectable (BMOE_XFER_FORMAT=2).
//
// The offloaded decode step is bound by PCIe: every on-demand miss moves a
// whole expert (336 MiB at the Mixtral shape) from the pinned host mirror
// into an HBM slot. bf16 weights carry little information in their exponent
// byte (a N(0, s) tensor has ~2.5 bits of exponent entropy), so the mirror
// stores each expert losslessly re-coded and the SMs rebuild the bf16 image
// in HBM as the pieces land. Per chunk of 2048 values:
//   - low byte = sign << 7 | mantissa, verbatim (8 bits);
//   - a 2-bit code per value: 0..2 = the chunk's three most frequent
//     exponents (t1), 3 = escape (two bit-planes: plane p byte t = bit p of
//     the codes of values 8t..8t+7);
//   - escaped values, in value order, carry a 3-bit second-level code packed
//     LSB-first into the chunk's level-2 stream: 0..6 = the next seven
//     exponents (t2), 7 = raw (the exponent sits in the piece's raw list as
//     {u16 position in chunk, u8 exponent}).
// ~10.9 bits per value for N(0, 1/fan_in) weights (v1, a flat 3-bit window
// code, took 11.2), bit-exact by construction.
//
// Blob (one expert)      : BlobHeader | pieces (256-byte aligned)
// Piece (<= 32M values)  : PieceHeader (32 B) | low[n] | planes[chunks][2][256] |
//                          meta[chunks] (24 B) | level-2 streams (+16 B slack) |
//                          raw[n_raw] (u32)
// Pieces are self-contained so a fetch streams them through a small staging
// ring: copy piece i+1 while piece i decodes (engine.cpp).
#include <stdlib.h>
#include <string.h>

#include <algorithm>
#include <vector>

#include "common.cuh"

namespace bm {
namespace {

constexpr int kChunk = 2048;
constexpr int kThreads = 256;
constexpr uint32_t kBlobMagic = 0x31435842u;   // "BXC1" (blob container)
constexpr uint32_t kPieceMagic = 0x32505842u;  // "BXP2" (piece format v2)

struct ChunkMeta {
    uint32_t t1;          // bytes 0..2: exponents of level-1 codes 0..2 (byte 3 = 0)
    uint32_t t2lo, t2hi;  // bytes 0..6: exponents of level-2 codes 0..6
    uint32_t l2off;       // byte offset of the chunk's level-2 stream in the piece's stream region
    uint32_t rawoff;      // first raw entry of the chunk in the piece's raw list
    uint32_t rawn;        // raw entries of the chunk
};
static_assert(sizeof(ChunkMeta) == 24, "chunk meta layout");

__host__ __device__ inline uint64_t align_up(uint64_t x, uint64_t a) { return (x + a - 1) / a * a; }

// exclusive block scan of one int per thread (256 threads)
__device__ __forceinline__ int block_exclusive_scan(int v, int *warp_tot) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    int x = v;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    if (lane == 31) warp_tot[warp] = x;
    __syncthreads();
    int pre = 0;
#pragma unroll
    for (int w = 0; w < kThreads / 32; ++w) pre += (w < warp) ? warp_tot[w] : 0;
    __syncthreads();  // warp_tot is reused by the next scan
    return pre + x - v;
}

__device__ __forceinline__ int warp_incl_scan(int x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

__device__ __forceinline__ const bm_xfer_piece_header *piece_at(const uint8_t *blob, int p) {
    const auto *bh = reinterpret_cast<const bm_xfer_blob_header *>(blob);
    return reinterpret_cast<const bm_xfer_piece_header *>(blob + bh->piece_off[p]);
}

__device__ __forceinline__ uint32_t byte_of(uint32_t lo, uint32_t hi, uint32_t i) {
    return __byte_perm(lo, hi, i) & 0xFFu;
}

#include "xfer_v3.cuh"

// Pass 1 of the encoder: per chunk, the three most frequent exponents (t1)
// and the next seven (t2), ties to the lower exponent; escape and raw counts.
__global__ void __launch_bounds__(kThreads) xfer_hist_kernel(const uint16_t *__restrict__ src, int64_t n_chunks,
                                                             ChunkMeta *__restrict__ meta_out,
                                                             uint32_t *__restrict__ n_esc_out) {
    __shared__ uint32_t hist[256];
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        hist[threadIdx.x] = 0;
        __syncthreads();
        const uint4 v = *reinterpret_cast<const uint4 *>(src + c * kChunk + threadIdx.x * 8);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            atomicAdd(&hist[(w[i] >> 7) & 0xFF], 1u);
            atomicAdd(&hist[(w[i] >> 23) & 0xFF], 1u);
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            uint32_t top[10], cov3 = 0, cov10 = 0;
            for (int r = 0; r < 10; ++r) {  // selection by count desc, exponent asc
                int best = -1;
                for (int b = 0; b < 256; ++b) {
                    bool used = false;
                    for (int q = 0; q < r; ++q) used |= top[q] == (uint32_t)b;
                    if (!used && (best < 0 || hist[b] > hist[best])) best = b;
                }
                top[r] = (uint32_t)best;
                if (r < 3) cov3 += hist[best];
                cov10 += hist[best];
            }
            ChunkMeta m;
            m.t1 = top[0] | (top[1] << 8) | (top[2] << 16);
            m.t2lo = top[3] | (top[4] << 8) | (top[5] << 16) | (top[6] << 24);
            m.t2hi = top[7] | (top[8] << 8) | (top[9] << 16);
            m.l2off = 0;
            m.rawoff = 0;
            m.rawn = kChunk - cov10;
            meta_out[c] = m;
            n_esc_out[c] = kChunk - cov3;
        }
        __syncthreads();
    }
}

// Pass 2 of the encoder: low bytes, level-1 planes, level-2 streams and raw
// entries of every chunk into its piece (headers and metas already in place,
// level-2 streams zeroed).
__global__ void __launch_bounds__(kThreads) xfer_pack_kernel(const uint16_t *__restrict__ src, int64_t n_chunks,
                                                             int64_t chunks_per_piece, uint8_t *__restrict__ blob) {
    __shared__ int warp_tot[kThreads / 32];
    const int t = threadIdx.x;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const int p = (int)(c / chunks_per_piece);
        const int64_t cl = c - (int64_t)p * chunks_per_piece;
        uint8_t *pb = const_cast<uint8_t *>(reinterpret_cast<const uint8_t *>(piece_at(blob, p)));
        const bm_xfer_piece_header ph = *reinterpret_cast<const bm_xfer_piece_header *>(pb);
        const ChunkMeta m = reinterpret_cast<const ChunkMeta *>(pb + ph.off_meta)[cl];
        const uint4 v = *reinterpret_cast<const uint4 *>(src + c * kChunk + t * 8);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        uint32_t lo[2] = {0, 0}, pl0 = 0, pl1 = 0;
        uint32_t c2[8], rawv[8];
        int n1 = 0, nr = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t x = (j & 1) ? (w[j >> 1] >> 16) : (w[j >> 1] & 0xFFFF);
            const uint32_t e = (x >> 7) & 0xFF;
            lo[j >> 2] |= (((x >> 8) & 0x80) | (x & 0x7F)) << (8 * (j & 3));
            uint32_t code = 3;
#pragma unroll
            for (int q = 2; q >= 0; --q)
                if (e == ((m.t1 >> (8 * q)) & 0xFF)) code = (uint32_t)q;
            pl0 |= (code & 1u) << j;
            pl1 |= ((code >> 1) & 1u) << j;
            if (code == 3) {
                uint32_t k2 = 7;
#pragma unroll
                for (int q = 6; q >= 0; --q)
                    if (e == byte_of(m.t2lo, m.t2hi, (uint32_t)q)) k2 = (uint32_t)q;
                c2[n1++] = k2;
                if (k2 == 7) rawv[nr++] = (uint32_t)(t * 8 + j) | (e << 16);
            }
        }
        const int pre1 = block_exclusive_scan(n1, warp_tot);
        const int prer = block_exclusive_scan(nr, warp_tot);
        *reinterpret_cast<uint2 *>(pb + sizeof(bm_xfer_piece_header) + cl * kChunk + t * 8) = make_uint2(lo[0], lo[1]);
        uint8_t *planes = pb + ph.off_planes + cl * 512;
        planes[t] = (uint8_t)pl0;
        planes[256 + t] = (uint8_t)pl1;
        uint32_t *l2 = reinterpret_cast<uint32_t *>(pb + ph.off_l2 + m.l2off);
        for (int i = 0; i < n1; ++i) {
            const uint32_t bit = 3u * (uint32_t)(pre1 + i);
            atomicOr(&l2[bit >> 5], c2[i] << (bit & 31));
            if ((bit & 31) > 29) atomicOr(&l2[(bit >> 5) + 1], c2[i] >> (32 - (bit & 31)));
        }
        uint32_t *raw = reinterpret_cast<uint32_t *>(pb + ph.off_raw) + m.rawoff + prer;
        for (int i = 0; i < nr; ++i) raw[i] = rawv[i];
        __syncthreads();
    }
}

// bits 0..3 of x -> bits 0, 4, 8, 12 (shifts OR-ed: a multiply would carry
// between the overlapping partial products)
__device__ __forceinline__ uint32_t spread4(uint32_t x) {
    x &= 0xFu;
    return (x | (x << 3) | (x << 6) | (x << 9)) & 0x1111u;
}

// 3 bits at relative bit r (0 <= r <= 125) of the 128-bit window {w0..w3},
// branch-free (selects + one funnel shift)
__device__ __forceinline__ uint32_t bits3(uint32_t w0, uint32_t w1, uint32_t w2, uint32_t w3, uint32_t r) {
    const uint32_t i = r >> 5;
    const uint32_t lo = i == 0 ? w0 : (i == 1 ? w1 : (i == 2 ? w2 : w3));
    const uint32_t hi = i == 0 ? w1 : (i == 1 ? w2 : w3);
    return __funnelshift_r(lo, hi, r & 31) & 7u;
}

// Decoder: a warp owns half a chunk (1024 values), a lane 32 consecutive
// values = one 32-bit word of each level-1 plane. Level-1 codes pick t1
// exponents for four values at once (PRMT with the codes as selectors);
// escaped values read their 3-bit level-2 code from a 128-bit window of the
// chunk's stream at 3 x (their escape index), raw ones search the chunk's
// (short) raw list. The upper half's escape prefix is the popcount of the
// lower half's plane words; no CTA barrier.
__device__ __forceinline__ void decode_half(const uint8_t *__restrict__ pb, const bm_xfer_piece_header &ph, int64_t c,
                                            int half, uint16_t *__restrict__ dst) {
    const int lane = threadIdx.x & 31, wi = half * 32 + lane;
    const uint4 *lo_p = reinterpret_cast<const uint4 *>(pb + sizeof(bm_xfer_piece_header) + c * kChunk + wi * 32);
    const uint4 la = __ldg(lo_p), lb = __ldg(lo_p + 1);
    const uint32_t *pw = reinterpret_cast<const uint32_t *>(pb + ph.off_planes + c * 512);
    const uint32_t w0 = __ldg(pw + wi), w1 = __ldg(pw + 64 + wi);
    const ChunkMeta *mp = reinterpret_cast<const ChunkMeta *>(pb + ph.off_meta) + c;
    const uint32_t t1 = __ldg(&mp->t1), t2lo = __ldg(&mp->t2lo), t2hi = __ldg(&mp->t2hi);
    const uint32_t l2off = __ldg(&mp->l2off), rawoff = __ldg(&mp->rawoff), rawn = __ldg(&mp->rawn);
    int before = 0;
    if (half) before = __popc(__ldg(pw + lane) & __ldg(pw + 64 + lane));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) before += half ? __shfl_xor_sync(0xffffffffu, before, o) : 0;
    const uint32_t escm = w0 & w1;
    const int mine = __popc(escm);
    const int pre = before + warp_incl_scan(mine) - mine;
    // 128-bit window of the level-2 stream starting at the word holding bit 3*pre
    const uint32_t sb = 3u * (uint32_t)pre;
    const uint32_t *l2 = reinterpret_cast<const uint32_t *>(pb + ph.off_l2 + l2off) + (sb >> 5);
    uint32_t x0 = 0, x1 = 0, x2 = 0, x3 = 0;
    if (mine) {
        x0 = __ldg(l2);
        x1 = __ldg(l2 + 1);
        x2 = __ldg(l2 + 2);
        x3 = __ldg(l2 + 3);
    }
    const uint32_t *raw = reinterpret_cast<const uint32_t *>(pb + ph.off_raw) + rawoff;
    const uint32_t lw[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
    uint32_t out[16];
    uint32_t r = sb & 31;  // window bit of the next escape
#pragma unroll
    for (int g = 0; g < 8; ++g) {
        // selector nibble j = level-1 code of value 4g + j
        const uint32_t sel = spread4(w0 >> (4 * g)) | (spread4(w1 >> (4 * g)) << 1);
        uint32_t e4 = __byte_perm(t1, 0, sel);  // code 3 picks t1's zero byte 3: patched below
        uint32_t em = (escm >> (4 * g)) & 0xFu;
        while (em) {  // the group's escapes, each consuming the next 3-bit level-2 code
            const int j = __ffs(em) - 1;
            em &= em - 1;
            const uint32_t k2 = bits3(x0, x1, x2, x3, r);
            r += 3;
            uint32_t e = byte_of(t2lo, t2hi, k2);  // code 7 selects t2hi's zero byte 3
            if (k2 == 7) {  // raw: the chunk's raw list, by position
                const uint32_t pos = (uint32_t)(wi * 32 + 4 * g + j);
                for (uint32_t i = 0; i < rawn; ++i) {
                    const uint32_t ent = __ldg(raw + i);
                    if ((ent & 0xFFFFu) == pos) e = (ent >> 16) & 0xFFu;
                }
            }
            e4 |= e << (8 * j);
        }
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t tl = __byte_perm(lw[g], 0, h ? 0x4342u : 0x4140u);  // low bytes -> [b, 0, b', 0]
            const uint32_t ep = __byte_perm(e4, 0, h ? 0x4342u : 0x4140u);
            out[2 * g + h] = (tl & 0x007F007Fu) | ((tl & 0x00800080u) << 8) | (ep << 7);
        }
    }
    uint4 *o = reinterpret_cast<uint4 *>(dst + c * kChunk + wi * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = make_uint4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
}

__global__ void __launch_bounds__(kThreads, 4) xfer_decode_piece_kernel(const uint8_t *__restrict__ piece,
                                                                     uint16_t *__restrict__ dst) {
    const int warps = kThreads / 32, warp = threadIdx.x >> 5;
    if (*reinterpret_cast<const uint32_t *>(piece) == kPieceMagic3) {  // v3: one warp per chunk
        __shared__ __align__(16) uint16_t table[1 << kTB];
        __shared__ uint32_t stage[kThreads / 32][kStageWords];
        const PieceV3 ph = *reinterpret_cast<const PieceV3 *>(piece);
        const uint4 *t = reinterpret_cast<const uint4 *>(piece + ph.off_table);
        for (int i = threadIdx.x; i < (2 << kTB) / 16; i += kThreads) reinterpret_cast<uint4 *>(table)[i] = __ldg(t + i);
        __syncthreads();
        for (uint32_t c = blockIdx.x * warps + warp; c < ph.n_chunks; c += gridDim.x * warps)
            x3_decode_chunk(piece, ph, c, table, stage[warp], dst);
        return;
    }
    const bm_xfer_piece_header ph = *reinterpret_cast<const bm_xfer_piece_header *>(piece);
    const int64_t units = (int64_t)ph.n_chunks * 2;
    for (int64_t u = (int64_t)blockIdx.x * warps + warp; u < units; u += (int64_t)gridDim.x * warps)
        decode_half(piece, ph, u >> 1, (int)(u & 1), dst);
}

// Whole blob, one warp per kC3 values: a v3 chunk, or the v2 half-chunks it spans.
__global__ void __launch_bounds__(kThreads, 4) xfer_decode_blob_kernel(const uint8_t *__restrict__ blob, int64_t n_values,
                                                                    uint16_t *__restrict__ dst) {
    const auto *bh = reinterpret_cast<const bm_xfer_blob_header *>(blob);
    const int64_t pv = bh->piece_values;
    const int warps = kThreads / 32;
    const int64_t units = (n_values + kC3 - 1) / kC3;
    for (int64_t u = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); u < units; u += (int64_t)gridDim.x * warps) {
        const int64_t v = u * kC3;
        const int p0 = (int)(v / pv);
        const uint8_t *pb0 = blob + bh->piece_off[p0];
        if (*reinterpret_cast<const uint32_t *>(pb0) == kPieceMagic3) {  // v3 pieces hold whole chunks
            const PieceV3 ph = *reinterpret_cast<const PieceV3 *>(pb0);
            x3_decode_chunk(pb0, ph, (uint32_t)((v - p0 * pv) / kC3),
                            reinterpret_cast<const uint16_t *>(pb0 + ph.off_table), nullptr, dst + p0 * pv);
            continue;
        }
        for (int h = 0; h < 2 * kC3 / kChunk; ++h) {
            const int64_t vh = v + (int64_t)h * (kChunk / 2);
            if (vh >= n_values) break;
            const int p = (int)(vh / pv);
            const int64_t vp = vh - p * pv;
            const uint8_t *pb = blob + bh->piece_off[p];
            const bm_xfer_piece_header ph = *reinterpret_cast<const bm_xfer_piece_header *>(pb);
            decode_half(pb, ph, vp / kChunk, (int)((vp / (kChunk / 2)) & 1), dst + p * pv);
        }
    }
}

int64_t header_bytes(int64_t n_pieces) {
    return (int64_t)align_up(sizeof(bm_xfer_blob_header) + sizeof(uint64_t) * (n_pieces + 1), 256);
}

// bytes of a chunk's level-2 stream (3 bits per escape, whole 32-bit words)
uint64_t l2_bytes(uint64_t n_esc) { return align_up((3 * n_esc + 7) / 8, 4); }

// piece layout for n_chunks chunks with l2 bytes of level-2 streams and n_raw raw entries
void piece_layout(int64_t n_chunks, uint64_t l2, uint64_t n_raw, bm_xfer_piece_header *h) {
    h->magic = kPieceMagic;
    h->n_chunks = (uint32_t)n_chunks;
    h->n_raw = (uint32_t)n_raw;
    uint64_t o = sizeof(bm_xfer_piece_header) + (uint64_t)n_chunks * kChunk;
    h->off_planes = (uint32_t)o;
    o += (uint64_t)n_chunks * 512;
    h->off_meta = (uint32_t)o;
    o = align_up(o + (uint64_t)n_chunks * sizeof(ChunkMeta), 16);
    h->off_l2 = (uint32_t)o;
    o = align_up(o + l2 + 16, 16);  // + slack: the decoder reads a 16-byte window
    h->off_raw = (uint32_t)o;
    o = align_up(o + 4 * n_raw, 256);
    h->bytes = (uint32_t)o;
}

// values per piece: BM_XFER_PIECE_VALUES, or BMOE_XFER_PIECE (a multiple of
// 2048, for A/B of the fetch pipeline's granularity); recorded in each blob
int64_t piece_values() {
    static const int64_t v = [] {
        const char *ev = getenv("BMOE_XFER_PIECE");
        const long long x = ev ? atoll(ev) : 0;
        return (x >= kChunk && x % kChunk == 0 && x <= (1LL << 30)) ? (int64_t)x : (int64_t)BM_XFER_PIECE_VALUES;
    }();
    return v;
}

// piece format of new blobs: BMOE_XFER_FORMAT = 2 or 3 (read per call, default 3);
// v3 needs pieces of whole kC3 chunks
int xfer_format() {
    const char *ev = getenv("BMOE_XFER_FORMAT");
    const int f = (ev && atoi(ev) == 2) ? 2 : 3;
    return (f == 3 && piece_values() % kC3 == 0) ? 3 : 2;
}

int grid_for(int64_t n_chunks) {
    const int64_t g = std::min<int64_t>(n_chunks, (int64_t)sm_count() * 8);
    return (int)std::max<int64_t>(g, 1);
}

}  // namespace
}  // namespace bm

using namespace bm;

extern "C" int64_t bm_xfer_blob_bound(int64_t n_values) {
    if (n_values <= 0 || n_values % kChunk) return -1;
    const int64_t n_chunks = n_values / kChunk;
    const int64_t cpp = piece_values() / kChunk;
    const int64_t n_pieces = (n_chunks + cpp - 1) / cpp;
    int64_t total = header_bytes(n_pieces);
    for (int64_t p = 0; p < n_pieces; ++p) {
        bm_xfer_piece_header h;
        const int64_t nc = std::min(cpp, n_chunks - p * cpp);
        piece_layout(nc, nc * l2_bytes(kChunk), (uint64_t)nc * kChunk, &h);  // worst case: every value raw
        int64_t b = h.bytes;
        if (piece_values() % kC3 == 0) {  // v3 worst case: every code kTB bits
            PieceV3 h3;
            const int64_t nv = nc * kChunk, nc3 = (nv + kC3 - 1) / kC3;
            x3_layout((uint32_t)nv, (uint32_t)nc3, (uint64_t)nc3 * (kC3 * kTB / 32), &h3);
            b = std::max<int64_t>(b, h3.bytes);
        }
        total += b;
    }
    return total;
}

namespace bm {
namespace {
// v3 encoder: exponent histograms per piece -> length-limited canonical
// Huffman tables (host) -> stream lengths per lane -> layout (host) -> pack.
int encode_v3(const uint16_t *src, int64_t n_values, uint8_t *blob, int64_t blob_cap, int64_t *blob_bytes_host,
              cudaStream_t s) {
    const int64_t pv = piece_values(), cpp = pv / kC3;
    const int64_t n_chunks = (n_values + kC3 - 1) / kC3, n_pieces = (n_values + pv - 1) / pv;
    uint32_t *d_hist = nullptr, *d_enc = nullptr;
    uint16_t *d_lens = nullptr;
    BM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&d_hist), n_pieces * 256 * 4, s));
    BM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&d_enc), n_pieces * 256 * 4, s));
    BM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&d_lens), n_chunks * 32 * 2, s));
    BM_CUDA_TRY(cudaMemsetAsync(d_hist, 0, n_pieces * 256 * 4, s));
    x3_hist_kernel<<<grid_for(n_chunks), 256, 0, s>>>(src, n_values, cpp, d_hist);
    BM_LAUNCH_CHECK();
    std::vector<uint32_t> hist(n_pieces * 256), enc(n_pieces * 256);
    std::vector<uint16_t> tables(n_pieces << kTB), lens(n_chunks * 32);
    BM_CUDA_TRY(cudaMemcpyAsync(hist.data(), d_hist, hist.size() * 4, cudaMemcpyDeviceToHost, s));
    BM_CUDA_TRY(cudaStreamSynchronize(s));
    for (int64_t p = 0; p < n_pieces; ++p) {
        uint8_t len[256];
        x3_code_lengths(hist.data() + p * 256, len);
        x3_tables(len, enc.data() + p * 256, tables.data() + (p << kTB));
    }
    BM_CUDA_TRY(cudaMemcpyAsync(d_enc, enc.data(), enc.size() * 4, cudaMemcpyHostToDevice, s));
    x3_lens_kernel<<<grid_for((n_chunks * 32 + 255) / 256), 256, 0, s>>>(src, n_values, cpp, d_enc, d_lens);
    BM_LAUNCH_CHECK();
    BM_CUDA_TRY(cudaMemcpyAsync(lens.data(), d_lens, lens.size() * 2, cudaMemcpyDeviceToHost, s));
    BM_CUDA_TRY(cudaStreamSynchronize(s));
    // layout: chunk stream bases and piece sizes
    const int64_t hb = header_bytes(n_pieces);
    std::vector<uint8_t> head(hb, 0);
    auto *bh = reinterpret_cast<bm_xfer_blob_header *>(head.data());
    bh->magic = kBlobMagic;
    bh->n_pieces = (uint32_t)n_pieces;
    bh->n_values = (uint64_t)n_values;
    bh->piece_values = (uint32_t)pv;
    std::vector<uint32_t> cbase(n_chunks);
    std::vector<PieceV3> phs(n_pieces);
    uint64_t off = hb;
    for (int64_t p = 0; p < n_pieces; ++p) {
        const int64_t c0 = p * cpp, nc = std::min(cpp, n_chunks - c0);
        uint64_t words = 0;
        for (int64_t c = c0; c < c0 + nc; ++c) {
            cbase[c] = (uint32_t)words;
            uint64_t bits = 0;
            for (int l = 0; l < 32; ++l) bits += lens[c * 32 + l];
            words += (bits + 31) / 32;
        }
        x3_layout((uint32_t)std::min<int64_t>(pv, n_values - p * pv), (uint32_t)nc, words, &phs[p]);
        bh->piece_off[p] = off;
        off += phs[p].bytes;
    }
    bh->piece_off[n_pieces] = off;
    BM_REQUIRE((int64_t)off <= blob_cap, BM_EINVAL, "bm_xfer_encode: blob_cap %lld < %llu bytes",
               (long long)blob_cap, (unsigned long long)off);
    BM_CUDA_TRY(cudaMemsetAsync(blob, 0, off, s));  // streams are OR-ed in
    BM_CUDA_TRY(cudaMemcpyAsync(blob, head.data(), hb, cudaMemcpyHostToDevice, s));
    for (int64_t p = 0; p < n_pieces; ++p) {
        uint8_t *pb = blob + bh->piece_off[p];
        const int64_t c0 = p * cpp, nc = std::min(cpp, n_chunks - c0);
        BM_CUDA_TRY(cudaMemcpyAsync(pb, &phs[p], sizeof(PieceV3), cudaMemcpyHostToDevice, s));
        BM_CUDA_TRY(cudaMemcpyAsync(pb + phs[p].off_table, tables.data() + (p << kTB), 2 << kTB,
                                    cudaMemcpyHostToDevice, s));
        BM_CUDA_TRY(cudaMemcpyAsync(pb + phs[p].off_lens, lens.data() + c0 * 32, nc * 64, cudaMemcpyHostToDevice, s));
        BM_CUDA_TRY(cudaMemcpyAsync(pb + phs[p].off_cbase, cbase.data() + c0, nc * 4, cudaMemcpyHostToDevice, s));
    }
    x3_pack_kernel<<<grid_for((n_chunks + 7) / 8), 256, 0, s>>>(src, n_values, cpp, d_enc, blob);
    BM_LAUNCH_CHECK();
    BM_CUDA_TRY(cudaStreamSynchronize(s));  // the host images above must outlive their copies
    BM_CUDA_TRY(cudaFreeAsync(d_hist, s));
    BM_CUDA_TRY(cudaFreeAsync(d_enc, s));
    BM_CUDA_TRY(cudaFreeAsync(d_lens, s));
    *blob_bytes_host = (int64_t)off;
    return BM_OK;
}
}  // namespace
}  // namespace bm

extern "C" int bm_xfer_encode(const uint16_t *src, int64_t n_values, uint8_t *blob, int64_t blob_cap,
                              int64_t *blob_bytes_host, bm_stream_t stream) {
    BM_REQUIRE(src && blob && blob_bytes_host, BM_EINVAL, "bm_xfer_encode: null argument");
    BM_REQUIRE(n_values > 0 && n_values % kChunk == 0, BM_EINVAL,
               "bm_xfer_encode: n_values (%lld) must be a positive multiple of %d", (long long)n_values, kChunk);
    BM_REQUIRE(((uintptr_t)src & 15) == 0 && ((uintptr_t)blob & 255) == 0, BM_EINVAL,
               "bm_xfer_encode: src must be 16-byte and blob 256-byte aligned");
    cudaStream_t s = as_stream(stream);
    if (xfer_format() == 3) return encode_v3(src, n_values, blob, blob_cap, blob_bytes_host, s);
    const int64_t n_chunks = n_values / kChunk;
    const int64_t cpp = piece_values() / kChunk;
    const int64_t n_pieces = (n_chunks + cpp - 1) / cpp;
    // pass 1: per-chunk exponent tables and escape / raw counts
    ChunkMeta *d_meta = nullptr;
    uint32_t *d_esc = nullptr;
    BM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&d_meta), n_chunks * sizeof(ChunkMeta), s));
    BM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&d_esc), n_chunks * 4, s));
    xfer_hist_kernel<<<grid_for(n_chunks), kThreads, 0, s>>>(src, n_chunks, d_meta, d_esc);
    BM_LAUNCH_CHECK();
    std::vector<ChunkMeta> meta(n_chunks);
    std::vector<uint32_t> esc(n_chunks);
    BM_CUDA_TRY(cudaMemcpyAsync(meta.data(), d_meta, n_chunks * sizeof(ChunkMeta), cudaMemcpyDeviceToHost, s));
    BM_CUDA_TRY(cudaMemcpyAsync(esc.data(), d_esc, n_chunks * 4, cudaMemcpyDeviceToHost, s));
    BM_CUDA_TRY(cudaStreamSynchronize(s));
    BM_CUDA_TRY(cudaFreeAsync(d_meta, s));
    BM_CUDA_TRY(cudaFreeAsync(d_esc, s));
    // piece headers and chunk metas (stream / raw offsets) on the host
    const int64_t hb = header_bytes(n_pieces);
    std::vector<uint8_t> head(hb, 0);
    auto *bh = reinterpret_cast<bm_xfer_blob_header *>(head.data());
    bh->magic = kBlobMagic;
    bh->n_pieces = (uint32_t)n_pieces;
    bh->n_values = (uint64_t)n_values;
    bh->piece_values = (uint32_t)piece_values();
    uint64_t off = hb;
    std::vector<bm_xfer_piece_header> phs(n_pieces);
    for (int64_t p = 0; p < n_pieces; ++p) {
        const int64_t c0 = p * cpp, nc = std::min(cpp, n_chunks - c0);
        uint64_t l2 = 0, nraw = 0;
        for (int64_t c = 0; c < nc; ++c) {
            ChunkMeta &m = meta[c0 + c];
            m.l2off = (uint32_t)l2;
            m.rawoff = (uint32_t)nraw;
            l2 += l2_bytes(esc[c0 + c]);
            nraw += m.rawn;
        }
        piece_layout(nc, l2, nraw, &phs[p]);
        bh->piece_off[p] = off;
        off += phs[p].bytes;
    }
    bh->piece_off[n_pieces] = off;
    BM_REQUIRE((int64_t)off <= blob_cap, BM_EINVAL, "bm_xfer_encode: blob_cap %lld < %llu bytes",
               (long long)blob_cap, (unsigned long long)off);
    BM_CUDA_TRY(cudaMemsetAsync(blob, 0, off, s));  // level-2 streams are OR-ed in
    BM_CUDA_TRY(cudaMemcpyAsync(blob, head.data(), hb, cudaMemcpyHostToDevice, s));
    for (int64_t p = 0; p < n_pieces; ++p) {
        uint8_t *pb = blob + bh->piece_off[p];
        const int64_t c0 = p * cpp, nc = std::min(cpp, n_chunks - c0);
        BM_CUDA_TRY(cudaMemcpyAsync(pb, &phs[p], sizeof(bm_xfer_piece_header), cudaMemcpyHostToDevice, s));
        BM_CUDA_TRY(cudaMemcpyAsync(pb + phs[p].off_meta, meta.data() + c0, nc * sizeof(ChunkMeta),
                                    cudaMemcpyHostToDevice, s));
    }
    xfer_pack_kernel<<<grid_for(n_chunks), kThreads, 0, s>>>(src, n_chunks, cpp, blob);
    BM_LAUNCH_CHECK();
    BM_CUDA_TRY(cudaStreamSynchronize(s));  // the host images above must outlive their copies
    *blob_bytes_host = (int64_t)off;
    return BM_OK;
}

extern "C" int bm_xfer_decode(const uint8_t *blob, uint16_t *dst, int64_t n_values, bm_stream_t stream) {
    BM_REQUIRE(blob && dst, BM_EINVAL, "bm_xfer_decode: null argument");
    BM_REQUIRE(n_values > 0 && n_values % kChunk == 0, BM_EINVAL, "bm_xfer_decode: bad n_values %lld",
               (long long)n_values);
    BM_REQUIRE(((uintptr_t)dst & 15) == 0 && ((uintptr_t)blob & 255) == 0, BM_EINVAL,
               "bm_xfer_decode: dst must be 16-byte and blob 256-byte aligned");
    xfer_decode_blob_kernel<<<grid_for((n_values + kC3 - 1) / kC3 / 8 + 1), kThreads, 0, as_stream(stream)>>>(
        blob, n_values, dst);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_xfer_decode_piece_ctas(const uint8_t *piece, uint16_t *dst, int64_t n_chunks, int32_t max_ctas,
                                         bm_stream_t stream) {
    BM_REQUIRE(piece && dst && n_chunks > 0 && max_ctas >= 0, BM_EINVAL, "bm_xfer_decode_piece: bad argument");
    BM_REQUIRE(((uintptr_t)dst & 15) == 0 && ((uintptr_t)piece & 255) == 0, BM_EINVAL,
               "bm_xfer_decode_piece: dst must be 16-byte and piece 256-byte aligned");
    int grid = grid_for(n_chunks / 4 + 1);
    if (max_ctas > 0) grid = std::min(grid, (int)max_ctas);
    xfer_decode_piece_kernel<<<grid, kThreads, 0, as_stream(stream)>>>(piece, dst);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_xfer_decode_piece(const uint8_t *piece, uint16_t *dst, int64_t n_chunks, bm_stream_t stream) {
    return bm_xfer_decode_piece_ctas(piece, dst, n_chunks, 0, stream);
}
