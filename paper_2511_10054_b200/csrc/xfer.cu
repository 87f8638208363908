// Exponent-coded expert transfer ("fetch codec").
//
// The offloaded decode step is bound by PCIe: every on-demand miss moves a
// whole expert (336 MiB at the Mixtral shape) from the pinned host mirror
// into an HBM slot. bf16 weights carry little information in their exponent
// byte (a N(0, s) tensor has ~2.5 bits of exponent entropy), so the mirror
// stores each expert losslessly re-coded and the SMs rebuild the bf16 image
// in HBM as the pieces land:
//   - low byte  = sign << 7 | mantissa (8 bits, stored verbatim);
//   - exponent  = 3-bit code c relative to a per-chunk window base
//                 (exp = base + c for c < 7), code 7 = escape, the exponent
//                 byte then comes from the chunk's escape stream in value order.
// 11.0-11.2 bits per value instead of 16, bit-exact by construction. A chunk
// is 2048 values = one 256-thread CTA x 8 values per thread: thread t owns
// values 8t..8t+7, reads 8 low bytes, one byte of each of the 3 code planes
// (plane p byte t = bit p of its 8 codes) and its escapes at the CTA-wide
// exclusive prefix of escape counts, then writes 16 bytes.
//
// Blob (one expert)      : BlobHeader | pieces (256-byte aligned)
// Piece (<= 32M values)  : PieceHeader (32 B) | low[n] | planes[chunks][3][256] |
//                          base[chunks] | escoff[chunks] u32 | esc[n_esc]
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
constexpr uint32_t kBlobMagic = 0x31435842u;   // "BXC1"
constexpr uint32_t kPieceMagic = 0x31505842u;  // "BXP1"

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
    return pre + x - v;
}

__device__ __forceinline__ const bm_xfer_piece_header *piece_at(const uint8_t *blob, int p) {
    const auto *bh = reinterpret_cast<const bm_xfer_blob_header *>(blob);
    return reinterpret_cast<const bm_xfer_piece_header *>(blob + bh->piece_off[p]);
}

// Pass 1 of the encoder: per chunk, the 7-binade window with the most values
// (ties to the lowest base) and the number of values outside it.
__global__ void __launch_bounds__(kThreads) xfer_hist_kernel(const uint16_t *__restrict__ src, int64_t n_chunks,
                                                             uint8_t *__restrict__ base_out,
                                                             uint32_t *__restrict__ esc_out) {
    __shared__ uint32_t hist[256];
    __shared__ uint32_t best[2];
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
            uint32_t s = 0, bs = 0, bb = 0;
            for (int b = 0; b < 7; ++b) s += hist[b];
            bs = s;
            for (int b = 1; b <= 249; ++b) {
                s += hist[b + 6] - hist[b - 1];
                if (s > bs) bs = s, bb = b;
            }
            best[0] = bb;
            best[1] = kChunk - bs;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            base_out[c] = (uint8_t)best[0];
            esc_out[c] = best[1];
        }
        __syncthreads();
    }
}

// Pass 2 of the encoder: write low bytes, code planes and the escapes of
// every chunk into its piece (headers and escape offsets already in place).
__global__ void __launch_bounds__(kThreads) xfer_pack_kernel(const uint16_t *__restrict__ src, int64_t n_chunks,
                                                             int64_t chunks_per_piece, uint8_t *__restrict__ blob) {
    __shared__ int warp_tot[kThreads / 32];
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const int p = (int)(c / chunks_per_piece);
        const int64_t cl = c - (int64_t)p * chunks_per_piece;
        const auto *ph = piece_at(blob, p);
        uint8_t *pb = const_cast<uint8_t *>(reinterpret_cast<const uint8_t *>(ph));
        const int base = pb[ph->off_base + cl];
        const uint4 v = *reinterpret_cast<const uint4 *>(src + c * kChunk + threadIdx.x * 8);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
        uint32_t lo[2] = {0, 0};
        uint32_t pl[3] = {0, 0, 0};
        uint8_t ex[8];
        int n_esc = 0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t x = (j & 1) ? (w[j >> 1] >> 16) : (w[j >> 1] & 0xFFFF);
            const uint32_t e = (x >> 7) & 0xFF;
            const uint32_t low = ((x >> 8) & 0x80) | (x & 0x7F);
            lo[j >> 2] |= low << (8 * (j & 3));
            uint32_t code = (e >= (uint32_t)base && e < (uint32_t)base + 7) ? e - base : 7;
            if (code == 7) ex[n_esc++] = (uint8_t)e;
#pragma unroll
            for (int q = 0; q < 3; ++q) pl[q] |= ((code >> q) & 1u) << j;
        }
        const int pre = block_exclusive_scan(n_esc, warp_tot);
        *reinterpret_cast<uint2 *>(pb + sizeof(bm_xfer_piece_header) + cl * kChunk + threadIdx.x * 8) =
            make_uint2(lo[0], lo[1]);
        uint8_t *planes = pb + ph->off_planes + cl * 768;
#pragma unroll
        for (int q = 0; q < 3; ++q) planes[q * 256 + threadIdx.x] = (uint8_t)pl[q];
        const uint32_t eo = reinterpret_cast<const uint32_t *>(pb + ph->off_escoff)[cl];
        for (int i = 0; i < n_esc; ++i) pb[ph->off_esc + eo + pre + i] = ex[i];
        __syncthreads();
    }
}

// Decoder core: chunk cl of piece ph -> 2048 bf16 at dst.
__device__ __forceinline__ void decode_chunk(const uint8_t *__restrict__ pb, const bm_xfer_piece_header &ph,
                                             int64_t cl, uint16_t *__restrict__ dst, int *warp_tot) {
    const int t = threadIdx.x;
    const uint2 lo = __ldg(reinterpret_cast<const uint2 *>(pb + sizeof(bm_xfer_piece_header) + cl * kChunk + t * 8));
    const uint8_t *planes = pb + ph.off_planes + cl * 768;
    const uint32_t p0 = __ldg(planes + t), p1 = __ldg(planes + 256 + t), p2 = __ldg(planes + 512 + t);
    const uint32_t esc = p0 & p1 & p2;
    const int pre = block_exclusive_scan(__popc(esc), warp_tot);
    const uint32_t base = __ldg(pb + ph.off_base + cl);
    const uint8_t *es = pb + ph.off_esc + __ldg(reinterpret_cast<const uint32_t *>(pb + ph.off_escoff) + cl) + pre;
    uint32_t out[4];
    int k = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t low = (((j < 4) ? lo.x : lo.y) >> (8 * (j & 3))) & 0xFF;
        const uint32_t code = ((p0 >> j) & 1u) | (((p1 >> j) & 1u) << 1) | (((p2 >> j) & 1u) << 2);
        uint32_t e = base + code;
        if (code == 7) e = __ldg(es + k++);
        const uint32_t x = ((low & 0x80) << 8) | (e << 7) | (low & 0x7F);
        if (j & 1)
            out[j >> 1] |= x << 16;
        else
            out[j >> 1] = x;
    }
    *reinterpret_cast<uint4 *>(dst + cl * kChunk + t * 8) = make_uint4(out[0], out[1], out[2], out[3]);
}

// Warp-granular decoder: a warp owns 256 values (one eighth of a chunk) and
// derives its escape prefix without a CTA barrier: the escape bits of the
// chunk's earlier threads are AND-ed from the code-plane words (L1 hits) and
// popcounted, then a warp scan places its own lanes. No __syncthreads, so
// the dependent escape loads of one warp overlap the others' streams.
__device__ __forceinline__ int warp_incl_scan(int x) {
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
    }
    return x;
}

__device__ __forceinline__ void decode_unit(const uint8_t *__restrict__ pb, const bm_xfer_piece_header &ph,
                                            int64_t c, int w, uint16_t *__restrict__ dst) {
    const int lane = threadIdx.x & 31, t = w * 32 + lane;
    const uint2 lo = __ldg(reinterpret_cast<const uint2 *>(pb + sizeof(bm_xfer_piece_header) + c * kChunk + t * 8));
    const uint8_t *planes = pb + ph.off_planes + c * 768;
    const uint32_t p0 = __ldg(planes + t), p1 = __ldg(planes + 256 + t), p2 = __ldg(planes + 512 + t);
    const uint32_t *pw = reinterpret_cast<const uint32_t *>(planes);
    int before = 0;  // escapes of threads 0 .. 32w-1 = plane words 0 .. 8w-1
    for (int i = lane; i < 8 * w; i += 32) before += __popc(__ldg(pw + i) & __ldg(pw + 64 + i) & __ldg(pw + 128 + i));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) before += __shfl_xor_sync(0xffffffffu, before, o);
    const int mine = __popc(p0 & p1 & p2);
    const int pre = before + warp_incl_scan(mine) - mine;
    const uint32_t base = __ldg(pb + ph.off_base + c);
    const uint8_t *es = pb + ph.off_esc + __ldg(reinterpret_cast<const uint32_t *>(pb + ph.off_escoff) + c) + pre;
    uint32_t out[4];
    int k = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const uint32_t low = (((j < 4) ? lo.x : lo.y) >> (8 * (j & 3))) & 0xFF;
        const uint32_t code = ((p0 >> j) & 1u) | (((p1 >> j) & 1u) << 1) | (((p2 >> j) & 1u) << 2);
        uint32_t e = base + code;
        if (code == 7) e = __ldg(es + k++);
        const uint32_t x = ((low & 0x80) << 8) | (e << 7) | (low & 0x7F);
        if (j & 1)
            out[j >> 1] |= x << 16;
        else
            out[j >> 1] = x;
    }
    *reinterpret_cast<uint4 *>(dst + c * kChunk + t * 8) = make_uint4(out[0], out[1], out[2], out[3]);
}

__global__ void __launch_bounds__(kThreads) xfer_decode_piece_warp_kernel(const uint8_t *__restrict__ piece,
                                                                          uint16_t *__restrict__ dst) {
    const bm_xfer_piece_header ph = *reinterpret_cast<const bm_xfer_piece_header *>(piece);
    const int warps = kThreads / 32;
    const int64_t units = (int64_t)ph.n_chunks * 8;
    for (int64_t u = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); u < units; u += (int64_t)gridDim.x * warps)
        decode_unit(piece, ph, u >> 3, (int)(u & 7), dst);
}

// Wide decoder (default): a warp owns half a chunk (1024 values), a lane 32
// consecutive values = one 32-bit word of each code plane. Every lane issues
// 2 x 16 B (low bytes) + 3 x 4 B (planes) loads up front and writes 64 B, so
// ~4x more bytes are in flight per thread than with 8 values per thread; the
// upper half's escape prefix is the popcount of the lower half's plane words.
__device__ __forceinline__ uint32_t expand_code(uint32_t w0, uint32_t w1, uint32_t w2, int j) {
    return ((w0 >> j) & 1u) | (((w1 >> j) & 1u) << 1) | (((w2 >> j) & 1u) << 2);
}

__device__ __forceinline__ void decode_half(const uint8_t *__restrict__ pb, const bm_xfer_piece_header &ph,
                                            int64_t c, int half, uint16_t *__restrict__ dst) {
    const int lane = threadIdx.x & 31, wi = half * 32 + lane;  // plane word / 32-value group in the chunk
    const uint4 *lo_p = reinterpret_cast<const uint4 *>(pb + sizeof(bm_xfer_piece_header) + c * kChunk + wi * 32);
    const uint4 la = __ldg(lo_p), lb = __ldg(lo_p + 1);
    const uint32_t *pw = reinterpret_cast<const uint32_t *>(pb + ph.off_planes + c * 768);
    const uint32_t w0 = __ldg(pw + wi), w1 = __ldg(pw + 64 + wi), w2 = __ldg(pw + 128 + wi);
    const uint32_t base = __ldg(pb + ph.off_base + c);
    const uint32_t eo = __ldg(reinterpret_cast<const uint32_t *>(pb + ph.off_escoff) + c);
    int before = 0;
    if (half) before = __popc(__ldg(pw + lane) & __ldg(pw + 64 + lane) & __ldg(pw + 128 + lane));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) before += half ? __shfl_xor_sync(0xffffffffu, before, o) : 0;
    const uint32_t escm = w0 & w1 & w2;
    const int mine = __popc(escm);
    const int pre = before + warp_incl_scan(mine) - mine;
    const uint8_t *es = pb + ph.off_esc + eo + pre;
    const uint32_t lw[8] = {la.x, la.y, la.z, la.w, lb.x, lb.y, lb.z, lb.w};
    const uint32_t base4 = base * 0x01010101u;
    uint32_t out[16];
    int k = 0;
#pragma unroll
    for (int g = 0; g < 8; ++g) {  // 4 values per step, SIMD within a register
        // the 4 exponents as bytes: bit j of each plane spread to byte j
        // ((x * 0x204081) & 0x01010101 moves bit i of a nibble to bit 8i)
        const uint32_t c4 = ((((w0 >> (4 * g)) & 0xFu) * 0x00204081u) & 0x01010101u) |
                            (((((w1 >> (4 * g)) & 0xFu) * 0x00204081u) & 0x01010101u) << 1) |
                            (((((w2 >> (4 * g)) & 0xFu) * 0x00204081u) & 0x01010101u) << 2);
        uint32_t e4 = c4 + base4;  // no carries: code <= 6 and base + 6 <= 255 unless escaped
        if ((escm >> (4 * g)) & 0xFu) {  // rare: rebuild the group byte by byte with its escapes
            e4 = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const uint32_t code = (c4 >> (8 * j)) & 0xFFu;
                const uint32_t e = code == 7 ? (uint32_t)__ldg(es + k++) : base + code;
                e4 |= e << (8 * j);
            }
        }
        // bf16 = sign << 15 | exp << 7 | mantissa, two per output word
#pragma unroll
        for (int h = 0; h < 2; ++h) {
            const uint32_t t = __byte_perm(lw[g], 0, h ? 0x4342u : 0x4140u);  // low bytes -> [b, 0, b', 0]
            const uint32_t ep = __byte_perm(e4, 0, h ? 0x4342u : 0x4140u);
            out[2 * g + h] = (t & 0x007F007Fu) | ((t & 0x00800080u) << 8) | (ep << 7);
        }
    }
    uint4 *o = reinterpret_cast<uint4 *>(dst + c * kChunk + wi * 32);
#pragma unroll
    for (int q = 0; q < 4; ++q) o[q] = make_uint4(out[4 * q], out[4 * q + 1], out[4 * q + 2], out[4 * q + 3]);
}

__global__ void __launch_bounds__(kThreads) xfer_decode_piece_wide_kernel(const uint8_t *__restrict__ piece,
                                                                          uint16_t *__restrict__ dst) {
    const bm_xfer_piece_header ph = *reinterpret_cast<const bm_xfer_piece_header *>(piece);
    const int warps = kThreads / 32;
    const int64_t units = (int64_t)ph.n_chunks * 2;
    for (int64_t u = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); u < units; u += (int64_t)gridDim.x * warps)
        decode_half(piece, ph, u >> 1, (int)(u & 1), dst);
}

__global__ void __launch_bounds__(kThreads) xfer_decode_blob_wide_kernel(const uint8_t *__restrict__ blob,
                                                                         int64_t n_chunks, uint16_t *__restrict__ dst) {
    const auto *bh = reinterpret_cast<const bm_xfer_blob_header *>(blob);
    const int64_t cpp = bh->piece_values / kChunk;
    const int warps = kThreads / 32;
    for (int64_t u = (int64_t)blockIdx.x * warps + (threadIdx.x >> 5); u < 2 * n_chunks;
         u += (int64_t)gridDim.x * warps) {
        const int64_t c = u >> 1;
        const int p = (int)(c / cpp);
        const uint8_t *pb = blob + bh->piece_off[p];
        const bm_xfer_piece_header ph = *reinterpret_cast<const bm_xfer_piece_header *>(pb);
        decode_half(pb, ph, c - (int64_t)p * cpp, (int)(u & 1), dst + (int64_t)p * bh->piece_values);
    }
}

__global__ void __launch_bounds__(kThreads) xfer_decode_piece_kernel(const uint8_t *__restrict__ piece,
                                                                     uint16_t *__restrict__ dst) {
    __shared__ int warp_tot[kThreads / 32];
    const bm_xfer_piece_header ph = *reinterpret_cast<const bm_xfer_piece_header *>(piece);
    for (int64_t c = blockIdx.x; c < ph.n_chunks; c += gridDim.x) {
        decode_chunk(piece, ph, c, dst, warp_tot);
        __syncthreads();
    }
}

__global__ void __launch_bounds__(kThreads) xfer_decode_blob_kernel(const uint8_t *__restrict__ blob, int64_t n_chunks,
                                                                    uint16_t *__restrict__ dst) {
    __shared__ int warp_tot[kThreads / 32];
    const auto *bh = reinterpret_cast<const bm_xfer_blob_header *>(blob);
    const int64_t cpp = bh->piece_values / kChunk;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        const int p = (int)(c / cpp);
        const uint8_t *pb = blob + bh->piece_off[p];
        const bm_xfer_piece_header ph = *reinterpret_cast<const bm_xfer_piece_header *>(pb);
        decode_chunk(pb, ph, c - (int64_t)p * cpp, dst + (int64_t)p * bh->piece_values, warp_tot);
        __syncthreads();
    }
}

int64_t header_bytes(int64_t n_pieces) {
    return (int64_t)align_up(sizeof(bm_xfer_blob_header) + sizeof(uint64_t) * (n_pieces + 1), 256);
}

// piece layout offsets for n_chunks chunks and n_esc escapes
void piece_layout(int64_t n_chunks, int64_t n_esc, bm_xfer_piece_header *h) {
    h->magic = kPieceMagic;
    h->n_chunks = (uint32_t)n_chunks;
    h->n_esc = (uint32_t)n_esc;
    uint64_t o = sizeof(bm_xfer_piece_header) + (uint64_t)n_chunks * kChunk;
    h->off_planes = (uint32_t)o;
    o += (uint64_t)n_chunks * 768;
    h->off_base = (uint32_t)o;
    o = align_up(o + n_chunks, 16);
    h->off_escoff = (uint32_t)o;
    o = align_up(o + 4 * n_chunks, 16);
    h->off_esc = (uint32_t)o;
    o = align_up(o + n_esc, 256);
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
        piece_layout(nc, nc * kChunk, &h);  // worst case: every value escapes
        total += h.bytes;
    }
    return total;
}

extern "C" int bm_xfer_encode(const uint16_t *src, int64_t n_values, uint8_t *blob, int64_t blob_cap,
                              int64_t *blob_bytes_host, bm_stream_t stream) {
    BM_REQUIRE(src && blob && blob_bytes_host, BM_EINVAL, "bm_xfer_encode: null argument");
    BM_REQUIRE(n_values > 0 && n_values % kChunk == 0, BM_EINVAL,
               "bm_xfer_encode: n_values (%lld) must be a positive multiple of %d", (long long)n_values, kChunk);
    BM_REQUIRE(((uintptr_t)src & 15) == 0 && ((uintptr_t)blob & 255) == 0, BM_EINVAL,
               "bm_xfer_encode: src must be 16-byte and blob 256-byte aligned");
    cudaStream_t s = as_stream(stream);
    const int64_t n_chunks = n_values / kChunk;
    const int64_t cpp = piece_values() / kChunk;
    const int64_t n_pieces = (n_chunks + cpp - 1) / cpp;
    // pass 1: per-chunk window bases and escape counts
    uint8_t *d_base = nullptr;
    uint32_t *d_esc = nullptr;
    BM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&d_base), n_chunks, s));
    BM_CUDA_TRY(cudaMallocAsync(reinterpret_cast<void **>(&d_esc), n_chunks * 4, s));
    xfer_hist_kernel<<<grid_for(n_chunks), kThreads, 0, s>>>(src, n_chunks, d_base, d_esc);
    BM_LAUNCH_CHECK();
    std::vector<uint8_t> base(n_chunks);
    std::vector<uint32_t> esc(n_chunks);
    BM_CUDA_TRY(cudaMemcpyAsync(base.data(), d_base, n_chunks, cudaMemcpyDeviceToHost, s));
    BM_CUDA_TRY(cudaMemcpyAsync(esc.data(), d_esc, n_chunks * 4, cudaMemcpyDeviceToHost, s));
    BM_CUDA_TRY(cudaStreamSynchronize(s));
    BM_CUDA_TRY(cudaFreeAsync(d_base, s));
    BM_CUDA_TRY(cudaFreeAsync(d_esc, s));
    // headers, bases and escape offsets (host), then pass 2 (device)
    const int64_t hb = header_bytes(n_pieces);
    std::vector<uint8_t> head(hb, 0);
    auto *bh = reinterpret_cast<bm_xfer_blob_header *>(head.data());
    bh->magic = kBlobMagic;
    bh->n_pieces = (uint32_t)n_pieces;
    bh->n_values = (uint64_t)n_values;
    bh->piece_values = (uint32_t)piece_values();
    uint64_t off = hb;
    std::vector<std::vector<uint8_t>> meta(n_pieces);
    for (int64_t p = 0; p < n_pieces; ++p) {
        const int64_t c0 = p * cpp, nc = std::min(cpp, n_chunks - c0);
        int64_t ne = 0;
        for (int64_t c = 0; c < nc; ++c) ne += esc[c0 + c];
        bm_xfer_piece_header ph;
        piece_layout(nc, ne, &ph);
        bh->piece_off[p] = off;
        // piece header + base + escoff (the region past low/planes), written as one host image
        std::vector<uint8_t> &m = meta[p];
        m.assign(ph.off_esc, 0);
        memcpy(m.data(), &ph, sizeof(ph));
        memcpy(m.data() + ph.off_base, base.data() + c0, nc);
        uint32_t acc = 0;
        for (int64_t c = 0; c < nc; ++c) {
            reinterpret_cast<uint32_t *>(m.data() + ph.off_escoff)[c] = acc;
            acc += esc[c0 + c];
        }
        off += ph.bytes;
    }
    bh->piece_off[n_pieces] = off;
    BM_REQUIRE((int64_t)off <= blob_cap, BM_EINVAL, "bm_xfer_encode: blob_cap %lld < %llu bytes",
               (long long)blob_cap, (unsigned long long)off);
    BM_CUDA_TRY(cudaMemsetAsync(blob, 0, off, s));
    BM_CUDA_TRY(cudaMemcpyAsync(blob, head.data(), hb, cudaMemcpyHostToDevice, s));
    for (int64_t p = 0; p < n_pieces; ++p) {
        const bm_xfer_piece_header *ph = reinterpret_cast<const bm_xfer_piece_header *>(meta[p].data());
        uint8_t *pb = blob + bh->piece_off[p];
        BM_CUDA_TRY(cudaMemcpyAsync(pb, meta[p].data(), sizeof(bm_xfer_piece_header), cudaMemcpyHostToDevice, s));
        BM_CUDA_TRY(cudaMemcpyAsync(pb + ph->off_base, meta[p].data() + ph->off_base, ph->off_esc - ph->off_base,
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
    const int64_t n_chunks = n_values / kChunk;
    if (const char *ev = getenv("BMOE_XFER_DECODER"); ev && atoi(ev) == 1)
        xfer_decode_blob_kernel<<<grid_for(n_chunks), kThreads, 0, as_stream(stream)>>>(blob, n_chunks, dst);
    else
        xfer_decode_blob_wide_kernel<<<grid_for(n_chunks / 4 + 1), kThreads, 0, as_stream(stream)>>>(blob, n_chunks,
                                                                                                    dst);
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_xfer_decode_piece(const uint8_t *piece, uint16_t *dst, int64_t n_chunks, bm_stream_t stream) {
    BM_REQUIRE(piece && dst && n_chunks > 0, BM_EINVAL, "bm_xfer_decode_piece: bad argument");
    BM_REQUIRE(((uintptr_t)dst & 15) == 0 && ((uintptr_t)piece & 255) == 0, BM_EINVAL,
               "bm_xfer_decode_piece: dst must be 16-byte and piece 256-byte aligned");
    static const int variant = [] {
        const char *ev = getenv("BMOE_XFER_DECODER");
        return ev ? atoi(ev) : 3;
    }();
    if (variant == 1)
        xfer_decode_piece_kernel<<<grid_for(n_chunks), kThreads, 0, as_stream(stream)>>>(piece, dst);
    else if (variant == 2)
        xfer_decode_piece_warp_kernel<<<grid_for(n_chunks), kThreads, 0, as_stream(stream)>>>(piece, dst);
    else
        xfer_decode_piece_wide_kernel<<<grid_for(n_chunks / 4 + 1), kThreads, 0, as_stream(stream)>>>(piece, dst);
    BM_LAUNCH_CHECK();
    return BM_OK;
}
