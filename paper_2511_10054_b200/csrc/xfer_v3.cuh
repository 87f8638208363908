// Fetch codec, piece format v3 ("BXP3"): per-piece canonical Huffman code of
// the exponent byte, sign+mantissa byte verbatim. Included by xfer.cu inside
// its anonymous namespace (uses warp_incl_scan and align_up from there).
//
// v2 spends ~2.9 bits per exponent (2-bit plane + 3-bit second level + raw
// entries + per-chunk tables); the exponent entropy of N(0, s) weights is
// ~2.55 bits and a Huffman code reaches ~2.58. One code per piece (a piece is
// 32M values of one matrix region, its exponent statistics are stationary),
// lengths limited to 12 bits so one 4096-entry table lookup decodes a symbol.
//
// Piece: PieceV3 (32 B) | low[n_values] (sign<<7 | mantissa) |
//        table[4096] u16 ((len << 8) | exponent, indexed by the next 12 stream bits) |
//        lens[n_chunks][32] u16 (bits of each lane's stream) |
//        cbase[n_chunks] u32 (first stream word of the chunk) |
//        streams (32-bit words, + 32 B slack)
// A chunk is 8192 values (the last one of a piece may hold fewer, always a
// multiple of 2048); lane l of the chunk's warp owns the groups of 16 values
// g*32 + l (g = 0 .. chunk values / 512 - 1), so the warp's loads and stores
// of a step cover one contiguous 512-value span, and the lane's codes (its
// groups in order) form one LSB-first bit stream; the chunk's 32 streams are
// bit-contiguous from word cbase, lane l starting at the sum of lens of lanes
// < l (a warp scan).
// The exponent of a value is the symbol whose bit-reversed canonical code
// is a prefix of the stream at that point.

constexpr int kC3 = 8192;                       // values per chunk
constexpr int kTB = 12;                         // table bits = maximum code length
constexpr uint32_t kPieceMagic3 = 0x33505842u;  // "BXP3"

struct PieceV3 {
    uint32_t magic, n_chunks, n_values;
    uint32_t off_table, off_lens, off_cbase, off_streams, bytes;
};
static_assert(sizeof(PieceV3) == 32, "piece header size");

constexpr int kStageWords = 1024;  // per warp: a chunk's streams up to 4 bits per value

// The lanes' decode loop over a word source: the chunk's stream words staged
// in shared memory (kStaged) or read from the piece. Each lane rebuilds its
// `per` values, one 16-value group per iteration (one 16-byte load of low
// bytes, issued two groups ahead; 16 table lookups; two 16-byte stores; the
// warp's accesses of an iteration are contiguous). w = the lane's first word.
template <bool kStaged>
__device__ __forceinline__ void x3_decode_lanes(const uint32_t *w, uint32_t start, const uint4 *lo, uint4 *o,
                                                uint32_t per, const uint16_t *table) {
    auto word = [&](uint32_t i) -> uint32_t { return kStaged ? w[i] : __ldg(w + i); };
    uint64_t buf = ((uint64_t)word(0) | ((uint64_t)word(1) << 32)) >> (start & 31);
    int nbits = 64 - (int)(start & 31);
    uint32_t wi = 2, nxt = word(2);
    const uint32_t groups = per >> 4;
    uint4 l0 = __ldg(lo), l1 = __ldg(lo + 32 * min(1u, groups - 1));
    for (uint32_t g = 0; g < groups; ++g) {
        const uint4 l2 = __ldg(lo + 32 * min(g + 2, groups - 1));
        const uint32_t lw[4] = {l0.x, l0.y, l0.z, l0.w};
        uint32_t out[8];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            uint32_t e4 = 0;
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                if ((j & 1) == 0 && nbits < 32) {  // >= 32 bits cover the next two codes (<= 12 bits each)
                    buf |= (uint64_t)nxt << nbits;
                    nbits += 32;
                    nxt = word(++wi);
                }
                const uint32_t ent = table[(uint32_t)buf & ((1u << kTB) - 1)];
                const uint32_t len = ent >> 8;
                buf >>= len;
                nbits -= (int)len;
                e4 |= (ent & 0xFFu) << (8 * j);
            }
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const uint32_t tl = __byte_perm(lw[q], 0, h ? 0x4342u : 0x4140u);  // [b, 0, b', 0]
                const uint32_t ep = __byte_perm(e4, 0, h ? 0x4342u : 0x4140u);
                out[2 * q + h] = (tl & 0x007F007Fu) | ((tl & 0x00800080u) << 8) | (ep << 7);
            }
        }
        o[64 * g] = make_uint4(out[0], out[1], out[2], out[3]);
        o[64 * g + 1] = make_uint4(out[4], out[5], out[6], out[7]);
        l0 = l1;
        l1 = l2;
    }
}

// Decode one chunk (one warp). With a staging buffer (stage: kStageWords
// warp-private shared words) the chunk's stream words are first copied in
// with coalesced loads, so a refill is a shared-memory read instead of a
// dependent global load; chunks whose streams exceed it read the piece.
__device__ __forceinline__ void x3_decode_chunk(const uint8_t *__restrict__ pb, const PieceV3 &ph, uint32_t c,
                                                const uint16_t *table, uint32_t *stage, uint16_t *__restrict__ dst) {
    const int lane = threadIdx.x & 31;
    const uint32_t v0 = c * (uint32_t)kC3;
    const uint32_t nv = min((uint32_t)kC3, ph.n_values - v0);
    const uint32_t per = nv >> 5;  // a multiple of 64
    const uint32_t my = __ldg(reinterpret_cast<const uint16_t *>(pb + ph.off_lens) + (size_t)c * 32 + lane);
    const uint32_t end = (uint32_t)warp_incl_scan((int)my), start = end - my;
    const uint32_t cb = __ldg(reinterpret_cast<const uint32_t *>(pb + ph.off_cbase) + c);
    const uint32_t *gw = reinterpret_cast<const uint32_t *>(pb + ph.off_streams) + cb;
    const uint4 *lo = reinterpret_cast<const uint4 *>(pb + sizeof(PieceV3) + v0) + lane;  // 16 low bytes per group
    uint4 *o = reinterpret_cast<uint4 *>(dst + v0) + 2 * lane;                           // 16 bf16 per group
    // words a lane may touch: its stream plus up to 3 words of read-ahead (in the piece: slack)
    const uint32_t need = (__shfl_sync(0xffffffffu, end, 31) + 31) / 32 + 3;
    if (stage != nullptr && need <= (uint32_t)kStageWords) {
        for (uint32_t i = lane; i < need; i += 32) stage[i] = __ldg(gw + i);
        __syncwarp();
        x3_decode_lanes<true>(stage + (start >> 5), start, lo, o, per, table);
        __syncwarp();  // the next chunk of this warp overwrites the stage
    } else {
        x3_decode_lanes<false>(gw + (start >> 5), start, lo, o, per, table);
    }
}

// ------------------------------------------------------------------ encoder

// Exponent histogram per piece (pieces of cpp chunks of kC3 values).
__global__ void __launch_bounds__(256) x3_hist_kernel(const uint16_t *__restrict__ src, int64_t n_values, int64_t cpp,
                                                      uint32_t *__restrict__ hist) {
    __shared__ uint32_t h[256];
    const int64_t n_chunks = (n_values + kC3 - 1) / kC3;
    for (int64_t c = blockIdx.x; c < n_chunks; c += gridDim.x) {
        h[threadIdx.x] = 0;
        __syncthreads();
        const int64_t v0 = c * kC3, nv = min((int64_t)kC3, n_values - v0);
        for (int64_t i = threadIdx.x; i < nv / 8; i += blockDim.x) {
            const uint4 v = *reinterpret_cast<const uint4 *>(src + v0 + 8 * i);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                atomicAdd(&h[(w[k] >> 7) & 0xFF], 1u);
                atomicAdd(&h[(w[k] >> 23) & 0xFF], 1u);
            }
        }
        __syncthreads();
        if (h[threadIdx.x]) atomicAdd(&hist[(c / cpp) * 256 + threadIdx.x], h[threadIdx.x]);
        __syncthreads();
    }
}

// One thread per (chunk, lane): its stream length in bits (enc[p][e] = code | len << 16).
__global__ void __launch_bounds__(256) x3_lens_kernel(const uint16_t *__restrict__ src, int64_t n_values, int64_t cpp,
                                                      const uint32_t *__restrict__ enc, uint16_t *__restrict__ lens) {
    const int64_t n_chunks = (n_values + kC3 - 1) / kC3;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n_chunks * 32;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int64_t c = i >> 5;
        const int lane = (int)(i & 31);
        const int64_t v0 = c * kC3, per = min((int64_t)kC3, n_values - v0) >> 5;
        const uint32_t *e = enc + (c / cpp) * 256;
        const uint16_t *s = src + v0 + 16 * lane;
        uint32_t bits = 0;
        for (int64_t k = 0; k < per; k += 8) {  // group k/16 of the lane: values (k/16*32 + lane)*16 + k%16
            const uint4 v = *reinterpret_cast<const uint4 *>(s + (k >> 4) * 512 + (k & 15));
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int q = 0; q < 4; ++q)
                bits += (__ldg(e + ((w[q] >> 7) & 0xFF)) >> 16) + (__ldg(e + ((w[q] >> 23) & 0xFF)) >> 16);
        }
        lens[i] = (uint16_t)bits;
    }
}

// One warp per chunk, one lane per stream: low bytes and the lane's codes
// (OR-ed into the zeroed stream region: neighbouring lanes share boundary words).
__global__ void __launch_bounds__(256) x3_pack_kernel(const uint16_t *__restrict__ src, int64_t n_values, int64_t cpp,
                                                      const uint32_t *__restrict__ enc, uint8_t *__restrict__ blob) {
    const int64_t n_chunks = (n_values + kC3 - 1) / kC3;
    const int lane = threadIdx.x & 31;
    const auto *bh = reinterpret_cast<const bm_xfer_blob_header *>(blob);
    for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < n_chunks;
         c += ((int64_t)gridDim.x * blockDim.x) >> 5) {
        const int64_t p = c / cpp, cl = c - p * cpp;
        uint8_t *pb = blob + bh->piece_off[p];
        const PieceV3 ph = *reinterpret_cast<const PieceV3 *>(pb);
        const int64_t v0 = c * kC3, per = min((int64_t)kC3, n_values - v0) >> 5;
        const uint32_t my = reinterpret_cast<const uint16_t *>(pb + ph.off_lens)[cl * 32 + lane];
        const uint32_t start = (uint32_t)warp_incl_scan((int)my) - my;
        const uint32_t cb = reinterpret_cast<const uint32_t *>(pb + ph.off_cbase)[cl];
        uint32_t *words = reinterpret_cast<uint32_t *>(pb + ph.off_streams) + cb + (start >> 5);
        const uint32_t *e = enc + p * 256;
        const uint16_t *s = src + v0 + 16 * lane;
        uint8_t *low = pb + sizeof(PieceV3) + (cl * kC3) + 16 * lane;
        uint64_t acc = 0;
        int nacc = (int)(start & 31);
        for (int64_t k = 0; k < per; k += 16) {
            const uint16_t *sg = s + (k >> 4) * 512;  // the lane's group k/16
            const uint4 va = *reinterpret_cast<const uint4 *>(sg), vb = *reinterpret_cast<const uint4 *>(sg + 8);
            const uint32_t w[8] = {va.x, va.y, va.z, va.w, vb.x, vb.y, vb.z, vb.w};
            uint32_t lb[4];
#pragma unroll
            for (int q = 0; q < 8; ++q) {
                const uint32_t a = w[q] & 0xFFFF, b = w[q] >> 16;
                const uint32_t la = ((a >> 8) & 0x80) | (a & 0x7F), lbb = ((b >> 8) & 0x80) | (b & 0x7F);
                const uint32_t two = la | (lbb << 8);
                if (q & 1) lb[q >> 1] |= two << 16;
                else lb[q >> 1] = two;
#pragma unroll
                for (int h = 0; h < 2; ++h) {
                    const uint32_t ce = __ldg(e + (((h ? b : a) >> 7) & 0xFF));
                    acc |= (uint64_t)(ce & 0xFFFF) << nacc;
                    nacc += (int)(ce >> 16);
                    if (nacc >= 32) {
                        atomicOr(words++, (uint32_t)acc);
                        acc >>= 32;
                        nacc -= 32;
                    }
                }
            }
            *reinterpret_cast<uint4 *>(low + (k >> 4) * 512) = make_uint4(lb[0], lb[1], lb[2], lb[3]);
        }
        if (nacc > 0) atomicOr(words, (uint32_t)acc);
    }
}

// Length-limited (<= kTB bits) Huffman code lengths of a 256-bin histogram:
// plain Huffman (ties by insertion order, deterministic), counts halved
// (kept >= 1) until the longest code fits.
inline void x3_code_lengths(const uint32_t *hist, uint8_t *len) {
    std::vector<uint64_t> cnt(hist, hist + 256);
    for (;;) {
        std::fill(len, len + 256, 0);
        std::vector<int> syms;
        for (int s = 0; s < 256; ++s)
            if (cnt[s]) syms.push_back(s);
        if (syms.empty()) return;
        if (syms.size() == 1) {
            len[syms[0]] = 1;
            return;
        }
        // nodes 0..255 leaves, 256.. internal; min-heap on (weight, id)
        std::vector<int> parent(512, -1);
        std::vector<std::pair<uint64_t, int>> heap;
        for (int s : syms) heap.push_back({cnt[s], s});
        auto cmp = [](const std::pair<uint64_t, int> &a, const std::pair<uint64_t, int> &b) { return a > b; };
        std::make_heap(heap.begin(), heap.end(), cmp);
        int next = 256;
        while (heap.size() > 1) {
            std::pop_heap(heap.begin(), heap.end(), cmp);
            const auto a = heap.back();
            heap.pop_back();
            std::pop_heap(heap.begin(), heap.end(), cmp);
            const auto b = heap.back();
            heap.pop_back();
            parent[a.second] = parent[b.second] = next;
            heap.push_back({a.first + b.first, next++});
            std::push_heap(heap.begin(), heap.end(), cmp);
        }
        int maxl = 0;
        for (int s : syms) {
            int d = 0;
            for (int x = s; parent[x] >= 0; x = parent[x]) ++d;
            len[s] = (uint8_t)d;
            maxl = std::max(maxl, d);
        }
        if (maxl <= kTB) return;
        for (int s : syms) cnt[s] = (cnt[s] + 1) / 2;
    }
}

// Canonical codes (by length, then symbol), bit-reversed for the LSB-first
// stream: enc[s] = rev_code | len << 16; table[i] = (len << 8) | s for every
// 12-bit i whose low len bits are s's reversed code.
inline void x3_tables(const uint8_t *len, uint32_t *enc, uint16_t *table) {
    std::fill(enc, enc + 256, 0u);
    std::fill(table, table + (1 << kTB), (uint16_t)0);
    std::vector<int> order;
    for (int s = 0; s < 256; ++s)
        if (len[s]) order.push_back(s);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return len[a] < len[b]; });
    uint32_t code = 0;
    int prev = order.empty() ? 0 : len[order[0]];
    for (int s : order) {
        code <<= (len[s] - prev);
        prev = len[s];
        uint32_t rev = 0;
        for (int b = 0; b < len[s]; ++b) rev |= ((code >> b) & 1u) << (len[s] - 1 - b);
        enc[s] = rev | ((uint32_t)len[s] << 16);
        for (uint32_t hi = 0; hi < (1u << (kTB - len[s])); ++hi)
            table[rev | (hi << len[s])] = (uint16_t)(((uint32_t)len[s] << 8) | (uint32_t)s);
        ++code;
    }
}

// Piece layout for n_values values (n_chunks chunks) and stream_words words.
inline void x3_layout(uint32_t n_values, uint32_t n_chunks, uint64_t stream_words, PieceV3 *h) {
    h->magic = kPieceMagic3;
    h->n_chunks = n_chunks;
    h->n_values = n_values;
    uint64_t o = align_up(sizeof(PieceV3) + (uint64_t)n_values, 16);
    h->off_table = (uint32_t)o;
    o += 2u << kTB;
    h->off_lens = (uint32_t)o;
    o = align_up(o + (uint64_t)n_chunks * 64, 16);
    h->off_cbase = (uint32_t)o;
    o = align_up(o + (uint64_t)n_chunks * 4, 16);
    h->off_streams = (uint32_t)o;
    o = align_up(o + 4 * stream_words + 32, 256);  // + slack: a lane reads up to 3 words ahead
    h->bytes = (uint32_t)o;
}
