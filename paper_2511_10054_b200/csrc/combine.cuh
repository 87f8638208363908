// K5 combine + layer_update for one token, shared by the standalone combine
// kernel (permute.cu) and the fused decode FFN's epilogue phase
// (ffn_decode.cu), so both compute bit-identical results. Not part of the ABI.
#pragma once

#include <stdint.h>
#include <string.h>

#include "common.cuh"

namespace bm {

constexpr int kCombineThreads = 256;

constexpr int kCombineMaxSlots = 64;
constexpr int kCombineUnroll = 2;     // vectors per thread and slot in flight together
constexpr int kCombineSlotGroup = 4;  // slots whose loads are in flight together

template <typename T, int VEC>
struct alignas(sizeof(T) * VEC) VecT {
    T v[VEC];
};

// L2 (coherent) load of a 4/8/16-byte vector
template <typename V>
__device__ __forceinline__ V ldcg_vec(const V *p) {
    V out;
    if constexpr (sizeof(V) == 16) {
        const uint4 u = __ldcg(reinterpret_cast<const uint4 *>(p));
        memcpy(&out, &u, 16);
    } else if constexpr (sizeof(V) == 8) {
        const uint2 u = __ldcg(reinterpret_cast<const uint2 *>(p));
        memcpy(&out, &u, 8);
    } else {
        const unsigned u = __ldcg(reinterpret_cast<const unsigned *>(p));
        memcpy(&out, &u, 4);
    }
    return out;
}

// read-only-path load of a 4/8/16-byte vector
template <typename V>
__device__ __forceinline__ V ldg_vec(const V *p) {
    V out;
    if constexpr (sizeof(V) == 16) {
        const uint4 u = __ldg(reinterpret_cast<const uint4 *>(p));
        memcpy(&out, &u, 16);
    } else if constexpr (sizeof(V) == 8) {
        const uint2 u = __ldg(reinterpret_cast<const uint2 *>(p));
        memcpy(&out, &u, 8);
    } else {
        const unsigned u = __ldg(reinterpret_cast<const unsigned *>(p));
        memcpy(&out, &u, 4);
    }
    return out;
}

// One CTA per token. The token's active slots (not dropped, with a row) are
// staged in shared memory first; each thread then owns VEC consecutive
// columns per vector (16-byte loads of y_perm and h: float4 / double2) and
// issues the loads of kCombineUnroll vectors of kCombineSlotGroup slots
// before their in-order fma chain: y = fma(p_s, y_s, y) over slots in slot
// order per column (model.py:334-340), then h + 0.5 y and the RMS
// normalisation of layer_update (model.py:343-347) in the same pass.
template <typename T>
struct CombineShared {
    T red[kCombineThreads / 32];
    int srow[kCombineMaxSlots];
    T sw[kCombineMaxSlots];
    int nsl;
};

// Token b by a CTA of kCombineThreads threads (hbuf: d values of shared
// memory). CG = true reads y_perm through L2 (coherent loads): the fused
// decode FFN calls this after a grid barrier, in the launch that wrote y_perm.
template <typename T, int VEC, bool CG>
__device__ __forceinline__ void combine_token(int b, const T *__restrict__ y_perm,
                                              const int32_t *__restrict__ slot_row, const T *__restrict__ probs,
                                              const uint8_t *__restrict__ kind, int k, int d, const T *h_in,
                                              T scale, T *out, T *hbuf, CombineShared<T> &sh) {
    using V = VecT<T, VEC>;
    T *red = sh.red;
    int *srow = sh.srow;
    T *sw = sh.sw;
    int &nsl = sh.nsl;
    if (threadIdx.x == 0) {
        int n = 0;
        for (int s = 0; s < k; ++s) {
            const int r = slot_row[b * k + s];
            if (r < 0 || kind[b * k + s] == BM_KIND_DROPPED) continue;
            srow[n] = r;
            sw[n] = probs[b * k + s];
            ++n;
        }
        nsl = n;
    }
    __syncthreads();
    const int ns = nsl;
    T ssq = 0;
    const int step = (int)blockDim.x * VEC;
    for (int i0 = (int)threadIdx.x * VEC; i0 < d; i0 += kCombineUnroll * step) {
        V y[kCombineUnroll], hv[kCombineUnroll];
#pragma unroll
        for (int u = 0; u < kCombineUnroll; ++u) {
            const int i = i0 + u * step;
#pragma unroll
            for (int c = 0; c < VEC; ++c) y[u].v[c] = hv[u].v[c] = 0;
            if (h_in && i < d) hv[u] = *reinterpret_cast<const V *>(h_in + (size_t)b * d + i);
        }
        for (int s0 = 0; s0 < ns; s0 += kCombineSlotGroup) {
            V a[kCombineSlotGroup][kCombineUnroll];
#pragma unroll
            for (int g = 0; g < kCombineSlotGroup; ++g) {
                if (s0 + g >= ns) break;
                const T *src = y_perm + (size_t)srow[s0 + g] * d;
#pragma unroll
                for (int u = 0; u < kCombineUnroll; ++u) {
                    const int i = i0 + u * step;
                    if (i < d) a[g][u] = CG ? ldcg_vec(reinterpret_cast<const V *>(src + i)) : ldg_vec(reinterpret_cast<const V *>(src + i));
                }
            }
#pragma unroll
            for (int g = 0; g < kCombineSlotGroup; ++g) {
                if (s0 + g >= ns) break;
                const T w = sw[s0 + g];
#pragma unroll
                for (int u = 0; u < kCombineUnroll; ++u)
#pragma unroll
                    for (int c = 0; c < VEC; ++c) y[u].v[c] = fma(w, a[g][u].v[c], y[u].v[c]);
            }
        }
#pragma unroll
        for (int u = 0; u < kCombineUnroll; ++u) {
            const int i = i0 + u * step;
            if (i >= d) continue;
            if (h_in) {
#pragma unroll
                for (int c = 0; c < VEC; ++c) {
                    const T h = fma(scale, y[u].v[c], hv[u].v[c]);
                    hbuf[i + c] = h;
                    ssq = fma(h, h, ssq);
                }
            } else {
                *reinterpret_cast<V *>(out + (size_t)b * d + i) = y[u];
            }
        }
    }
    if (!h_in) return;
    for (int o = 16; o > 0; o >>= 1) ssq += __shfl_xor_sync(0xffffffffu, ssq, o);
    if (lane_id() == 0) red[threadIdx.x >> 5] = ssq;
    __syncthreads();
    T tot = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) tot += red[w];
    const T rms = sqrt(tot / (T)d);
    const T inv = (T)1 / fmax(rms, (T)1e-12);
    for (int i = threadIdx.x; i < d; i += blockDim.x) out[(size_t)b * d + i] = hbuf[i] * inv;
}


}  // namespace bm
