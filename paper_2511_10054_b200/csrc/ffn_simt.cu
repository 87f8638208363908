// fp32 parity mode of the grouped expert FFN: SIMT FFMA tiles (tcgen05 has
// no true fp32 MMA, and kind::tf32 would miss the rel 1e-5 contract), and the
// same tiles in f64 for the reference-precision Python API (model.forward_batch).
// out[r, j] = act( sum_i in[r,i] * A[j,i] ) per expert segment of rows;
// for SwiGLU the gate and up accumulators are computed together.
// Reference: Expert.__call__ / forward_batch (model.py:85-99, 318-340).
#include <math.h>

#include "common.cuh"

namespace bm {
namespace {

constexpr int TM = 16;   // rows per tile (== permute row alignment)
constexpr int TN = 64;   // outputs per tile
constexpr int TK = 32;   // K chunk
constexpr int kThreads = 256;  // each thread: 1 row-quad x 1 output... (16*64)/256 = 4 outputs

enum { ACT_NONE = -1 };

template <typename T, int ACT, bool TWO>
__global__ void __launch_bounds__(kThreads) simt_gemm_kernel(const T *__restrict__ in, int K,
                                                             const int32_t *__restrict__ expert_offset, int E,
                                                             const T *__restrict__ arena, long long buf_elems,
                                                             const int32_t *__restrict__ buf_of_expert,
                                                             long long a_off, long long a2_off, int Nout,
                                                             T *__restrict__ out) {
    __shared__ T xs[TM][TK + 1];
    __shared__ T ws[TWO ? 2 : 1][TN][TK + 1];
    __shared__ int s_e;
    const int r0 = blockIdx.y * TM;
    const int j0 = blockIdx.x * TN;
    if (threadIdx.x == 0) {
        int e = -1;
        if (r0 < expert_offset[E]) {
            // segment containing r0 (segments are TM-aligned): the largest e
            // with offset[e] <= r0 is non-empty because offset[E] > r0.
            int lo = 0, hi = E - 1;
            while (lo < hi) {
                int mid = (lo + hi + 1) >> 1;
                if (expert_offset[mid] <= r0) lo = mid; else hi = mid - 1;
            }
            e = lo;
        }
        s_e = e;
    }
    __syncthreads();
    const int e = s_e;
    if (e < 0 || e >= E) return;
    const T *A = arena + (long long)buf_of_expert[e] * buf_elems + a_off;
    const T *A2 = arena + (long long)buf_of_expert[e] * buf_elems + a2_off;
    const int tr = threadIdx.x / TN;  // 0..3 -> rows tr*4 .. tr*4+3
    const int tj = threadIdx.x % TN;
    T acc[4] = {0, 0, 0, 0}, acc2[4] = {0, 0, 0, 0};
    for (int k0 = 0; k0 < K; k0 += TK) {
        for (int i = threadIdx.x; i < TM * TK; i += kThreads) {
            int rr = i / TK, kk = i % TK;
            xs[rr][kk] = (k0 + kk < K) ? in[(size_t)(r0 + rr) * K + k0 + kk] : T(0);
        }
        for (int i = threadIdx.x; i < TN * TK; i += kThreads) {
            int jj = i / TK, kk = i % TK;
            bool ok = (j0 + jj < Nout) && (k0 + kk < K);
            ws[0][jj][kk] = ok ? A[(size_t)(j0 + jj) * K + k0 + kk] : T(0);
            if (TWO) ws[TWO ? 1 : 0][jj][kk] = ok ? A2[(size_t)(j0 + jj) * K + k0 + kk] : T(0);
        }
        __syncthreads();
#pragma unroll 8
        for (int kk = 0; kk < TK; ++kk) {
            T w = ws[0][tj][kk];
            T w2 = TWO ? ws[TWO ? 1 : 0][tj][kk] : T(0);
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                T xv = xs[tr * 4 + q][kk];
                acc[q] = fma(xv, w, acc[q]);
                if (TWO) acc2[q] = fma(xv, w2, acc2[q]);
            }
        }
        __syncthreads();
    }
    if (j0 + tj >= Nout) return;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        T v = acc[q];
        if (ACT == BM_ACT_TANH) v = tanh(v);
        if (ACT == BM_ACT_SWIGLU) v = (v / (T(1) + exp(-v))) * acc2[q];
        out[(size_t)(r0 + tr * 4 + q) * Nout + j0 + tj] = v;
    }
}

}  // namespace
}  // namespace bm

using namespace bm;

template <typename T>
static int expert_ffn_simt(const T *x_perm, const int32_t *expert_offset, int64_t E, int64_t d, int64_t f,
                           int32_t act, const T *w_arena, int64_t buf_elems, const int32_t *buf_of_expert,
                           int64_t r_max, T *h_ws, T *y_perm, bm_stream_t stream) {
    BM_REQUIRE(x_perm && expert_offset && w_arena && buf_of_expert && h_ws && y_perm, BM_EINVAL,
               "bm_expert_ffn (SIMT): null pointer");
    BM_REQUIRE(E >= 1 && d >= 1 && f >= 1 && r_max >= 0 && r_max % TM == 0, BM_EINVAL,
               "bm_expert_ffn (SIMT): bad shape (r_max must be a multiple of %d)", TM);
    BM_REQUIRE(act == BM_ACT_TANH || act == BM_ACT_SWIGLU, BM_EINVAL, "bad activation %d", act);
    if (r_max == 0) return BM_OK;
    const long long need = act == BM_ACT_SWIGLU ? 3 * d * f : 2 * d * f;
    BM_REQUIRE(buf_elems >= need, BM_EINVAL, "buffer too small for the expert layout");
    cudaStream_t s = as_stream(stream);
    dim3 g1((unsigned)((f + TN - 1) / TN), (unsigned)(r_max / TM));
    dim3 g2((unsigned)((d + TN - 1) / TN), (unsigned)(r_max / TM));
    if (act == BM_ACT_SWIGLU) {
        simt_gemm_kernel<T, BM_ACT_SWIGLU, true><<<g1, kThreads, 0, s>>>(x_perm, (int)d, expert_offset, (int)E,
                                                                        w_arena, buf_elems, buf_of_expert, 0, f * d,
                                                                        (int)f, h_ws);
        BM_LAUNCH_CHECK();
        simt_gemm_kernel<T, ACT_NONE, false><<<g2, kThreads, 0, s>>>(h_ws, (int)f, expert_offset, (int)E, w_arena,
                                                                    buf_elems, buf_of_expert, 2 * f * d, 0, (int)d,
                                                                    y_perm);
    } else {
        simt_gemm_kernel<T, BM_ACT_TANH, false><<<g1, kThreads, 0, s>>>(x_perm, (int)d, expert_offset, (int)E,
                                                                       w_arena, buf_elems, buf_of_expert, 0, 0,
                                                                       (int)f, h_ws);
        BM_LAUNCH_CHECK();
        simt_gemm_kernel<T, ACT_NONE, false><<<g2, kThreads, 0, s>>>(h_ws, (int)f, expert_offset, (int)E, w_arena,
                                                                    buf_elems, buf_of_expert, f * d, 0, (int)d,
                                                                    y_perm);
    }
    BM_LAUNCH_CHECK();
    return BM_OK;
}

extern "C" int bm_expert_ffn_f32(const float *x_perm, const int32_t *expert_count, const int32_t *expert_offset,
                                 int64_t E, int64_t d, int64_t f, int32_t act, const float *w_arena,
                                 int64_t buf_elems, const int32_t *buf_of_expert, int64_t r_max, float *h_ws,
                                 float *y_perm, bm_stream_t stream) {
    (void)expert_count;
    return expert_ffn_simt<float>(x_perm, expert_offset, E, d, f, act, w_arena, buf_elems, buf_of_expert, r_max, h_ws,
                                  y_perm, stream);
}

extern "C" int bm_expert_ffn_f64(const double *x_perm, const int32_t *expert_count, const int32_t *expert_offset,
                                 int64_t E, int64_t d, int64_t f, int32_t act, const double *w_arena,
                                 int64_t buf_elems, const int32_t *buf_of_expert, int64_t r_max, double *h_ws,
                                 double *y_perm, bm_stream_t stream) {
    (void)expert_count;
    return expert_ffn_simt<double>(x_perm, expert_offset, E, d, f, act, w_arena, buf_elems, buf_of_expert, r_max,
                                   h_ws, y_perm, stream);
}
