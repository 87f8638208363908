// numpy's float64 summation order, restated for the device so the
// bit-exact paths (buddy ranking, Psi z-scores) round exactly like the
// reference's `row.sum()` / `z.mean()` / `z.std()`:
// numpy/_core/src/umath/loops_utils.h.src pairwise_sum, PW_BLOCKSIZE = 128.
// Pinned on the host by tests/test_oracle_golden.py::test_pairwise_sum_matches_numpy.
#pragma once

#include "common.cuh"

namespace bm {

// Sum of f(i) for i in [lo, lo+n) in numpy's pairwise order. Single thread.
// Iterative post-order walk of numpy's recursion (depth <= 8 for n <= 2^15).
template <typename F>
__device__ double pairwise_sum_fn(F f, int lo, int n) {
    struct Frame {
        int lo, n, n2;
        double left;
        int state;
    };
    Frame st[12];
    int sp = 0;
    st[0] = {lo, n, 0, 0.0, 0};
    double ret = 0.0;
    while (true) {
        Frame &fr = st[sp];
        if (fr.state == 0 && fr.n <= 128) {
            double res;
            if (fr.n < 8) {
                res = 0.0;
                for (int i = 0; i < fr.n; ++i) res = dadd(res, f(fr.lo + i));
            } else {
                double r[8];
#pragma unroll
                for (int j = 0; j < 8; ++j) r[j] = f(fr.lo + j);
                int i = 8;
                for (; i < fr.n - (fr.n % 8); i += 8) {
#pragma unroll
                    for (int j = 0; j < 8; ++j) r[j] = dadd(r[j], f(fr.lo + i + j));
                }
                res = dadd(dadd(dadd(r[0], r[1]), dadd(r[2], r[3])), dadd(dadd(r[4], r[5]), dadd(r[6], r[7])));
                for (; i < fr.n; ++i) res = dadd(res, f(fr.lo + i));
            }
            ret = res;
            if (sp == 0) return ret;
            --sp;
            continue;  // parent consumes `ret`
        }
        if (fr.state == 0) {
            int n2 = fr.n / 2;
            n2 -= n2 % 8;
            fr.n2 = n2;
            fr.state = 1;
            st[++sp] = {fr.lo, n2, 0, 0.0, 0};
            continue;
        }
        if (fr.state == 1) {
            fr.left = ret;
            fr.state = 2;
            st[sp + 1] = {fr.lo + fr.n2, fr.n - fr.n2, 0, 0.0, 0};
            ++sp;
            continue;
        }
        // state 2: right child done
        ret = dadd(fr.left, ret);
        if (sp == 0) return ret;
        --sp;
    }
}

struct ArrayTerm {
    const double *a;
    __device__ double operator()(int i) const { return a[i]; }
};

struct SqDevTerm {
    const double *a;
    double mean;
    __device__ double operator()(int i) const {
        double x = dsub(a[i], mean);
        return dmul(x, x);
    }
};

__device__ inline double pairwise_sum(const double *a, int n) { return pairwise_sum_fn(ArrayTerm{a}, 0, n); }
__device__ inline double pairwise_sum_sq_dev(const double *a, int n, double mean) {
    return pairwise_sum_fn(SqDevTerm{a, mean}, 0, n);
}

}  // namespace bm
