// Shared helpers for libbmoe.so (sm_100a). Not part of the ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <string>

#include "../../include/bmoe.h"

namespace bm {

void set_error(const char *fmt, ...);

// Status helpers: every ABI function returns through these so the message
// lands in bm_last_error().
#define BM_REQUIRE(cond, code, ...)            \
    do {                                       \
        if (!(cond)) {                         \
            ::bm::set_error(__VA_ARGS__);      \
            return (code);                     \
        }                                      \
    } while (0)

#define BM_CUDA_TRY(expr)                                                                       \
    do {                                                                                        \
        cudaError_t _e = (expr);                                                                \
        if (_e != cudaSuccess) {                                                                \
            ::bm::set_error("%s:%d %s: %s", __FILE__, __LINE__, #expr, cudaGetErrorString(_e)); \
            return BM_ECUDA;                                                                    \
        }                                                                                       \
    } while (0)

#define BM_LAUNCH_CHECK() BM_CUDA_TRY(cudaGetLastError())

inline cudaStream_t as_stream(bm_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// IEEE f64 ops without FMA contraction: the bit-exact paths (ranking,
// Psi scores, z-scores) must round each operation like numpy does.
__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double ddiv(double a, double b) { return __ddiv_rn(a, b); }

}  // namespace bm
