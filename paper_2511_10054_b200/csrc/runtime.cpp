// Error plumbing and device queries shared by every ABI entry point.
#include <cuda_runtime.h>
#include <stdarg.h>
#include <stdio.h>

#include "../../include/bmoe.h"

namespace bm {

static thread_local char g_err[1024] = "";

void set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

int sm_count() {
    static int cached = -1;
    if (cached < 0) {
        int dev = 0;
        if (cudaGetDevice(&dev) != cudaSuccess) return 148;
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) return 148;
        cached = n;
    }
    return cached;
}

}  // namespace bm

extern "C" int bm_abi_version(void) { return BM_ABI_VERSION; }

extern "C" const char *bm_last_error(void) { return bm::g_err; }

extern "C" int bm_device_sm_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();
        return -1;
    }
    return bm::sm_count();
}
