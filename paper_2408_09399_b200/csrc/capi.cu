// capi.cu -- ABI version and error reporting for libtmfg_b200.so.
#include <stdio.h>
#include <atomic>
#include "common.cuh"

static thread_local char g_last_error[512] = "";

void tg_set_last_error(cudaError_t e, const char *file, int line) {
    snprintf(g_last_error, sizeof(g_last_error), "%s (%s) at %s:%d", cudaGetErrorName(e), cudaGetErrorString(e),
             file, line);
}

TG_API int tg_abi_version(void) { return TG_ABI_VERSION; }
TG_API const char *tg_last_error(void) { return g_last_error; }

static std::atomic<long long> g_launches{0};
void tg_count_launch(int k) { g_launches.fetch_add(k, std::memory_order_relaxed); }

/* number of kernels this library has launched (evidence for bench.py's gpu_launches) */
TG_API long long tg_launch_count(void) { return g_launches.load(std::memory_order_relaxed); }
