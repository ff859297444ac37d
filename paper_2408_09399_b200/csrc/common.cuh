// common.cuh -- shared helpers for the sm_100a TMFG-DBHT kernels.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>
#include <limits.h>

#include "../../include/tmfg_b200.h"

#define TG_API extern "C" __attribute__((visibility("default")))

#define TG_CUDA_CHECK(expr)                                   \
    do {                                                      \
        cudaError_t _e = (expr);                              \
        if (_e != cudaSuccess) {                              \
            tg_set_last_error(_e, __FILE__, __LINE__);        \
            return TG_ERR_CUDA;                               \
        }                                                     \
    } while (0)

#define TG_LAUNCH_CHECK() TG_CUDA_CHECK(cudaGetLastError())

void tg_set_last_error(cudaError_t e, const char *file, int line);
void tg_count_launch(int k);

static inline cudaStream_t tg_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

static inline int tg_num_sms() {
    static int sms = 0;
    if (!sms) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        if (sms <= 0) sms = 148;
    }
    return sms;
}

static inline size_t tg_align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// Simple bump allocator over a caller-provided workspace.
struct TgArena {
    char *base;
    size_t cap;
    size_t used;
    __host__ TgArena(void *b, size_t c) : base((char *)b), cap(c), used(0) {}
    template <class T>
    __host__ T *take(size_t count) {
        size_t off = tg_align_up(used, 256);
        size_t bytes = count * sizeof(T);
        if (off + bytes > cap) return nullptr;
        used = off + bytes;
        return reinterpret_cast<T *>(base + off);
    }
};

// ---------------------------------------------------------------- device helpers
__device__ __forceinline__ unsigned long long tg_dbits(double x) {
    return (unsigned long long)__double_as_longlong(x);
}

// Order-preserving map for NON-NEGATIVE doubles (distances, heights): the raw bits.
__device__ __forceinline__ double tg_atomic_min_nonneg(double *addr, double v) {
    unsigned long long old = atomicMin((unsigned long long *)addr, tg_dbits(v));
    return __longlong_as_double((long long)old);
}
__device__ __forceinline__ double tg_atomic_max_nonneg(double *addr, double v) {
    unsigned long long old = atomicMax((unsigned long long *)addr, tg_dbits(v));
    return __longlong_as_double((long long)old);
}

// Total-order key for any double (for descending/ascending selections):
// larger double -> larger key; -0.0 and +0.0 map to the same key.
__device__ __forceinline__ unsigned long long tg_order_key(double x) {
    if (x == 0.0) x = 0.0;
    unsigned long long b = tg_dbits(x);
    return (b >> 63) ? ~b : (b | 0x8000000000000000ull);
}

__device__ __forceinline__ int tg_lane() { return threadIdx.x & 31; }
__device__ __forceinline__ int tg_warp() { return threadIdx.x >> 5; }
