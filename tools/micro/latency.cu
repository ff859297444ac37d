// Pointer-chase latency (cycles per dependent load) for L2-resident and HBM-resident buffers.
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <cuda_runtime.h>
__global__ void chase(const unsigned *next, int steps, unsigned start, long long *cyc, unsigned *sink) {
    unsigned p = start;
    for (int i = 0; i < 64; i++) p = next[p];   // warm TLB / first touches
    long long t0 = clock64();
    for (int i = 0; i < steps; i++) p = __ldcg(next + p);
    long long t1 = clock64();
    *cyc = t1 - t0;
    *sink = p;
}
int main() {
    for (size_t mb : {4, 32, 96, 512, 4096}) {
        size_t n = mb * 1024 * 1024 / 4;
        std::vector<unsigned> h(n);
        // random cycle with stride of at least 128 B between consecutive elements
        size_t m = n / 32;
        std::vector<unsigned> perm(m);
        for (size_t i = 0; i < m; i++) perm[i] = (unsigned)i;
        srand(1);
        for (size_t i = m - 1; i > 0; i--) { size_t j = ((size_t)rand() * RAND_MAX + rand()) % (i + 1); std::swap(perm[i], perm[j]); }
        for (size_t i = 0; i < m; i++) h[perm[i] * 32] = perm[(i + 1) % m] * 32;
        unsigned *d; long long *c; unsigned *s;
        cudaMalloc(&d, n * 4); cudaMalloc(&c, 8); cudaMalloc(&s, 4);
        cudaMemcpy(d, h.data(), n * 4, cudaMemcpyHostToDevice);
        int steps = 20000;
        chase<<<1, 1>>>(d, steps, perm[0] * 32, c, s);
        chase<<<1, 1>>>(d, steps, perm[0] * 32, c, s);
        long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
        printf("%5zu MB: %.0f cycles per dependent load\n", mb, (double)cyc / steps);
        cudaFree(d); cudaFree(c); cudaFree(s);
    }
}
