// fp64 tensor-pipe peak on this B200: DMMA (mma.sync m8n8k4 f64) from registers, no memory traffic.
// Every warp keeps 8 independent accumulator chains in flight; grid = SMs x blocks-per-SM.
// Prints TF/s (2*8*8*4 flops per warp-level mma) for a sweep of warps per SM.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_peak dmma_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(int iters, double *sink) {
    double a = 1.0 + threadIdx.x * 1e-9, b = 0.5 - threadIdx.x * 1e-9;
    double c[CHAINS][2];
#pragma unroll
    for (int k = 0; k < CHAINS; k++) c[k][0] = c[k][1] = 0.0;
    for (int i = 0; i < iters; i++) {
#pragma unroll
        for (int k = 0; k < CHAINS; k++)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[k][0]), "+d"(c[k][1]) : "d"(a), "d"(b));
    }
    double s = 0.0;
#pragma unroll
    for (int k = 0; k < CHAINS; k++) s += c[k][0] + c[k][1];
    if (s == 12345.678) *sink = s;
}

int main() {
    int dev = 0, sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    double *sink;
    cudaMalloc(&sink, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 20000;
    double best = 0.0;
    for (int warps : {4, 8, 16, 32}) {
        dim3 grid(sms * (warps / 4)), block(128);
        dmma_loop<8><<<grid, block>>>(100, sink);   // warm-up
        cudaEventRecord(e0);
        dmma_loop<8><<<grid, block>>>(iters, sink);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, e0, e1);
        double flops = 2.0 * 8 * 8 * 4 * 8.0 * iters * (double)grid.x * 4;   // per warp-mma 512 flops
        double tf = flops / (ms * 1e-3) / 1e12;
        if (tf > best) best = tf;
        printf("{\"warps_per_sm\": %d, \"ms\": %.3f, \"dmma_tflops\": %.2f}\n", warps, ms, tf);
    }
    printf("{\"dmma_peak_tflops\": %.2f, \"sms\": %d}\n", best, sms);
    cudaError_t err = cudaGetLastError();
    if (err != cudaSuccess) { printf("error %s\n", cudaGetErrorString(err)); return 1; }
    return 0;
}
