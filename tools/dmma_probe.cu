// Does FP64 mma.sync (DMMA, m8n8k4) run on a pipe separate from the FP64 DFMA units on
// B200?  Times (a) DFMA-only warps, (b) DMMA-only warps, (c) both roles in one launch.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe tools/dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

__global__ void probe(int mode, int iters, double* out) {
    const int warp = threadIdx.x >> 5;
    const bool fma_role = mode == 0 || (mode == 2 && (warp & 1) == 0);
    double x[8], acc = 0.0;
    for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
    if (fma_role) {
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 8; ++i) x[i] = fma(x[i], 0.999999, 1e-7);
        for (int i = 0; i < 8; ++i) acc += x[i];
    } else {
        double d[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        const double a = threadIdx.x * 1e-3, b = 0.5;
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int i = 0; i < 4; ++i) dmma(d[2 * i], d[2 * i + 1], a, b);
        for (int i = 0; i < 8; ++i) acc += d[i];
    }
    if (acc == 12345.678) out[0] = acc;
}

int main() {
    double* out;
    cudaMalloc(&out, 8);
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    const int iters = 20000, threads = 512, blocks = nsm * 2;
    for (int mode = 0; mode < 3; ++mode) {
        probe<<<blocks, threads>>>(mode, 100, out);
        cudaEventRecord(a);
        probe<<<blocks, threads>>>(mode, iters, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0;
        cudaEventElapsedTime(&ms, a, b);
        const double warps = (double)blocks * threads / 32;
        // DFMA role: 8 FMA x 32 lanes per iteration; DMMA role: 4 x 256 FMA per iteration
        double fma_w = mode == 0 ? warps : (mode == 2 ? warps / 2 : 0);
        double mma_w = mode == 1 ? warps : (mode == 2 ? warps / 2 : 0);
        double flops = 2.0 * iters * (fma_w * 8 * 32 + mma_w * 4 * 256);
        printf("mode %d (%s): %.3f ms, %.2f TFLOP/s\n", mode, mode == 0 ? "DFMA" : mode == 1 ? "DMMA" : "both",
               ms, flops / (ms * 1e-3) / 1e12);
    }
    return 0;
}
