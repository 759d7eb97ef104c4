// TMEM probe: allocate tensor memory, store per-lane FP64 data with
// tcgen05.st, read it back with tcgen05.ld, check, and time the read path.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tmem_probe tools/tmem_probe.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void __launch_bounds__(256, 1) tmem_probe(double* out, int iters, unsigned long long* cycles) {
    __shared__ uint32_t tbase;
    const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t base = tbase;
    const uint32_t lane_base = (uint32_t)(32 * (warp % 4)) << 16;
    // warps 0..3 write: column c holds (lane, c) pattern as doubles in pairs of columns
    if (warp < 4) {
        for (int c = 0; c < 512; c += 4) {
            double a = 1000.0 * (32 * warp + lane) + c, b = a + 1.0;
            uint32_t r0 = __double2loint(a), r1 = __double2hiint(a), r2 = __double2loint(b), r3 = __double2hiint(b);
            asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(base + lane_base + c),
                         "r"(r0), "r"(r1), "r"(r2), "r"(r3));
        }
        asm volatile("tcgen05.wait::st.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    // every warp reads its lane quarter back
    double acc = 0.0;
    int bad = 0;
    for (int c = 0; c < 512; c += 4) {
        uint32_t r0, r1, r2, r3;
        asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                     : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
                     : "r"(base + lane_base + c));
        asm volatile("tcgen05.wait::ld.sync.aligned;");
        double a = __hiloint2double(r1, r0), b = __hiloint2double(r3, r2);
        double ea = 1000.0 * (32 * (warp % 4) + lane) + c;
        if (a != ea || b != ea + 1.0) bad++;
        acc += a;
    }
    // timed read loop: x16 loads (8 doubles per lane) with one wait per batch
    unsigned long long t0 = clock64();
    double s = 0.0;
    for (int it = 0; it < iters; ++it) {
        for (int c = 0; c < 512; c += 16) {
            uint32_t r[16];
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
                : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
                  "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
                : "r"(base + lane_base + c));
            asm volatile("tcgen05.wait::ld.sync.aligned;");
#pragma unroll
            for (int q = 0; q < 16; q += 2) s += __hiloint2double(r[q + 1], r[q]);
        }
    }
    unsigned long long t1 = clock64();
    if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc + s * 1e-30 + bad * 1e9;
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(base));
}

int main() {
    double* out;
    unsigned long long* cyc;
    int blocks = 148, threads = 256, iters = 200;
    cudaMalloc(&out, sizeof(double) * blocks * threads);
    cudaMalloc(&cyc, sizeof(unsigned long long) * blocks);
    tmem_probe<<<blocks, threads>>>(out, iters, cyc);
    cudaError_t e = cudaDeviceSynchronize();
    printf("status: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 1;
    double* h = new double[blocks * threads];
    unsigned long long hc[148];
    cudaMemcpy(h, out, sizeof(double) * blocks * threads, cudaMemcpyDeviceToHost);
    cudaMemcpy(hc, cyc, sizeof(hc), cudaMemcpyDeviceToHost);
    int nbad = 0;
    for (int i = 0; i < blocks * threads; ++i)
        if (h[i] >= 1e9) nbad++;
    double bytes = (double)iters * 512 * 4 * threads;  // per CTA
    printf("threads with mismatches: %d\n", nbad);
    printf("tcgen05.ld x16 read: %.1f bytes/clk/SM (cycles %llu)\n", bytes / hc[0], hc[0]);
    return nbad ? 2 : 0;
}
