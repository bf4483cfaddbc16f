// Which warps of a CTA share a warp scheduler (and FP64 pipe)?  Warp 0 runs a dependent DFMA
// chain; one other warp w runs back-to-back DMMAs; the chain's time rises when w sits on
// warp 0's scheduler.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 sched_map.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
__global__ void k(double* out, long long* cyc, unsigned busy_mask, volatile int* stop) {
    const int wid = threadIdx.x >> 5;
    __shared__ volatile int done;
    if (threadIdx.x == 0) done = 0;
    __syncthreads();
    if (wid == 0) {
        double a = 1.0 + threadIdx.x * 1e-9;
        long long t0 = clock64();
#pragma unroll 1
        for (int it = 0; it < 256; ++it) {
#pragma unroll
            for (int u = 0; u < 16; ++u) a = fma(a, 1.0000001, 1e-9);
        }
        long long t1 = clock64();
        if (threadIdx.x == 0) { cyc[0] = t1 - t0; done = 1; }
        if (a == 123.456) out[0] = a;
    } else if ((busy_mask >> wid) & 1) {
        double c[4][2] = {};
        double a = threadIdx.x * 1e-3, b = 1e-3;
        while (!done) {
#pragma unroll
            for (int u = 0; u < 8; ++u)
#pragma unroll
                for (int q = 0; q < 4; ++q) dmma(c[q][0], c[q][1], a, b);
        }
        double s = 0;
        for (int q = 0; q < 4; ++q) s += c[q][0] + c[q][1];
        if (s == 123.456) out[1] = s;
    }
}
int main() {
    double* d; long long* dc; int* st;
    cudaMalloc(&d, 16); cudaMalloc(&dc, 8); cudaMalloc(&st, 4);
    auto run = [&](unsigned mask) {
        k<<<1, 512>>>(d, dc, mask, st);
        cudaDeviceSynchronize();
        long long h; cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost);
        return h / 4096.0;
    };
    run(0);
    printf("alone: %.1f cycles per DFMA\n", run(0));
    for (int w = 1; w < 16; ++w) printf("DMMA warp %2d: %.1f\n", w, run(1u << w));
    printf("DMMA warps 1,2,3: %.1f\n", run(0xEu));
    printf("DMMA warps 4,8,12: %.1f\n", run((1u << 4) | (1u << 8) | (1u << 12)));
    printf("DMMA warps all but 0,4,8,12: %.1f\n", run(0xEEEEu));
    printf("DMMA warps all but 0: %.1f\n", run(0xFFFEu));
    return 0;
}
