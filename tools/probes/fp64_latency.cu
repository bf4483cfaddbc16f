// Dependent-issue latencies of FP64 instructions on B200 (one warp per SM, clock64 around
// an unrolled dependent chain).  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_latency.cu
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};" : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
template <int OP>
__global__ void k(double* out, long long* cyc, double seed, int nwarps_active) {
    __shared__ double sh[64];
    sh[threadIdx.x & 63] = seed;
    __syncthreads();
    if ((threadIdx.x >> 5) >= nwarps_active) return;
    double a = seed + threadIdx.x * 1e-9, b = 1.0000001, c = 1e-9, c1 = 0;
    int idx = threadIdx.x & 31;
    double v8[8];
    for (int q = 0; q < 8; ++q) v8[q] = a + q;
    long long t0 = clock64();
#pragma unroll 1
    for (int it = 0; it < 64; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
            if (OP == 0) a = fma(a, b, c);
            if (OP == 1) a = a + b;
            if (OP == 2) a += __shfl_xor_sync(0xffffffffu, a, 1);
            if (OP == 3) dmma(a, c1, b, c);
            if (OP == 4) a = sqrt(a + 2.0);
            if (OP == 5) a = 1.0 / (a + 2.0);
            if (OP == 6) { idx = (int)sh[idx & 63] ; a += idx; }
            if (OP == 7) a = __shfl_xor_sync(0xffffffffu, a, 1);
            if (OP == 8) a = a * b;
        }
        if (OP == 9) {  // 16 x 8 independent DFMA chains
#pragma unroll
            for (int u = 0; u < 16; ++u)
#pragma unroll
                for (int q = 0; q < 8; ++q) v8[q] = fma(v8[q], b, c);
        }
        if (OP == 10) {  // 16 x (8 independent shfl.f64 + DADD)
#pragma unroll
            for (int u = 0; u < 16; ++u)
#pragma unroll
                for (int q = 0; q < 8; ++q) v8[q] += __shfl_xor_sync(0xffffffffu, v8[q], 1 << (u % 5));
        }
        if (OP == 11) {  // 16 x 8 independent DMMA pairs (4 accumulators)
#pragma unroll
            for (int u = 0; u < 16; ++u)
#pragma unroll
                for (int q = 0; q < 4; ++q) dmma(v8[2 * q], v8[2 * q + 1], b, c);
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    for (int q = 0; q < 8; ++q) a += v8[q];
    if (a == 12345.678) out[0] = a + c1;
}
template <int OP>
void run(const char* name, double* d, long long* dc, int nw) {
    k<OP><<<1, 32 * 8>>>(d, dc, 1.0, nw);
    k<OP><<<1, 32 * 8>>>(d, dc, 1.0, nw);
    cudaDeviceSynchronize();
    long long h;
    cudaMemcpy(&h, dc, 8, cudaMemcpyDeviceToHost);
    printf("%-28s warps %d: %.1f cycles per op\n", name, nw, h / 1024.0);
}
int main() {
    double* d; long long* dc;
    cudaMalloc(&d, 8); cudaMalloc(&dc, 8);
    for (int nw : {1, 4, 8}) {
        run<0>("DFMA dependent", d, dc, nw);
        run<1>("DADD dependent", d, dc, nw);
        run<8>("DMUL dependent", d, dc, nw);
        run<2>("shfl.f64 + DADD", d, dc, nw);
        run<7>("shfl.f64 only", d, dc, nw);
        run<3>("DMMA dependent", d, dc, nw);
        run<4>("sqrt(a+2)", d, dc, nw);
        run<5>("1/(a+2)", d, dc, nw);
        run<6>("LDS->cvt->add chain", d, dc, nw);
        run<9>("8 indep DFMA (per 8)", d, dc, nw);
        run<10>("8 indep shfl.f64+DADD (per 8)", d, dc, nw);
        run<11>("4 indep DMMA (per 4)", d, dc, nw);
    }
    return 0;
}
