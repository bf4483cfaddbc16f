// FP64 roofline probe for B200 (sm_100a): DFMA and DMMA (mma.sync m8n8k4 f64)
// issue-bound throughput.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_peak.cu -o fp64_peak
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, int iters) {
    double a[8];
    for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
    const double b = 1.000001, c = 1e-9;
    for (int it = 0; it < iters; ++it)
#pragma unroll
        for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
    double s = 0;
    for (int i = 0; i < 8; ++i) s += a[i];
    if (s == 12345.0) out[0] = s;
}

__global__ void k_dmma(double* out, int iters) {
    double a = threadIdx.x * 1e-3, b = 1e-3;
    double c[4][2] = {};
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int t = 0; t < 4; ++t)
            asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                         : "+d"(c[t][0]), "+d"(c[t][1]) : "d"(a), "d"(b));
    }
    double s = 0;
    for (int t = 0; t < 4; ++t) s += c[t][0] + c[t][1];
    if (s == 12345.0) out[0] = s;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* d;
    cudaMalloc(&d, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 4096;
    for (int rep = 0; rep < 2; ++rep) {
        for (int bs : {256, 512, 1024}) {
            const int grid = sms * (2048 / bs);
            cudaEventRecord(e0);
            k_dfma<<<grid, bs>>>(d, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const double fl = 2.0 * 8 * iters * double(grid) * bs;
            if (rep) printf("DFMA block %4d: %.2f TFLOP/s\n", bs, fl / ms / 1e9);
            cudaEventRecord(e0);
            k_dmma<<<grid, bs>>>(d, iters);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            const double fm = 2.0 * 8 * 8 * 4 * 4 * double(iters) * (double(grid) * bs / 32);
            if (rep) printf("DMMA block %4d: %.2f TFLOP/s\n", bs, fm / ms / 1e9);
        }
    }
    printf("SMs %d\n", sms);
    return 0;
}
