// Library comparator for BASELINE config 5: the same batches of
// i.i.d. N(0,1) fronts as tools/microbench.py, factored by cuBLAS / cuSOLVER
// called directly (no torch in between).
//
//   geqrf_batched : cublasDgeqrfBatched on the m x n panels (QR only, no Q^T apply)
//   geqrf_ormqr   : per front, cusolverDnDgeqrf on the panel + cusolverDnDormqr(Q^T)
//                   on the m x 256 neighbour block, all on one stream
//
// Device time from CUDA events, best of 3 after one warm-up; one JSON line per shape.
// Build: make -C tools cusolver_c5   (links -lcublas -lcusolver)
#include <cublas_v2.h>
#include <cuda_runtime.h>
#include <cusolverDn.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#define CK(x)                                                                              \
    do {                                                                                   \
        auto e_ = (x);                                                                     \
        if (static_cast<int>(e_) != 0) {                                                   \
            std::fprintf(stderr, "%s:%d %s -> %d\n", __FILE__, __LINE__, #x, (int)e_);     \
            std::exit(1);                                                                  \
        }                                                                                  \
    } while (0)

static double qr_flops(double m, double n, double k) {
    return 2 * m * n * n - 2.0 / 3.0 * n * n * n + 4 * m * n * k - 2 * n * n * k;
}

int main(int argc, char** argv) {
    const double peak = argc > 1 ? std::atof(argv[1]) : 37.1;  // TF/s, measured DMMA peak
    struct Shape { int m, n, nb; };
    const Shape shapes[] = {{128, 32, 4096}, {512, 128, 1024}, {4096, 1024, 64}};
    const int k = 256;
    cublasHandle_t cb;
    cusolverDnHandle_t cs;
    CK(cublasCreate(&cb));
    CK(cusolverDnCreate(&cs));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    CK(cublasSetStream(cb, st));
    CK(cusolverDnSetStream(cs, st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    for (const Shape& s : shapes) {
        const int m = s.m, n = s.n, nb = s.nb;
        const size_t pa = static_cast<size_t>(m) * n, px = static_cast<size_t>(m) * k;
        std::vector<double> h(pa * nb + px * nb);
        std::mt19937_64 rng(0);
        std::normal_distribution<double> nd;
        for (auto& v : h) v = nd(rng);
        double *dA0, *dA, *dX0, *dX, *dTau;
        CK(cudaMalloc(&dA0, pa * nb * 8));
        CK(cudaMalloc(&dA, pa * nb * 8));
        CK(cudaMalloc(&dX0, px * nb * 8));
        CK(cudaMalloc(&dX, px * nb * 8));
        CK(cudaMalloc(&dTau, static_cast<size_t>(n) * nb * 8));
        CK(cudaMemcpy(dA0, h.data(), pa * nb * 8, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dX0, h.data() + pa * nb, px * nb * 8, cudaMemcpyHostToDevice));
        std::vector<double*> hAp(nb), hTp(nb);
        for (int b = 0; b < nb; ++b) {
            hAp[b] = dA + pa * b;
            hTp[b] = dTau + static_cast<size_t>(n) * b;
        }
        double **dAp, **dTp;
        CK(cudaMalloc(&dAp, nb * sizeof(double*)));
        CK(cudaMalloc(&dTp, nb * sizeof(double*)));
        CK(cudaMemcpy(dAp, hAp.data(), nb * sizeof(double*), cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dTp, hTp.data(), nb * sizeof(double*), cudaMemcpyHostToDevice));

        // 1) cublasDgeqrfBatched (panel QR only)
        float best_b = 1e30f;
        for (int r = 0; r < 4; ++r) {
            CK(cudaMemcpyAsync(dA, dA0, pa * nb * 8, cudaMemcpyDeviceToDevice, st));
            int info = 0;
            CK(cudaEventRecord(e0, st));
            CK(cublasDgeqrfBatched(cb, m, n, dAp, m, dTp, &info, nb));
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (r > 0) best_b = std::min(best_b, ms);
        }

        // 2) cusolverDn geqrf + ormqr(Q^T) per front
        int lw1 = 0, lw2 = 0;
        CK(cusolverDnDgeqrf_bufferSize(cs, m, n, dA, m, &lw1));
        CK(cusolverDnDormqr_bufferSize(cs, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, m, k, n, dA, m, dTau, dX, m, &lw2));
        const int lw = std::max(lw1, lw2);
        double* dWork;
        int* dInfo;
        CK(cudaMalloc(&dWork, static_cast<size_t>(lw) * 8));
        CK(cudaMalloc(&dInfo, sizeof(int)));
        float best_s = 1e30f;
        for (int r = 0; r < 4; ++r) {
            CK(cudaMemcpyAsync(dA, dA0, pa * nb * 8, cudaMemcpyDeviceToDevice, st));
            CK(cudaMemcpyAsync(dX, dX0, px * nb * 8, cudaMemcpyDeviceToDevice, st));
            CK(cudaEventRecord(e0, st));
            for (int b = 0; b < nb; ++b) {
                double* A = dA + pa * b;
                double* X = dX + px * b;
                double* t = dTau + static_cast<size_t>(n) * b;
                CK(cusolverDnDgeqrf(cs, m, n, A, m, t, dWork, lw, dInfo));
                CK(cusolverDnDormqr(cs, CUBLAS_SIDE_LEFT, CUBLAS_OP_T, m, k, n, A, m, t, X, m, dWork, lw, dInfo));
            }
            CK(cudaEventRecord(e1, st));
            CK(cudaEventSynchronize(e1));
            float ms;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            if (r > 0) best_s = std::min(best_s, ms);
        }
        const double fl_qr = qr_flops(m, n, 0) * nb, fl = qr_flops(m, n, k) * nb;
        std::printf("{\"shape\": \"%dx%d+%d\", \"batch\": %d, \"cublasDgeqrfBatched_ms\": %.3f, "
                    "\"cublasDgeqrfBatched_TFLOPs_qr_only\": %.3f, \"cusolverDn_geqrf_ormqr_ms\": %.3f, "
                    "\"cusolverDn_TFLOPs\": %.3f, \"cusolverDn_frac_fp64\": %.4f}\n",
                    m, n, k, nb, best_b, fl_qr / best_b / 1e9, best_s, fl / best_s / 1e9, fl / best_s / 1e9 / peak);
        std::fflush(stdout);
        CK(cudaFree(dA0));
        CK(cudaFree(dA));
        CK(cudaFree(dX0));
        CK(cudaFree(dX));
        CK(cudaFree(dTau));
        CK(cudaFree(dAp));
        CK(cudaFree(dTp));
        CK(cudaFree(dWork));
        CK(cudaFree(dInfo));
    }
    return 0;
}
