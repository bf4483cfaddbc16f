// W sweeps and preconditioned CGLS on the device (proj/src/transforms.cpp:40-111,
// proj/src/solve.cpp:24-108).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "dev.h"
#include "devmem.h"
#include "engine.h"

namespace spqr {

// Level schedule of W: one batch per engine phase, chronological.
struct SolvePlan {
    struct Batch {
        const WFac* fac = nullptr;  // warp per factor
        int nf = 0, maxc = 0;
        const WFac* bfac = nullptr;  // CTA per factor (c >= kBigFactorCols)
        int nbf = 0, bmaxc = 0;
        const int *rptr = nullptr, *ridx = nullptr, *rcol = nullptr;  // wt reduce lists
        int ncol = 0;
    };
    std::vector<Batch> batches;
    double* contrib = nullptr;
    std::unique_ptr<DeviceArena> mem;
    long long launches_per_sweep_t = 0, launches_per_sweep = 0;
};
SolvePlan build_solve_plan(const DeviceFactorization& F, cudaStream_t st);

enum SweepMode { kWSolve = 0, kWtSolve = 1, kWApply = 2, kWtApply = 3 };
long long sweep(const SolvePlan& P, SweepMode mode, double* d_z, cudaStream_t st);  // returns launches

// A on the device in both orientations (row dots for A x and A^T y).
struct DevMatrix {
    int m = 0, n = 0;
    int *rp = nullptr, *ri = nullptr;  // CSR of A
    double* rv = nullptr;
    int *cp = nullptr, *ci = nullptr;  // CSC of A (= CSR of A^T)
    double* cv = nullptr;
    std::unique_ptr<DeviceArena> mem;
};
DevMatrix upload_matrix(const Csc& A, cudaStream_t st);

struct SolveReport {
    int iterations = 0;
    bool converged = false;
    std::vector<double> residual_history;
    double t_solve = 0.0;
    long long launches = 0;
};

// Device workspace for CGLS (vectors of length M and N, scalars).
struct CglsWork {
    double *r, *t, *s, *p, *y, *v, *q, *partial, *scal;
    int* brk;
    int nblocks = 0;
    std::unique_ptr<DeviceArena> mem;
};
CglsWork make_cgls_work(int m, int n);

// Right-preconditioned CGLS (solve.cpp:24-76); d_b (M) and d_w (weights, N, may
// be null) on the device; u (N) written to d_u.
SolveReport gpu_cgls(const DevMatrix& A, const SolvePlan* W, const double* d_b, double* d_u, double tol, int maxit,
                     const double* d_w, CglsWork& ws, cudaStream_t st);

// Seminormal equations with refinement (solve.cpp:78-108).
SolveReport gpu_csne(const DevMatrix& A, const SolvePlan& W, const double* d_b, double* d_u, int refine, const double* d_w,
                     double tol, CglsWork& ws, cudaStream_t st);

}  // namespace spqr
