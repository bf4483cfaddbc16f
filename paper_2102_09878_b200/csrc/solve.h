// W sweeps and preconditioned CGLS on the device (proj/src/transforms.cpp:40-111,
// proj/src/solve.cpp:24-108).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "dev.h"
#include "devmem.h"
#include "engine.h"

namespace spqr {

enum SweepMode { kWSolve = 0, kWtSolve = 1, kWApply = 2, kWtApply = 3 };

// Level schedules of W (transforms.cpp:40-111), one per sweep mode.  A sweep walks W
// forward (w_apply, wt_solve) or backward (w_solve, wt_apply); each factor reads and
// writes z[cols] and either reads z[coupled] (w_solve / w_apply) or accumulates into it
// (wt_solve / wt_apply).  A factor's level is one past the last level of any earlier
// (in walk order) factor it conflicts with — read-after-write, write-after-read,
// write-after-write on cols, and a read of an accumulated column — while two
// accumulations into one column may share a level (the per-level reduction applies
// them in walk order).  Every level is one launch (+ one for the wide factors, + one
// reduction): C2 goes from ~400 engine batches per sweep to ~35 levels.
struct SolvePlan {
    struct Level {
        const WFac* fac = nullptr;  // warp per factor
        int nf = 0, maxc = 0;
        const WFac* bfac = nullptr;  // CTA per factor (c >= kBigFactorCols)
        int nbf = 0, bmaxc = 0;
        const int *rptr = nullptr, *ridx = nullptr, *rcol = nullptr;  // accumulation lists
        int ncol = 0;
    };
    struct Schedule {
        std::vector<Level> levels;
        long long launches = 0;
        bool built = false;
    };
    Schedule sched[4];  // by SweepMode; w_apply / wt_apply are built on first use
    const int* d_idx = nullptr;
    double* contrib = nullptr;
    long long ncontrib = 0;
    int maxc = 1, bmaxc = 1;
    std::unique_ptr<DeviceArena> mem;
    long long launches_per_sweep_t = 0, launches_per_sweep = 0;  // wt_solve / w_solve
    double t_build = 0.0;
    // algorithmic HBM bytes of one sweep: 8 nnz(W) + 16 (gathered entries:
    // z[cols] read + written, z[coupled] read or accumulated)
    double sweep_bytes = 0.0;
};
SolvePlan build_solve_plan(const DeviceFactorization& F, cudaStream_t st);
void ensure_schedule(SolvePlan& P, const DeviceFactorization& F, SweepMode mode, cudaStream_t st);

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
    double sweep_ms = 0.0;  // device time of the W sweeps (CUDA events, also inside the graphs)
    int sweeps = 0;
};

// Device workspace for CGLS (vectors of length M and N, scalars).
struct CglsWork {
    double *r = nullptr, *t = nullptr, *s = nullptr, *p = nullptr, *y = nullptr, *v = nullptr, *q = nullptr;
    double *partial = nullptr, *scal = nullptr;
    int* brk = nullptr;
    double* hpin = nullptr;  // pinned: ||w.t||^2 and the breakdown flag of each iteration
    int nblocks = 0;
    std::unique_ptr<DeviceArena> mem;
    CglsWork() = default;
    CglsWork(CglsWork&& o) noexcept { *this = std::move(o); }
    CglsWork& operator=(CglsWork&& o) noexcept {
        std::swap(r, o.r), std::swap(t, o.t), std::swap(s, o.s), std::swap(p, o.p), std::swap(y, o.y);
        std::swap(v, o.v), std::swap(q, o.q), std::swap(partial, o.partial), std::swap(scal, o.scal);
        std::swap(brk, o.brk), std::swap(hpin, o.hpin), std::swap(nblocks, o.nblocks), std::swap(mem, o.mem);
        return *this;
    }
    ~CglsWork() {
        if (hpin) cudaFreeHost(hpin);
    }
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
