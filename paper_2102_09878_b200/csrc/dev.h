// Device-side descriptors and launchers for the spaQR front kernels (sm_100a).
//
// All front data is FP64 column-major in HBM.  Every batched kernel takes a
// flat array of per-problem descriptors built by the host engine each phase,
// so one launch covers every front of a stage (thousands of tiny, variable
// size problems) — the reference's per-cluster Eigen calls
// (proj/src/factorize.cpp) become one launch per phase.
#pragma once

#include <cstddef>
#include <cstdint>

#include <cuda_runtime.h>

#include <atomic>
#include <mutex>
#include <vector>

namespace spqr {

// Householder sign rule.  Eigen's makeHouseholder (the arithmetic
// behind block_householder_qr, dense_kernels.cpp:11-35) takes beta = -sign(c0)*||x||,
// beta = -||x|| for c0 >= 0.  When c0 is roundoff-sized next to the tail
// (c0^2 <= 1e-20 * ||x_tail||^2, i.e. |c0| <= 1e-10 ||x_tail||) its sign is not a
// property of the data — Eigen's own blocked arithmetic decides it by roundoff — yet
// it selects which of two valid reflectors is used, and with it the complement rows
// that move_extras redistributes.  Every restatement (GPU kernels, oracle/orc_dense.cpp,
// oracle/eigen_shim) therefore takes beta = -||x|| there.
constexpr double kHhSignTol2 = 1e-20;
__host__ __device__ __forceinline__ bool hh_beta_negative(double c0, double tail2) {
    return c0 >= 0.0 || c0 * c0 <= kHhSignTol2 * tail2;
}

// Opt in to `bytes` of dynamic shared memory for `func` on the current device.  The 48 KB
// default limit covers static + dynamic shared memory together, so the attribute is raised
// whenever a launch needs more than any earlier one.  `configured` is a per-call-site static
// holding the opted-in size per device (the attribute is per device); the slow path is
// serialised so a concurrent caller never launches before the attribute covers it.
constexpr int kMaxDevices = 64;
struct SmemCfg {
    std::atomic<size_t> v[kMaxDevices] = {};
};
inline void smem_optin(const void* func, size_t bytes, SmemCfg& configured) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= kMaxDevices) dev = 0;
    if (configured.v[dev].load(std::memory_order_acquire) >= bytes) return;
    static std::mutex mu;
    std::lock_guard<std::mutex> lk(mu);
    if (configured.v[dev].load(std::memory_order_relaxed) >= bytes) return;
    if (cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(bytes)) ==
        cudaSuccess)
        configured.v[dev].store(bytes, std::memory_order_release);
}

// ---- generic gather ("assemble"): builds a destination matrix from rows of
// up to a few source matrices.  The destination's columns are split into
// segments (seg_off[q] <= j < seg_off[q+1]); kmap[q*nsrc + t] gives the
// first source column of segment q in source slot t (-1: unmapped, -2: the
// segment is an identity block, value 1 on dst row == offset in segment).
// rowref = (s1, r1, s2, r2): dst(i,j) comes from slot s1 row r1 if that
// slot maps j's segment, else from slot s2 row r2, else 0.  s1 == -2 selects
// scan mode: the first slot mapping the segment supplies row r1.
// Covers stack gathers, scatter-back, row appends, merges and transposed
// copies (element (r,c) of a source lives at p[r*rs + c*cs]).
struct AsmSrc {
    const double* p;
    long long rs, cs;
};
struct AsmDst {
    double* p;
    int ld, nrows, ncols, nsrc, nseg;
    int trans;           // 1: (nrows x ncols) is the logical view; stored transposed (p[j + i*ld])
    long long row_off;   // into rowref (int4 per logical row)
    long long seg_off;   // into segoff (nseg + 1 ints)
    long long kmap_off;  // into kmap (nseg * nsrc)
    long long src_off;   // into src table
    long long elem_off;  // exclusive prefix of nrows*ncols (work split)
};

// ---- row / block statistics (decisions made on the host from these)
// mode 0: out_sq[off+i] = sum_j a(r0+i, c0+j)^2 (j ascending), out_nz[off+i] = any nonzero
// mode 1: out_sq[off]   = max |a| over the block,             out_nz[off]   = any nonzero
// mode 2: out_nz[off]   = block is exactly [I; 0]
struct StatDesc {
    const double* p;
    int ld, r0, nrows, c0, ncols, mode;
    long long out_off;
    long long work_off;  // see layout_stats
};

// Assigns work_off: mode 0 = one thread per row; modes 1/2 = warps of 32
// threads, 256 elements per warp, starting 32-aligned.  Returns the total.
inline long long layout_stats(StatDesc* v, size_t n) {
    long long w = 0;
    for (size_t i = 0; i < n; ++i) {
        StatDesc& d = v[i];
        if (d.mode == 0) {
            d.work_off = w;
            w += d.nrows;
        } else {
            w = (w + 31) & ~31LL;
            d.work_off = w;
            w += 32 * ((static_cast<long long>(d.nrows) * d.ncols + 255) / 256);
        }
    }
    return w;
}

// ---- batched Householder QR of the first n columns of an m x ntot block,
// reflectors applied (H^T, then the sign flip) to columns [n, ntot).  Eigen's
// makeHouseholder convention + the reference's nonnegative-diagonal flip
// (dense_kernels.cpp:11-35, 96-99).  R (flipped) stays in the upper triangle,
// V (unit diagonal implicit) below it.
struct QrDesc {
    double* a;
    int ld, m, n, ntot;
    double* tau;      // n  (may be null)
    double* sign;     // n  (may be null)
    double* rout;     // optional copy of R (n x n, ld = n)
    int* flag;        // atomicMin'd with the first i with |R_ii| < DBL_MIN (init INT_MAX; dense_kernels.cpp:234-240)
    int set_identity; // after the update: A(:, :n) := [I; 0]  (factorize.cpp:473-474)
    int zero_lower;   // after the update: clear V below the diagonal (R alone remains)
};

// ---- B <- B R^{-1} (right, upper, no transpose): factorize.cpp:475-478
struct TrsmDesc {
    double* b;
    int ldb, nrows, n;
    const double* r;
    int ldr;
    long long work_off;  // exclusive prefix of nrows
};

// ---- truncated column-pivoted QR in place (dense_kernels.cpp:124-232).
// On exit rows [0, rank) of the block hold R in the ORIGINAL column order.
struct CpqrDesc {
    double* a;
    int ld, m, n;
    double eps;
    int* rank;         // out
    double* r11;       // out
    double* V;         // optional: m x rank reflectors (ld = ldv), unit diag
    int ldv;
    double* tau;       // optional
    double* sign;      // optional
    int* perm;         // optional: pivot order (original column ids)
    double* work;      // 2n doubles + n ints scratch
};

// launchers (kernels.cu); all enqueue on `st`
void launch_assemble(const AsmDst* d_dst, int ndst, long long total_elems, const int4* d_rowref, const int* d_segoff,
                     const int* d_kmap, const AsmSrc* d_src, cudaStream_t st);
void launch_stats(const StatDesc* d, int nd, long long total_work, double* out_sq, unsigned char* out_nz,
                  cudaStream_t st);
// Size-split launches: problems listed in d_small are staged in shared memory
// (smem_small = the largest staged footprint), the rest run in place in HBM.
constexpr size_t kSmemBudget = 100 * 1024;  // two CTAs per SM
inline size_t qr_smem_bytes(int m, int n, int ntot) { return 8ull * (static_cast<size_t>(m) * ntot + n); }
inline size_t cpqr_smem_bytes(int m, int n) { return 8ull * (static_cast<size_t>(m) * n + 2ull * n + m) + 4ull * n + 16; }
void launch_qr_split(const QrDesc* d_desc, const int* d_small, int n_small, size_t smem_small, const int* d_large,
                     int n_large, cudaStream_t st);
void launch_cpqr_split(const CpqrDesc* d_desc, const int* d_small, int n_small, size_t smem_small, const int* d_large,
                       int n_large, int max_m_large, cudaStream_t st);
void launch_trsm(const TrsmDesc* d, int nd, long long total_rows, cudaStream_t st);
// store_q: reflectors of an in-place QR copied out (unit diagonal), then the block restored
enum { VCOPY_ZERO_LOWER = 1, VCOPY_SET_IDENTITY = 2 };
struct VCopyDesc {
    double* src;
    int lds, m, n, mode;
    double* dst;  // m x n, ld m
};
void launch_vcopy(const VCopyDesc* d, int nd, cudaStream_t st);
void launch_scatter_values(const long long* off, const double* val, long long n, double* base, cudaStream_t st);

// W-sweep kernels (solve) ------------------------------------------------------
struct WFac {
    int kind;     // 0 triangular (R | C), 1 rotation (V, tau, sign)
    int c;        // |cols|
    int k;        // |coupled| (triangular) or reflector count (rotation)
    int pad;
    const int* cols;
    const int* coupled;
    const double* a;  // triangular: [R | C] c x (c+k), ld = c ; rotation: V c x k, ld = c
    const double* tau;
    const double* sign;
    long long contrib_off;  // wt_solve: offset of this factor's C^T zs contribution
};
// mode 0 w_solve, 1 wt_solve (writes C^T zs contributions), 2 w_apply, 3 wt_apply (contributions)
void launch_wsweep(const WFac* f, int nf, double* z, double* contrib, int mode, int maxc, cudaStream_t st);
// factors with c >= kBigFactorCols: one CTA each (k_wsweep_big)
constexpr int kBigFactorCols = 192;
void launch_wsweep_big(const WFac* f, int nf, double* z, double* contrib, int mode, int maxc, cudaStream_t st);
// d_info[i] == INT_MAX (no singular pivot) -> -1, on st
void launch_info_fixup(int* info, int n, cudaStream_t st);
// opt in to the largest dynamic shared memory any level needs, before graph capture
void prepare_wsweep(int maxc, int bmaxc);
// z[col[t]] (+/-)= contrib[idx[ptr[t]..ptr[t+1])] in order
void launch_wreduce(const int* ptr, const int* idx, const int* col, int ncol, const double* contrib, double* z,
                    double sgn, cudaStream_t st);

// CGLS vector kernels
void launch_spmv_csr(int m, const int* ptr, const int* idx, const double* val, const double* x, double* y,
                     cudaStream_t st);
void launch_dot_partial(int n, const double* a, const double* b, const double* w, double* partial, int nblocks,
                        cudaStream_t st);
void launch_finish_sum(const double* partial, int nblocks, double* out, cudaStream_t st);
void launch_cgls_alpha(const double* gamma, const double* qq, double* alpha, int* brk, cudaStream_t st);
void launch_axpy_dev(int n, const double* alpha, double sgn, const double* x, double* y, cudaStream_t st);
void launch_cgls_p_update(int n, const double* s, const double* gnew, const double* gold, double* p, cudaStream_t st);
void launch_copy(int n, const double* a, double* b, cudaStream_t st);

// blocked batched QR + compact-WY apply (mbqr.cu) for fronts too large to stage:
// d_T needs nbatch * 32 * 32 doubles of scratch
void blocked_qr_apply(int nbatch, int m, int n, int ntot, double* d_a, double* d_tau, double* d_sign, int* d_info,
                      double* d_T, cudaStream_t st, int ld = 0);
void blocked_qr_post(double* a, int ld, int m, int n, double* rout, int set_identity, int zero_lower, cudaStream_t st);
constexpr size_t kBlockedQrBytes = size_t(2) << 20;  // fronts above this use the blocked DMMA path

// column-tiled QR (qr_tile.cu): panel m x n staged in shared memory, trailing
// columns in tiles [work.y, work.z) of front work.x; work.w = number of tiles of
// that front.  Class -1 = not eligible.
constexpr int kQrTileMaxN = 128;
constexpr size_t kQrTileSmem = 200 * 1024;
int qr_tile_class(int m, int n);
size_t qr_tile_smem(int cls, int n);  // dynamic smem of class cls (rows padded to 32 << cls)
// d_count: one int per descriptor, zero on entry (left zero on exit)
void launch_qr_tile(int cls, const QrDesc* d_desc, const int4* d_work, int nwork, size_t smem, int* d_count,
                    cudaStream_t st);
// work list for the fronts idx[] of one class (host); tiles sized so the launch
// has about two CTAs per SM
std::vector<int4> qr_tile_plan(const QrDesc* hq, const int* idx, int cnt, int sms);
// compact-WY tensor-core variant for fronts of 65..128 rows, panels of <= 32 columns and a
// trailing block of >= 64 columns (same work plan and election counter as the tiled kernel)
bool qr_wy_ok(int m, int n, int ntot);  // shape test
bool qr_wy_enabled();                  // SPQR_NO_WY=1 keeps every front on the column-tiled kernel (comparisons, tests)
void launch_qr_wy(const QrDesc* d_desc, const int4* d_work, int nwork, int* d_count, cudaStream_t st);

// grid-cooperative CPQR of one large problem (cpqr_big.cu); d.work needs
// cpqr_big_work_doubles(n) doubles
// short-wide CPQR (cpqr_narrow.cu): m <= 128, n <= 2048
// class 0..11 (see cpqr_narrow.cu); -1 not eligible
int cpqr_narrow_class(int m, int n);
size_t cpqr_narrow_smem(int m, int n);
void launch_cpqr_narrow(int cls, const CpqrDesc* d_desc, const int* d_idx, int cnt, size_t smem, cudaStream_t st);
// taller blocks (128 < m <= 512, n <= 2048), in place, warp per column (cpqr_narrow.cu)
int cpqr_tall_class(int m, int n);
void launch_cpqr_tall(int cls, const CpqrDesc* d_desc, const int* d_idx, int cnt, cudaStream_t st);
void launch_cpqr_big(const CpqrDesc& d, cudaStream_t st);
// one problem per thread-block cluster of cpqr_clus_ctas() CTAs (cpqr_big.cu k_cpqr_clus)
int cpqr_clus_ctas();
size_t cpqr_clus_smem_bytes(int m, int n);
void launch_cpqr_clus(const CpqrDesc* ds, const int* idx, int np, size_t smem, cudaStream_t st);
size_t cpqr_big_smem_bytes(int m, int n);  // dynamic smem of one launch (<= 200 KB to be eligible)
inline size_t cpqr_big_work_doubles(int n) { return 3 * static_cast<size_t>(n) + 2 * 512 + 16; }
constexpr size_t kBigCpqrBytes = size_t(2) << 20;

int sm_count();

}  // namespace spqr
