// Blocked batched Householder QR + compact-WY apply for large fronts on B200.
//
// Reference semantics: block_householder_qr (Eigen HouseholderQR, makeHouseholder
// convention) + apply_reflectors_left_t on the neighbour block
// (proj/src/dense_kernels.cpp:11-99).  The reference applies Q^T to the
// neighbour block through the compact-WY form H = I - V T V^T with T built by
// accumulate_wy (:41-53); here every panel of NB columns is factored once,
// its T is built the same way, and the panel's block reflector is applied to
// all trailing columns (the rest of the front and the neighbour block) as
// DMMA (mma.sync.m8n8k4.f64) GEMMs:  W = V^T C,  W = T^T W,  C -= V W.
// The final nonnegative-diagonal flip (dense_kernels.cpp:29-34, 89-92) is a
// separate row-flip pass.
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdlib>

#include <cooperative_groups.h>

#include "dev.h"

namespace spqr {

namespace {

constexpr int NB = 32;      // panel width
constexpr int CH = 64;      // row chunk staged per step
// padded leading dims: every DMMA fragment load (t4 + 4g or g + 8t4 patterns
// mod 16 doubles) touches 16 distinct bank pairs, i.e. the 2-wavefront minimum
constexpr int LDV = CH + 4;   // V chunk, (row, col) at row + col*LDV      (pass 1: A = V^T)
constexpr int LDVT = NB + 4;  // V chunk transposed, (row, col) at col + row*LDVT (pass 2: A = V)
constexpr int LDC = CH + 4;
constexpr int LDW = NB + 4;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ void dmma(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Panel factorisation, row-group layout: warp g owns a contiguous chunk of
// rows of the w <= 32 panel columns; within a warp, lanes stride the rows
// (coalesced in HBM or shared memory alike).  Per reflector: warps reduce the
// tail norm of column k over their rows (barrier), every thread forms the same
// Householder scalars (Eigen makeHouseholder), the warps scale their rows of
// column k and publish v (barrier), then each warp accumulates v^T a_j for all
// 32 columns in registers and folds them with a 31-shuffle transpose reduction
// (lane j ends with column j); per-warp partials are reduced (barrier) before
// the rank-1 update.  Lanes left of k carry v_j^T v_k from the same pass, which
// builds the compact-WY factor T column by column (accumulate_wy,
// dense_kernels.cpp:41-53).  The panel is staged in shared memory when it
// fits, else it is walked in place.
template <int NWP>
__global__ void __launch_bounds__(32 * NWP) k_panel2(double* __restrict__ a, int ld, long long stride, int m, int j0,
                                                     int w, double* __restrict__ tau_all, int tau_stride,
                                                     double* __restrict__ T_all, int smem_rows) {
    const int b = blockIdx.x;
    double* A = a + b * stride;
    double* tau = tau_all + static_cast<long long>(b) * tau_stride;
    double* T = T_all + static_cast<long long>(b) * NB * NB;
    extern __shared__ double sm[];
    __shared__ double red[NWP], part[NWP][32], Ts[NB * NB], gv[NB];
    __shared__ double s_c0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int rows = m - j0;
    const bool staged = rows <= smem_rows;
    double* P;
    long long pld;
    double* vsh;
    if (staged) {
        pld = rows;
        P = sm;
        vsh = sm + pld * w;
        for (int e = threadIdx.x; e < rows * w; e += blockDim.x) {
            const int j = e / rows, i = e - j * rows;
            P[i + j * pld] = A[(j0 + i) + static_cast<long long>(j0 + j) * ld];
        }
    } else {
        pld = ld;
        P = A + j0 + static_cast<long long>(j0) * ld;
        vsh = sm;
    }
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) Ts[e] = 0.0;
    __syncthreads();
    const int per = (((rows + NWP - 1) / NWP) + 31) & ~31;  // whole warps of rows
    const int r_lo = min(rows, wid * per), r_hi = min(rows, r_lo + per);
    const int kmax = min(w, rows);
    for (int k = 0; k < kmax; ++k) {
        double* pk = P + static_cast<long long>(k) * pld;
        double s = 0.0;
        for (int r = max(r_lo, k + 1) + lane; r < r_hi; r += 32) s = fma(pk[r], pk[r], s);
        s = wsum(s);
        if (lane == 0) red[wid] = s;
        if (lane == 0 && r_lo <= k && k < r_hi) s_c0 = pk[k];
        __syncthreads();
        double tail2 = 0.0;
#pragma unroll
        for (int g = 0; g < NWP; ++g) tail2 += red[g];
        const double c0 = s_c0;
        double t = 0.0, den = 0.0, beta = c0;
        if (!(tail2 <= DBL_MIN)) {
            beta = sqrt(c0 * c0 + tail2);
            if (c0 >= 0.0) beta = -beta;
            den = c0 - beta;
            t = (beta - c0) / beta;
        }
        for (int r = max(r_lo, k + 1) + lane; r < r_hi; r += 32) {
            const double v = (t == 0.0) ? 0.0 : pk[r] / den;
            pk[r] = v;
            vsh[r] = v;
        }
        if (lane == 0 && r_lo <= k && k < r_hi) {
            pk[k] = beta;
            vsh[k] = 1.0;
        }
        if (threadIdx.x == 0) tau[j0 + k] = t;
        __syncthreads();
        if (t != 0.0) {
            // acc[j] = sum over this warp's rows >= k of v * a_j (all 32 columns)
            double acc[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) acc[j] = 0.0;
            for (int r = max(r_lo, k) + lane; r < r_hi; r += 32) {
                const double v = vsh[r];
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < w) acc[j] = fma(v, P[r + j * pld], acc[j]);
            }
            // transpose reduction: lane j ends with column j's warp total
#pragma unroll
            for (int o = 16, cnt = 16; o >= 1; o >>= 1, cnt >>= 1) {
                const bool up = lane & o;
#pragma unroll
                for (int i = 0; i < cnt; ++i) {
                    const double send = up ? acc[i] : acc[i + cnt];
                    const double keep = up ? acc[i + cnt] : acc[i];
                    acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            part[wid][lane] = acc[0];
        }
        __syncthreads();
        if (t != 0.0) {
            double wl = 0.0;
#pragma unroll
            for (int g = 0; g < NWP; ++g) wl += part[g][lane];
            const double twl = (lane > k && lane < w) ? -t * wl : 0.0;
            double tws[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) tws[j] = __shfl_sync(0xffffffffu, twl, j);
            for (int r = max(r_lo, k) + lane; r < r_hi; r += 32) {
                const double v = vsh[r];
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j > k && j < w) P[r + j * pld] = fma(tws[j], v, P[r + j * pld]);
            }
            if (wid == 0) {  // T(:, k) = -t T(0:k, 0:k) (V^T v_k),  T(k, k) = t
                if (lane < k) gv[lane] = wl;
                __syncwarp();
                if (lane < k) {
                    double sacc = 0.0;
                    for (int l = lane; l < k; ++l) sacc = fma(Ts[lane + l * NB], gv[l], sacc);
                    Ts[lane + k * NB] = -t * sacc;
                }
                if (lane == 0) Ts[k + k * NB] = t;
                __syncwarp();
            }
        }
    }
    __syncthreads();
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) T[e] = Ts[e];
    if (staged)
        for (int e = threadIdx.x; e < rows * w; e += blockDim.x) {
            const int j = e / rows, i = e - j * rows;
            A[(j0 + i) + static_cast<long long>(j0 + j) * ld] = P[i + j * pld];
        }
}

// Tall panels (more rows than one SM's shared memory holds): a thread-block
// cluster of kCS CTAs per panel, CTA r keeping rows [r R, (r+1) R) of the w <= 32
// panel columns in its shared memory.  Per reflector there are two cluster
// barriers: the per-CTA partial tail norms of column k are exchanged through
// distributed shared memory (every CTA forms the same Householder scalars), then
// the per-CTA partial dot products of v_k with all panel columns (lanes left of
// k give V^T v_k for T).  Partials are double-buffered by step parity, so a
// CTA can start the next step while slower ones still read the previous one.
constexpr int kCS = 8;  // CTAs per cluster (portable maximum)

__global__ void __cluster_dims__(kCS, 1, 1) __launch_bounds__(256)
    k_panel_cluster(double* __restrict__ a, int ld, long long stride, int m, int j0, int w,
                    double* __restrict__ tau_all, int tau_stride, double* __restrict__ T_all, int R) {
    namespace cg = cooperative_groups;
    cg::cluster_group cluster = cg::this_cluster();
    const int rank = static_cast<int>(cluster.block_rank());
    const int b = blockIdx.x / kCS;
    double* A = a + b * stride;
    double* tau = tau_all + static_cast<long long>(b) * tau_stride;
    double* T = T_all + static_cast<long long>(b) * NB * NB;
    extern __shared__ double P[];  // R x w, column-major, ld R (this CTA's rows)
    __shared__ double nrm[2][2];   // [parity][tail sumsq, c0 (owner only)]
    __shared__ double dots[2][32]; // [parity][column]
    __shared__ double red[8][33];
    __shared__ double Ts[NB * NB], gv[NB];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int rows = m - j0;
    const int g0 = rank * R;                       // first panel row of this CTA
    const int nr = max(0, min(R, rows - g0));      // rows held here
    for (int e = threadIdx.x; e < nr * w; e += blockDim.x) {
        const int j = e / nr, i = e - j * nr;
        P[i + j * R] = A[(j0 + g0 + i) + static_cast<long long>(j0 + j) * ld];
    }
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) Ts[e] = 0.0;
    __syncthreads();
    const int kmax = min(w, rows);
    for (int k = 0; k < kmax; ++k) {
        const int par = k & 1;
        double* pk = P + k * R;
        // local rows > k of column k (global row index g0 + i)
        const int lo = max(0, k + 1 - g0);
        double s = 0.0;
        for (int i = lo + threadIdx.x; i < nr; i += blockDim.x) s = fma(pk[i], pk[i], s);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
        if (lane == 0) red[wid][0] = s;
        __syncthreads();
        if (threadIdx.x == 0) {
            double t = 0.0;
            for (int q = 0; q < 8; ++q) t += red[q][0];
            nrm[par][0] = t;
            nrm[par][1] = (k >= g0 && k < g0 + nr) ? pk[k - g0] : 0.0;
        }
        cluster.sync();
        double tail2 = 0.0, c0 = 0.0;
        for (int r = 0; r < kCS; ++r) {  // same order in every CTA
            const double* rn = cluster.map_shared_rank(&nrm[par][0], r);
            tail2 += rn[0];
            c0 += rn[1];  // only the owner of row k contributes
        }
        double t = 0.0, den = 0.0, beta = c0;
        if (!(tail2 <= DBL_MIN)) {
            beta = sqrt(c0 * c0 + tail2);
            if (c0 >= 0.0) beta = -beta;
            den = c0 - beta;
            t = (beta - c0) / beta;
        }
        for (int i = lo + threadIdx.x; i < nr; i += blockDim.x) pk[i] = (t == 0.0) ? 0.0 : pk[i] / den;
        if (threadIdx.x == 0) {
            if (k >= g0 && k < g0 + nr) pk[k - g0] = beta;
            if (rank == 0) tau[j0 + k] = t;
        }
        __syncthreads();
        // partial dots over local rows >= k: v_k^T a_j for every panel column j
        const int lo2 = max(0, k - g0);
        double acc[32];
#pragma unroll
        for (int j = 0; j < 32; ++j) acc[j] = 0.0;
        if (t != 0.0) {
            for (int i = lo2 + threadIdx.x; i < nr; i += blockDim.x) {
                const double v = (g0 + i == k) ? 1.0 : pk[i];
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j < w && j != k) acc[j] = fma(v, P[i + j * R], acc[j]);
            }
        }
        // lane j ends with column j's warp total, then the CTA total
#pragma unroll
        for (int o = 16, cnt = 16; o >= 1; o >>= 1, cnt >>= 1) {
            const bool up = lane & o;
#pragma unroll
            for (int i = 0; i < cnt; ++i) {
                const double send = up ? acc[i] : acc[i + cnt];
                const double keep = up ? acc[i + cnt] : acc[i];
                acc[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
            }
        }
        red[wid][lane] = acc[0];
        __syncthreads();
        if (wid == 0) {
            double tsum = 0.0;
            for (int q = 0; q < 8; ++q) tsum += red[q][lane];
            dots[par][lane] = tsum;
        }
        cluster.sync();
        double wl = 0.0;  // lane j: total v_k^T a_j over the cluster
        for (int r = 0; r < kCS; ++r) wl += cluster.map_shared_rank(&dots[par][0], r)[lane];
        if (t != 0.0) {
            const double twl = (lane > k && lane < w) ? -t * wl : 0.0;
            double tws[32];
#pragma unroll
            for (int j = 0; j < 32; ++j) tws[j] = __shfl_sync(0xffffffffu, twl, j);
            for (int i = lo2 + threadIdx.x; i < nr; i += blockDim.x) {
                const double v = (g0 + i == k) ? 1.0 : pk[i];
#pragma unroll
                for (int j = 0; j < 32; ++j)
                    if (j > k && j < w) P[i + j * R] = fma(tws[j], v, P[i + j * R]);
            }
            if (rank == 0 && wid == 0) {  // T(:, k) = -t T(0:k, 0:k) (V^T v_k),  T(k, k) = t
                if (lane < k) gv[lane] = wl;
                __syncwarp();
                if (lane < k) {
                    double sacc = 0.0;
                    for (int l = lane; l < k; ++l) sacc = fma(Ts[lane + l * NB], gv[l], sacc);
                    Ts[lane + k * NB] = -t * sacc;
                }
                if (lane == 0) Ts[k + k * NB] = t;
                __syncwarp();
            }
        }
        __syncthreads();
    }
    cluster.sync();  // no CTA exits while another may still read its partials
    if (rank == 0)
        for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) T[e] = Ts[e];
    for (int e = threadIdx.x; e < nr * w; e += blockDim.x) {
        const int j = e / nr, i = e - j * nr;
        A[(j0 + g0 + i) + static_cast<long long>(j0 + j) * ld] = P[i + j * R];
    }
}

// Block reflector on a TC-column tile of the trailing matrix:
//   W = V^T C (w x TC), W = T^T W, C -= V W.   16 warps, DMMA 8x8x4.
constexpr int TC2 = 128;

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool ok) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src), "r"(ok ? 8 : 0));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// The C chunks stream through two shared-memory buffers: the copy of chunk
// c+1 (cp.async, zero-filled outside the block) is in flight while the DMMA
// tiles of chunk c run.  Pass 2 writes the updated chunk back through shared
// memory so the global stores are coalesced column runs.
// NWARP = 16: warp tiles 8x32 (W) and 8x64 (C chunk); NWARP = 8: 16x32 and 16x64,
// half the fragment loads per DMMA and twice the accumulators per warp.
template <int NWARP>
__global__ void __launch_bounds__(32 * NWARP) k_wy(double* __restrict__ a, int ld, long long stride, int m, int ntot,
                                                   int j0, int w, const double* __restrict__ T_all) {
    constexpr int PM = 64 / (NWARP * 4), PN = 4;   // pass 1 / T^T W: m-tiles x n-tiles per warp
    constexpr int MG = 4 / PM;                    // m-groups over the 4 W row tiles
    constexpr int QM = 128 / (NWARP * 8), QN = 8;  // pass 2: m-tiles x n-tiles per warp
    constexpr int QG = 8 / QM;                     // m-groups over the 8 chunk row tiles
    const int b = blockIdx.y;
    double* A = a + b * stride;
    const double* T = T_all + static_cast<long long>(b) * NB * NB;
    const int c0 = j0 + w + blockIdx.x * TC2;  // first column of this tile
    const int nc = min(TC2, ntot - c0);
    if (nc <= 0) return;
    extern __shared__ double dsm[];
    // V chunks (pass 1: CH x NB column-major, ld LDV; pass 2 transposed, ld LDVT)
    constexpr int VSZ = (NB * LDV > CH * LDVT) ? NB * LDV : CH * LDVT;
    double* sVb[2] = {dsm, dsm + VSZ};
    double* sCb[2] = {dsm + 2 * VSZ, dsm + 2 * VSZ + TC2 * LDC};  // C chunks, ld LDC
    double* sW = sCb[1] + TC2 * LDC;   // W (NB x TC2), column-major, ld LDW
    double* sT = sW + TC2 * LDW;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) {
        const int i = e % NB, j = e / NB;
        sT[i + j * LDW] = (i < w && j < w) ? T[e] : 0.0;
    }
    const int rows = m - j0;
    const int nchunk = (rows + CH - 1) / CH;
    // chunk c of C and of V (unit lower trapezoid: the rows at or above the
    // diagonal are written directly, the rest streams in with cp.async)
    auto issue = [&](int c, bool transposed) {
        const int r0 = c * CH, rc = min(CH, rows - r0);
        double* cb = sCb[c & 1];
        double* vb = sVb[c & 1];
        for (int e = threadIdx.x; e < CH * TC2; e += blockDim.x) {
            const int i = e % CH, j = e / CH;
            const bool ok = i < rc && j < nc;
            cp_async8(cb + i + j * LDC, ok ? A + (j0 + r0 + i) + static_cast<long long>(c0 + j) * ld : A, ok);
        }
        for (int e = threadIdx.x; e < CH * NB; e += blockDim.x) {
            const int i = e % CH, j = e / CH, r = r0 + i;
            double* dst = transposed ? vb + j + i * LDVT : vb + i + j * LDV;
            if (i < rc && j < w && r <= j)
                *dst = (r == j) ? 1.0 : 0.0;
            else {
                const bool ok = i < rc && j < w;
                cp_async8(dst, ok ? A + (j0 + r) + static_cast<long long>(j0 + j) * ld : A, ok);
            }
        }
        cp_commit();
    };
    // ---- pass 1: W = V^T C; warp: W row tiles mg*PM.., column tiles ng*PN..
    const int mg = wid % MG, ng = wid / MG;
    double acc[PM][PN][2] = {};
    issue(0, false);
    for (int c = 0; c < nchunk; ++c) {
        if (c + 1 < nchunk) issue(c + 1, false);
        if (c + 1 < nchunk)
            cp_wait<1>();
        else
            cp_wait<0>();
        __syncthreads();
        const double* sC = sCb[c & 1];
        const double* sV = sVb[c & 1];
#pragma unroll 4
        for (int k0 = 0; k0 < CH; k0 += 4) {
            double av[PM], bv[PN];
#pragma unroll
            for (int i = 0; i < PM; ++i) av[i] = sV[(k0 + t4) + ((mg * PM + i) * 8 + g) * LDV];
#pragma unroll
            for (int q = 0; q < PN; ++q) bv[q] = sC[(k0 + t4) + ((ng * PN + q) * 8 + g) * LDC];
#pragma unroll
            for (int i = 0; i < PM; ++i)
#pragma unroll
                for (int q = 0; q < PN; ++q) dmma(acc[i][q][0], acc[i][q][1], av[i], bv[q]);
        }
        __syncthreads();
    }
    issue(0, true);  // pass 2's first chunk streams in while W is finished
#pragma unroll
    for (int i = 0; i < PM; ++i)
#pragma unroll
        for (int q = 0; q < PN; ++q) {
            sW[((mg * PM + i) * 8 + g) + ((ng * PN + q) * 8 + 2 * t4) * LDW] = acc[i][q][0];
            sW[((mg * PM + i) * 8 + g) + ((ng * PN + q) * 8 + 2 * t4 + 1) * LDW] = acc[i][q][1];
        }
    __syncthreads();
    // ---- W2 = T^T W
    double acc2[PM][PN][2] = {};
#pragma unroll
    for (int k0 = 0; k0 < NB; k0 += 4) {
        double av[PM], bv[PN];
#pragma unroll
        for (int i = 0; i < PM; ++i) av[i] = sT[(k0 + t4) + ((mg * PM + i) * 8 + g) * LDW];
#pragma unroll
        for (int q = 0; q < PN; ++q) bv[q] = sW[(k0 + t4) + ((ng * PN + q) * 8 + g) * LDW];
#pragma unroll
        for (int i = 0; i < PM; ++i)
#pragma unroll
            for (int q = 0; q < PN; ++q) dmma(acc2[i][q][0], acc2[i][q][1], av[i], bv[q]);
    }
    __syncthreads();
#pragma unroll
    for (int i = 0; i < PM; ++i)
#pragma unroll
        for (int q = 0; q < PN; ++q) {
            sW[((mg * PM + i) * 8 + g) + ((ng * PN + q) * 8 + 2 * t4) * LDW] = acc2[i][q][0];
            sW[((mg * PM + i) * 8 + g) + ((ng * PN + q) * 8 + 2 * t4 + 1) * LDW] = acc2[i][q][1];
        }
    // ---- pass 2: C -= V W2; warp: chunk row tiles qg*QM.., column tiles qn*QN..
    const int qg = wid % QG, qn = wid / QG;
    for (int c = 0; c < nchunk; ++c) {
        const int r0 = c * CH, rc = min(CH, rows - r0);
        if (c + 1 < nchunk) issue(c + 1, true);
        if (c + 1 < nchunk)
            cp_wait<1>();
        else
            cp_wait<0>();
        __syncthreads();
        double* sC = sCb[c & 1];
        const double* sVt = sVb[c & 1];
        double o[QM][QN][2] = {};
#pragma unroll
        for (int k0 = 0; k0 < NB; k0 += 4) {
            double av[QM], bv[QN];
#pragma unroll
            for (int i = 0; i < QM; ++i) av[i] = sVt[(k0 + t4) + ((qg * QM + i) * 8 + g) * LDVT];
#pragma unroll
            for (int q = 0; q < QN; ++q) bv[q] = sW[(k0 + t4) + ((qn * QN + q) * 8 + g) * LDW];
#pragma unroll
            for (int i = 0; i < QM; ++i)
#pragma unroll
                for (int q = 0; q < QN; ++q) dmma(o[i][q][0], o[i][q][1], av[i], bv[q]);
        }
#pragma unroll
        for (int i = 0; i < QM; ++i)
#pragma unroll
            for (int q = 0; q < QN; ++q) {  // each element is read and written by its own thread only
                const int row = (qg * QM + i) * 8 + g, col = (qn * QN + q) * 8 + 2 * t4;
                sC[row + col * LDC] -= o[i][q][0];
                sC[row + (col + 1) * LDC] -= o[i][q][1];
            }
        __syncthreads();
        for (int e = threadIdx.x; e < CH * TC2; e += blockDim.x) {
            const int i = e % CH, j = e / CH;
            if (i < rc && j < nc) A[(j0 + r0 + i) + static_cast<long long>(c0 + j) * ld] = sC[i + j * LDC];
        }
        __syncthreads();
    }
}

// nonnegative diagonal: flip rows of R (cols i..) and of the neighbour block;
// sign and first zero/denormal pivot per problem
__global__ void k_flip(double* __restrict__ a, int ld, long long stride, int n, int ntot, double* __restrict__ sign_all,
                       int* __restrict__ info) {
    const int b = blockIdx.y;
    double* A = a + b * stride;
    for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < ntot; j += gridDim.x * blockDim.x) {
        const int top = j < n ? j + 1 : n;
        for (int i = 0; i < top; ++i)
            if (A[i + static_cast<long long>(i) * ld] < 0.0 && i != j) A[i + static_cast<long long>(j) * ld] = -A[i + static_cast<long long>(j) * ld];
    }
    __syncthreads();
    if (blockIdx.x == 0) {
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double r = A[i + static_cast<long long>(i) * ld];
            sign_all[static_cast<long long>(b) * n + i] = r < 0.0 ? -1.0 : 1.0;
            if (info && !(fabs(r) >= DBL_MIN)) atomicMin(info + b, i);
        }
    }
}

__global__ void k_flip_diag(double* __restrict__ a, int ld, long long stride, int n) {
    const int b = blockIdx.x;
    double* A = a + b * stride;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double* d = A + i + static_cast<long long>(i) * ld;
        if (*d < 0.0) *d = -*d;
    }
}

// epilogue for engine fronts factored by the blocked path: R copy (upper n x n),
// optional [I;0] overwrite of the factored columns, or clearing V below the diagonal
__global__ void k_qr_post(double* __restrict__ a, int ld, int m, int n, double* __restrict__ rout, int set_identity,
                          int zero_lower) {
    const long long total = static_cast<long long>(m) * n;
    for (long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; e < total;
         e += static_cast<long long>(gridDim.x) * blockDim.x) {
        const int i = static_cast<int>(e % m), j = static_cast<int>(e / m);
        double* x = a + i + static_cast<long long>(j) * ld;
        if (rout && i < n) rout[i + static_cast<long long>(j) * n] = (i <= j) ? *x : 0.0;
        if (set_identity)
            *x = (i == j) ? 1.0 : 0.0;
        else if (zero_lower && i > j)
            *x = 0.0;
    }
}

}  // namespace

void blocked_qr_post(double* a, int ld, int m, int n, double* rout, int set_identity, int zero_lower, cudaStream_t st) {
    const long long total = static_cast<long long>(m) * n;
    const int grid = static_cast<int>(std::min<long long>((total + 255) / 256, 4096));
    if (total > 0) k_qr_post<<<grid, 256, 0, st>>>(a, ld, m, n, rout, set_identity, zero_lower);
}

// nb problems, each m x ntot column-major (ld = m, packed), QR of the first n
// columns + H^T applied to the rest; tau/sign n per problem; info per problem.
void blocked_qr_apply(int nbatch, int m, int n, int ntot, double* d_a, double* d_tau, double* d_sign, int* d_info,
                      double* d_T, cudaStream_t st, int ld_in) {
    const int ldA = ld_in > 0 ? ld_in : m;
    const long long stride = static_cast<long long>(ldA) * ntot;
    const size_t smem_cap = 160 * 1024;
    for (int j0 = 0; j0 < n; j0 += NB) {
        const int w = std::min(NB, n - j0);
        const int rows = m - j0;
        // staged panel: (rows|1) x w plus v (rows); else in place with v in shared memory
        const int smem_rows = static_cast<int>(smem_cap / (sizeof(double) * (NB + 1))) - 2;
        const size_t smem = rows <= smem_rows ? sizeof(double) * (rows * static_cast<size_t>(w) + rows)
                                              : sizeof(double) * static_cast<size_t>(rows);
        // tall panels: a cluster of kCS CTAs holds the rows in distributed shared memory
        const int Rc = ((rows + kCS - 1) / kCS + 31) & ~31;
        if (rows > smem_rows && static_cast<size_t>(Rc) * w * sizeof(double) <= 200 * 1024 &&
            !std::getenv("SPQR_NO_CLUSTER_PANEL")) {
            const size_t csmem = sizeof(double) * static_cast<size_t>(Rc) * w;
            static size_t cfg = 0;
            smem_optin(reinterpret_cast<const void*>(k_panel_cluster), csmem, cfg);
            k_panel_cluster<<<nbatch * kCS, 256, csmem, st>>>(d_a, ldA, stride, m, j0, w, d_tau, n, d_T, Rc);
        } else if (rows <= 512) {
            static size_t cfg = 0;
            smem_optin(reinterpret_cast<const void*>(k_panel2<8>), smem, cfg);
            k_panel2<8><<<nbatch, 256, smem, st>>>(d_a, ldA, stride, m, j0, w, d_tau, n, d_T, smem_rows);
        } else {
            static size_t cfg = 0;
            smem_optin(reinterpret_cast<const void*>(k_panel2<16>), smem, cfg);
            k_panel2<16><<<nbatch, 512, smem, st>>>(d_a, ldA, stride, m, j0, w, d_tau, n, d_T, smem_rows);
        }
        const int trail = ntot - (j0 + w);
        if (trail > 0) {
            dim3 grid((trail + TC2 - 1) / TC2, nbatch);
            const size_t vsz = std::max(NB * LDV, CH * LDVT);
            const size_t wsm = sizeof(double) * (2 * vsz + 2 * TC2 * LDC + TC2 * LDW + NB * LDW);
            static const bool wy8 = std::getenv("SPQR_WY8") != nullptr;  // 8-warp variant: measured no faster
            if (wy8) {
                static size_t cfg = 0;
                smem_optin(reinterpret_cast<const void*>(k_wy<8>), wsm, cfg);
                k_wy<8><<<grid, 256, wsm, st>>>(d_a, ldA, stride, m, ntot, j0, w, d_T);
            } else {
                static size_t cfg = 0;
                smem_optin(reinterpret_cast<const void*>(k_wy<16>), wsm, cfg);
                k_wy<16><<<grid, 512, wsm, st>>>(d_a, ldA, stride, m, ntot, j0, w, d_T);
            }
        }
    }
    dim3 g2((ntot + 255) / 256, nbatch);
    k_flip<<<g2, 256, 0, st>>>(d_a, ldA, stride, n, ntot, d_sign, d_info);
    k_flip_diag<<<nbatch, 256, 0, st>>>(d_a, ldA, stride, n);
}

}  // namespace spqr
