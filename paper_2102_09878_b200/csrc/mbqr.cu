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
#include <cstdint>
#include <algorithm>
#include <mutex>
#include <stdexcept>
#include <string>

#include <cooperative_groups.h>

#include "dev.h"
#include "devmem.h"

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
            if (hh_beta_negative(c0, tail2)) beta = -beta;
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
            if (hh_beta_negative(c0, tail2)) beta = -beta;
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
__device__ __forceinline__ void cp_async16(double* dst, const double* src) {
    const unsigned d = static_cast<unsigned>(__cvta_generic_to_shared(dst));
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(d), "l"(src));
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
// sign and first zero/denormal pivot per problem.  CTA = 32 columns of one
// problem: the diagonal's signs are staged in shared memory, then threads walk
// the rows of each column (coalesced).  The diagonal itself is flipped by
// k_flip_diag afterwards.
constexpr int kFlipCols = 32, kFlipMaxN = 8192;
__global__ void __launch_bounds__(256) k_flip(double* __restrict__ a, int ld, long long stride, int n, int ntot,
                                              double* __restrict__ sign_all, int* __restrict__ info) {
    const int b = blockIdx.y;
    double* A = a + b * stride;
    __shared__ unsigned char neg[kFlipMaxN];
    for (int i = threadIdx.x; i < n; i += blockDim.x) neg[i] = A[i + static_cast<long long>(i) * ld] < 0.0;
    __syncthreads();
    const int c0 = blockIdx.x * kFlipCols;
    for (int j = c0; j < min(ntot, c0 + kFlipCols); ++j) {
        const int top = j < n ? j : n;  // rows i < top (the diagonal excluded)
        double* col = A + static_cast<long long>(j) * ld;
        for (int i = threadIdx.x; i < top; i += blockDim.x)
            if (neg[i]) col[i] = -col[i];
    }
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


// Register-resident panel factorisation for the two-level path, row layout:
// CTA rank r of a CS-CTA cluster holds panel rows [r NW 32 RR, (r+1) NW 32 RR);
// thread (warp g, lane l) holds rows base + g 32 RR + l + 32 q (q < RR), all w <= 32
// panel columns, in registers.  The reflector loop is unrolled UB at a time with the register
// columns rotated after every group (see below), so column indices are compile-time.  Per
// reflector ONE reduction round: the products of the
// pivot column's tail with every column (its own: the tail norm) by a transpose
// reduction (lane j ends with column j) and the pivot row, one block barrier; the same
// Householder scalars in every thread (Eigen makeHouseholder), v formed in place,
// v^T x_j = x_j(k) + (tail^T x_j) / (c0 - beta) broadcast through a per-warp shared-memory
// row and the rank-1 update of the columns right of k.  Lanes left of k carry V^T v_k, which builds the
// panel's compact-WY T (accumulate_wy, dense_kernels.cpp:41-53).  With CS > 1 each CTA
// pushes its column sums (rank 0: and the pivot row) into every CTA's shared memory
// (remote stores), one cluster barrier per reflector, and every CTA adds the CS partials
// in rank order (double-buffered by parity).
constexpr int kPanelUB = 8;  // reflectors unrolled per group (NB must be a multiple)
template <int NW, int RR, int CS, int UB>
__device__ __forceinline__ void panel_row_body(double* __restrict__ a, int ld, long long stride, int m, int j0, int w,
                                               double* __restrict__ tau_all, int tau_stride,
                                               double* __restrict__ T_all) {
    namespace cg = cooperative_groups;
    constexpr int R = NW * 32 * RR;
    const int rank = CS > 1 ? static_cast<int>(cg::this_cluster().block_rank()) : 0;
    const int b = blockIdx.x / CS;
    double* A = a + b * stride;
    // one reduction round per reflector (double-buffered by parity): per-warp column sums,
    // the pivot row, and with CS > 1 every CTA's column sums and rank 0's pivot row pushed to
    // all CTAs of the cluster
    __shared__ double part[2][NW][32], prow[2][32], tws[NW][32];
    __shared__ double dots[2][CS][32], crow[2][32];
    __shared__ double Ts[NB * NB], gv[NB];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int rows = m - j0;
    int row[RR];
#pragma unroll
    for (int q = 0; q < RR; ++q) row[q] = rank * R + wid * 32 * RR + 32 * q + lane;
    double x[RR][NB];
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
        for (int q = 0; q < RR; ++q)
            x[q][j] = (row[q] < rows && j < w) ? A[(j0 + row[q]) + static_cast<long long>(j0 + j) * ld] : 0.0;
    for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) Ts[e] = 0.0;
    const int kmax = min(w, rows);
    // The reflector loop is unrolled UB at a time and the register columns are rotated by UB
    // after every group, so the pivot column always sits at a static position kk < UB: column
    // indices stay compile-time without unrolling all 32 reflectors (whose code overflowed the
    // instruction cache: 44 % of the stall samples were instruction fetches) and without
    // select chains.  Position p holds panel column (p + k0) mod 32; lanes map the same way.
#pragma unroll 1
    for (int k0 = 0; k0 < NB; k0 += UB) {
#pragma unroll
        for (int kk = 0; kk < UB; ++kk) {
            const int k = k0 + kk;
            if (k < kmax) {
            const int par = kk & 1;
            double xk[RR];
#pragma unroll
            for (int q = 0; q < RR; ++q) xk[q] = x[q][kk];
            // p[j] = sum over this thread's rows below the pivot row of x_k x_j for every column
            // (j = k: the tail norm), then a transpose reduction: lane j ends with column j's
            // warp total.  The first butterfly level is folded into the products so that only
            // 16 partials are live at a time.  With v = tail / (c0 - beta), v^T x_j is
            // x_j(k) + (tail^T x_j) / (c0 - beta): the norm and the dot products share one round.
            double p[16];
            const bool up16 = lane & 16;
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                double lo = 0.0, hi = 0.0;
#pragma unroll
                for (int q = 0; q < RR; ++q) {
                    const double t = row[q] > k ? xk[q] : 0.0;
                    lo = fma(t, x[q][i], lo);
                    hi = fma(t, x[q][i + 16], hi);
                }
                const double send = up16 ? lo : hi;
                const double keep = up16 ? hi : lo;
                p[i] = keep + __shfl_xor_sync(0xffffffffu, send, 16);
            }
#pragma unroll
            for (int o = 8, cnt = 8; o >= 1; o >>= 1, cnt >>= 1) {
                const bool up = lane & o;
#pragma unroll
                for (int i = 0; i < cnt; ++i) {
                    const double send = up ? p[i] : p[i + cnt];
                    const double keep = up ? p[i + cnt] : p[i];
                    p[i] = keep + __shfl_xor_sync(0xffffffffu, send, o);
                }
            }
            part[par][wid][lane] = p[0];
#pragma unroll
            for (int q = 0; q < RR; ++q)
                if (row[q] == k) {  // the pivot row (one thread of rank 0)
#pragma unroll
                    for (int j = 0; j < NB; ++j) prow[par][j] = x[q][j];
                }
            __syncthreads();
            double wl = 0.0, pr = 0.0;
            if constexpr (CS == 1) {
#pragma unroll
                for (int g = 0; g < NW; ++g) wl += part[par][g][lane];
                pr = prow[par][lane];
            } else {
                if (wid < CS) {  // warp q pushes this CTA's column sums (rank 0: and the pivot row) to ranks q, q + NW, ...
                    double s2 = 0.0;
#pragma unroll
                    for (int g = 0; g < NW; ++g) s2 += part[par][g][lane];
                    for (int r = wid; r < CS; r += NW) {
                        cg::this_cluster().map_shared_rank(&dots[par][rank][0], r)[lane] = s2;
                        if (rank == 0) cg::this_cluster().map_shared_rank(&crow[par][0], r)[lane] = prow[par][lane];
                    }
                }
                cg::this_cluster().sync();
#pragma unroll
                for (int r = 0; r < CS; ++r) wl += dots[par][r][lane];
                pr = crow[par][lane];
            }
            const double tail2 = __shfl_sync(0xffffffffu, wl, kk), c0 = __shfl_sync(0xffffffffu, pr, kk);
            double t = 0.0, den = 0.0, beta = c0;
            if (!(tail2 <= DBL_MIN)) {
                beta = sqrt(c0 * c0 + tail2);
                if (hh_beta_negative(c0, tail2)) beta = -beta;
                den = c0 - beta;
                t = (beta - c0) / beta;
            }
            const double rden = (t == 0.0) ? 0.0 : 1.0 / den;
            double v[RR];
#pragma unroll
            for (int q = 0; q < RR; ++q) {
                const double nv = row[q] > k ? xk[q] * rden : (row[q] == k ? beta : xk[q]);
                x[q][kk] = nv;
                v[q] = row[q] > k ? nv : (row[q] == k ? 1.0 : 0.0);
            }
            if (rank == 0 && threadIdx.x == 0) tau_all[static_cast<long long>(b) * tau_stride + j0 + k] = t;
            const double vx = fma(wl, rden, pr);  // lane p: v^T x of the column at position p
            const int oc = (lane + k0) & (NB - 1);  // that column
            // -tau v^T x_j to every lane through the warp's own shared-memory row (broadcast
            // loads); zero for the columns already factored (rotated to the high positions)
            tws[wid][lane] = (t != 0.0 && oc > k) ? -t * vx : 0.0;
            __syncwarp();
#pragma unroll
            for (int pp = kk + 1; pp < NB; ++pp) {
                const double tw = tws[wid][pp];
#pragma unroll
                for (int q = 0; q < RR; ++q) x[q][pp] = fma(tw, v[q], x[q][pp]);
            }
            __syncwarp();
            if (rank == 0 && wid == 0) {  // V^T v_k and tau_k for T, built after the loop
                if (oc < k) Ts[oc + k * NB] = t != 0.0 ? vx : 0.0;
                if (lane == 0) gv[k] = t;
            }
            }
        }
        // rotate the columns by UB positions
#pragma unroll
        for (int q = 0; q < RR; ++q) {
            double tmp[UB];
#pragma unroll
            for (int i = 0; i < UB; ++i) tmp[i] = x[q][i];
#pragma unroll
            for (int pp = 0; pp + UB < NB; ++pp) x[q][pp] = x[q][pp + UB];
#pragma unroll
            for (int i = 0; i < UB; ++i) x[q][NB - UB + i] = tmp[i];
        }
    }
    if constexpr (CS > 1) cg::this_cluster().sync();  // no remote store may target an exited CTA
    // store addresses formed here (an opaque copy of ld keeps the compiler from
    // hoisting 32 column addresses across the reflector loop into registers)
    long long ldo;
    asm volatile("mov.b64 %0, %1;" : "=l"(ldo) : "l"(static_cast<long long>(ld)));
    double* base = A + j0 + ldo * j0;
#pragma unroll
    for (int j = 0; j < NB; ++j)
#pragma unroll
        for (int q = 0; q < RR; ++q)
            if (row[q] < rows && j < w) base[row[q] + ldo * j] = x[q][j];
    // compact-WY T from the recorded V^T v_k (strict upper part of Ts) and tau
    // (accumulate_wy, dense_kernels.cpp:41-53): T(0:k, k) = -tau_k T(0:k, 0:k) (V^T v_k),
    // T(k, k) = tau_k; one warp, off the per-reflector critical path
    // Lane i keeps row i of T in registers (fully unrolled: the recorded V^T v_k are independent
    // broadcast loads, the recurrence itself is ~500 FMAs in four chains per step) - this tail
    // runs while every other warp of the CTA (and cluster) has finished, so it is serial time.
    if (rank == 0 && wid == 0) {
        __syncwarp();
        double trow[NB];
#pragma unroll
        for (int k = 0; k < NB; ++k) {
            const double tk = k < kmax ? gv[k] : 0.0;
            double acc[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
            for (int l = 0; l < k; ++l) acc[l & 3] = fma(trow[l], Ts[l + k * NB], acc[l & 3]);  // trow[l] = 0 for l < lane
            trow[k] = lane < k ? -tk * ((acc[0] + acc[1]) + (acc[2] + acc[3])) : (lane == k ? tk : 0.0);
        }
        __syncwarp();
#pragma unroll
        for (int k = 0; k < NB; ++k)
            if (lane <= k) Ts[lane + k * NB] = trow[k];
    }
    __syncthreads();
    if (rank == 0) {
        double* T = T_all + static_cast<long long>(b) * NB * NB;
        for (int e = threadIdx.x; e < NB * NB; e += blockDim.x) T[e] = Ts[e];
    }
}

template <int NW, int RR>
__global__ void __launch_bounds__(32 * NW, NW * RR <= 8 ? 2 : 1) k_panel_row(double* a, int ld, long long stride,
                                                                           int m, int j0, int w, double* tau_all,
                                                                           int tau_stride, double* T_all) {
    panel_row_body<NW, RR, 1, kPanelUB>(a, ld, stride, m, j0, w, tau_all, tau_stride, T_all);
}

template <int NW, int RR>
__global__ void __cluster_dims__(kCS, 1, 1) __launch_bounds__(32 * NW, NW * RR <= 8 ? 2 : 1)
    k_panel_rowc(double* a, int ld, long long stride, int m, int j0, int w, double* tau_all, int tau_stride,
                 double* T_all) {
    panel_row_body<NW, RR, kCS, kPanelUB>(a, ld, stride, m, j0, w, tau_all, tau_stride, T_all);
}

// register-resident panel launch; false when the panel is too tall
bool launch_panel_reg(int nbatch, int m, int ld, long long stride, double* d_a, int j0, int w, double* d_tau, int n,
                      double* d_T, cudaStream_t st) {
    const int rows = m - j0;
    const bool cl = rows > 512;
    const int per = cl ? (rows + kCS - 1) / kCS : rows;  // rows per CTA
    if (per > 512) return false;
    const int g = cl ? nbatch * kCS : nbatch;
#define SPQR_PANEL(NW_, RR_)                                                                                    \
    (cl ? k_panel_rowc<NW_, RR_><<<g, 32 * NW_, 0, st>>>(d_a, ld, stride, m, j0, w, d_tau, n, d_T)                \
        : k_panel_row<NW_, RR_><<<g, 32 * NW_, 0, st>>>(d_a, ld, stride, m, j0, w, d_tau, n, d_T))
    if (per <= 64) SPQR_PANEL(2, 1);
    else if (per <= 128) SPQR_PANEL(4, 1);
    else if (per <= 256) SPQR_PANEL(8, 1);
    else SPQR_PANEL(8, 2);
#undef SPQR_PANEL
    return true;
}

// ---- two-level blocking for large fronts ------------------------------------
// The NB = 32 panels of an outer block of KO = 128 columns are factored and
// applied to the rest of that outer block (KB = 32); the outer block's 128
// reflectors are then applied to every trailing column at once (KB = 128),
// which lifts the trailing update from ~5 flop/B (below the FP64 ridge) to
// ~21 flop/B.  Each block-reflector application  C -= V T^T-free form
//   W = V^T C,  W2 = T^T W,  C -= V W2
// runs as three kernels so that rows and columns are both split across CTAs:
//   k_vtc  partial W over a row slice (deterministic per-slice partials),
//   k_tw   sum of the partials in fixed order, then T^T (DMMA),
//   k_cvw  C -= V W2 over (row tile, column tile).
// The outer T (128 x 128) is built from the Gram matrix V^T V (k_vtc on the
// panel's own columns) by accumulate_wy's recurrence (dense_kernels.cpp:41-53):
//   T(0:k, k) = -tau_k T(0:k, 0:k) V(:, 0:k)^T v_k,  T(k, k) = tau_k.
constexpr int KO = 128;   // outer block width
constexpr int TCG = 64;   // trailing columns per CTA
constexpr int CHG = 32;   // rows per staged chunk
constexpr int LDS_ = CHG + 4;

// V(i, j) of the block starting at panel row 0 / column J0 (i, j panel-relative):
// unit lower trapezoidal, columns >= kw are zero
__device__ __forceinline__ bool v_direct(int i, int j, int kw, double& val) {
    if (j >= kw || i < j) { val = 0.0; return true; }
    if (i == j) { val = 1.0; return true; }
    return false;
}

// partial W[s] = V(rows of slice s)^T C(rows of slice s, column tile t)
// gram = 1: C is V itself (columns 0..KB of the block), i.e. W = V^T V
template <int KB>
__global__ void __launch_bounds__(256) k_vtc(const double* __restrict__ a, int ld, long long stride, int m, int J0,
                                             int kw, int cbeg, int cend, int rs, int gram,
                                             double* __restrict__ wp, const double* __restrict__ T_all) {
    constexpr int PM = KB / 32, PN = TCG / 16;
    const int t = blockIdx.x, s = blockIdx.y, b = blockIdx.z;
    const int ntile = gram ? KB / TCG : gridDim.x, nsl = gridDim.y;  // Gram: one CTA per slice, KB / TCG tiles in the layout
    const double* A = a + b * stride;
    const int rows = m - J0;
    const int c0 = cbeg + t * TCG, nc = min(TCG, cend - c0);
    const int rlo = s * rs, rhi = min(rows, rlo + rs);
    extern __shared__ double dsm[];
    double* const sV0 = dsm;                     // two V chunks, KB * LDS_ each
    double* const sC0 = dsm + 2 * KB * LDS_;     // two C chunks, TCG * LDS_ each
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int mw = wid & 3, nw = wid >> 2;
    const int nchunk = rhi > rlo ? (rhi - rlo + CHG - 1) / CHG : 0;
    // 16-byte copies for chunks below the unit-triangular rows when row pairs are aligned
    const bool vec = ((ld & 1) == 0) && ((J0 & 1) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0);
    auto issue = [&](int c) {
        const int r0 = rlo + c * CHG, rc = min(CHG, rhi - r0);
        double* vb = sV0 + (c & 1) * (KB * LDS_);
        double* cb = sC0 + (c & 1) * (TCG * LDS_);
        if (vec && rc == CHG && r0 >= KB) {
            for (int e = threadIdx.x; e < CHG * KB / 2; e += 256) {
                const int i = 2 * (e % (CHG / 2)), j = e / (CHG / 2);
                if (j < kw)
                    cp_async16(vb + i + j * LDS_, A + (J0 + r0 + i) + static_cast<long long>(J0 + j) * ld);
                else
                    vb[i + j * LDS_] = vb[i + 1 + j * LDS_] = 0.0;
            }
            for (int e = threadIdx.x; e < (gram ? 0 : CHG * TCG / 2); e += 256) {  // Gram: B operand is the V chunk
                const int i = 2 * (e % (CHG / 2)), j = e / (CHG / 2);
                if (j < nc && (!gram || c0 - cbeg + j < kw))  // Gram: V's columns beyond kw are zero
                    cp_async16(cb + i + j * LDS_, A + (J0 + r0 + i) + static_cast<long long>(c0 + j) * ld);
                else
                    cb[i + j * LDS_] = cb[i + 1 + j * LDS_] = 0.0;
            }
            cp_commit();
            return;
        }
        for (int e = threadIdx.x; e < CHG * KB; e += 256) {
            const int i = e % CHG, j = e / CHG, r = r0 + i;
            double* dst = vb + i + j * LDS_;
            double v;
            if (i >= rc) *dst = 0.0;
            else if (v_direct(r, j, kw, v)) *dst = v;
            else cp_async8(dst, A + (J0 + r) + static_cast<long long>(J0 + j) * ld, true);
        }
        for (int e = threadIdx.x; e < (gram ? 0 : CHG * TCG); e += 256) {
            const int i = e % CHG, j = e / CHG, r = r0 + i;
            double* dst = cb + i + j * LDS_;
            double v;
            if (i >= rc || j >= nc) *dst = 0.0;
            else if (gram && v_direct(r, c0 - cbeg + j, kw, v)) *dst = v;
            else cp_async8(dst, A + (J0 + r) + static_cast<long long>(c0 + j) * ld, true);
        }
        cp_commit();
    };
    // Gram mode (KB = KO): k_tmerge reads only the six 32 x 32 blocks above the block diagonal
    // (G01, G23, GAB), so warps 0..5 take one each (two per scheduler at most) with both operands
    // from the V chunk; rbk / gcb = the block's row / column index
    int rbk = mw, gcb = 0;
    if (gram) {
        rbk = wid < 3 ? 0 : (wid < 5 ? 1 : 2);
        gcb = wid < 3 ? wid + 1 : (wid < 5 ? wid - 1 : 3);
    }
    double acc[PM][PN][2] = {};
    if (nchunk > 0) issue(0);
    for (int c = 0; c < nchunk; ++c) {
        if (c + 1 < nchunk) {
            issue(c + 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const double* sV = sV0 + (c & 1) * (KB * LDS_);
        const double* sC = gram ? sV + (gcb * PN * 8) * LDS_ : sC0 + (c & 1) * (TCG * LDS_) + (nw * PN * 8) * LDS_;
        if (!gram || wid < 6)
#pragma unroll
        for (int k0 = 0; k0 < CHG; k0 += 4) {
            double av[PM], bv[PN];
#pragma unroll
            for (int i = 0; i < PM; ++i) av[i] = sV[(k0 + t4) + ((rbk * PM + i) * 8 + g) * LDS_];
#pragma unroll
            for (int q = 0; q < PN; ++q) bv[q] = sC[(k0 + t4) + (q * 8 + g) * LDS_];
#pragma unroll
            for (int i = 0; i < PM; ++i)
#pragma unroll
                for (int q = 0; q < PN; ++q) dmma(acc[i][q][0], acc[i][q][1], av[i], bv[q]);
        }
        __syncthreads();
    }
    double* W = wp + ((static_cast<long long>(b) * nsl + s) * ntile + t) * (KB * TCG);
    if (T_all != nullptr) {  // one row slice: W2 = T^T W here (k_tw's work, no W round trip)
        constexpr int LDW = KB + 4;  // KB x TCG in the (free) staging buffers
        double* sW = dsm;
#pragma unroll
        for (int i = 0; i < PM; ++i)
#pragma unroll
            for (int q = 0; q < PN; ++q) {
                const int row = (mw * PM + i) * 8 + g, col = (nw * PN + q) * 8 + 2 * t4;
                sW[row + col * LDW] = acc[i][q][0];
                sW[row + (col + 1) * LDW] = acc[i][q][1];
            }
        __syncthreads();
        const double* T = T_all + static_cast<long long>(b) * KB * KB;
        double acc2[PM][PN][2] = {};
        const int kend = min((mw + 1) * PM * 8, (kw + 3) & ~3);  // T^T lower triangular
        for (int k0 = 0; k0 < kend; k0 += 4) {
            double av[PM], bv[PN];
#pragma unroll
            for (int i = 0; i < PM; ++i) av[i] = __ldg(T + (k0 + t4) + ((mw * PM + i) * 8 + g) * KB);
#pragma unroll
            for (int q = 0; q < PN; ++q) bv[q] = sW[(k0 + t4) + ((nw * PN + q) * 8 + g) * LDW];
#pragma unroll
            for (int i = 0; i < PM; ++i)
#pragma unroll
                for (int q = 0; q < PN; ++q) dmma(acc2[i][q][0], acc2[i][q][1], av[i], bv[q]);
        }
#pragma unroll
        for (int i = 0; i < PM; ++i)
#pragma unroll
            for (int q = 0; q < PN; ++q) acc[i][q][0] = acc2[i][q][0], acc[i][q][1] = acc2[i][q][1];
    }
    if (gram) {
        if (wid < 6)
#pragma unroll
            for (int i = 0; i < PM; ++i)
#pragma unroll
                for (int q = 0; q < PN; ++q) {
                    const int row = (rbk * PM + i) * 8 + g, colg = (gcb * PN + q) * 8 + 2 * t4;
                    double* Wt = W + static_cast<long long>(colg / TCG) * (KB * TCG);
                    Wt[row + (colg % TCG) * KB] = acc[i][q][0];
                    Wt[row + (colg % TCG + 1) * KB] = acc[i][q][1];
                }
        return;
    }
#pragma unroll
    for (int i = 0; i < PM; ++i)
#pragma unroll
        for (int q = 0; q < PN; ++q) {
            const int row = (mw * PM + i) * 8 + g, col = (nw * PN + q) * 8 + 2 * t4;
            W[row + col * KB] = acc[i][q][0];
            W[row + (col + 1) * KB] = acc[i][q][1];
        }
}

// W2 = T^T (sum_s W[s]) for column tile t; written over slice 0's partial
template <int KB>
__global__ void __launch_bounds__(256) k_tw(double* __restrict__ wp, int nsl, const double* __restrict__ T_all,
                                            int kw) {
    constexpr int PM = KB / 32, PN = TCG / 16, LDW = KB + 4;
    const int t = blockIdx.x, b = blockIdx.y, ntile = gridDim.x;
    extern __shared__ double sW[];  // KB x TCG, ld LDW
    const double* T = T_all + static_cast<long long>(b) * KB * KB;
    double* W0 = wp + (static_cast<long long>(b) * nsl * ntile + t) * (KB * TCG);
    for (int e = threadIdx.x; e < KB * TCG; e += 256) {
        double v = 0.0;
        for (int s = 0; s < nsl; ++s) v += W0[static_cast<long long>(s) * ntile * (KB * TCG) + e];
        sW[(e % KB) + (e / KB) * LDW] = v;
    }
    __syncthreads();
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int mw = wid & 3, nw = wid >> 2;
    double acc[PM][PN][2] = {};
    const int kend = min((mw + 1) * PM * 8, (kw + 3) & ~3);  // T^T lower triangular
    for (int k0 = 0; k0 < kend; k0 += 4) {
        double av[PM], bv[PN];
#pragma unroll
        for (int i = 0; i < PM; ++i) av[i] = __ldg(T + (k0 + t4) + ((mw * PM + i) * 8 + g) * KB);
#pragma unroll
        for (int q = 0; q < PN; ++q) bv[q] = sW[(k0 + t4) + ((nw * PN + q) * 8 + g) * LDW];
#pragma unroll
        for (int i = 0; i < PM; ++i)
#pragma unroll
            for (int q = 0; q < PN; ++q) dmma(acc[i][q][0], acc[i][q][1], av[i], bv[q]);
    }
#pragma unroll
    for (int i = 0; i < PM; ++i)
#pragma unroll
        for (int q = 0; q < PN; ++q) {
            const int row = (mw * PM + i) * 8 + g, col = (nw * PN + q) * 8 + 2 * t4;
            W0[row + col * KB] = acc[i][q][0];
            W0[row + (col + 1) * KB] = acc[i][q][1];
        }
}

// C(row tile, column tile) -= V W2
template <int KB>
__global__ void __launch_bounds__(256) k_cvw(double* __restrict__ a, int ld, long long stride, int m, int J0, int kw,
                                             int cbeg, int cend, int rt, const double* __restrict__ wp, int nsl) {
    constexpr int LDV = KB + 4, LDW = KB + 4;
    const int t = blockIdx.x, rtile = blockIdx.y, b = blockIdx.z, ntile = gridDim.x;
    double* A = a + b * stride;
    const int rows = m - J0;
    const int c0 = cbeg + t * TCG, nc = min(TCG, cend - c0);
    const int rlo = rtile * rt, rhi = min(rows, rlo + rt);
    if (rlo >= rhi) return;
    extern __shared__ double dsm[];
    double* sW = dsm;                                  // KB x TCG, ld LDW
    double* const sV0 = dsm + TCG * LDW;                  // two V chunks: (row, refl) at refl + row*LDV
    double* const sC0 = dsm + TCG * LDW + 2 * CHG * LDV;  // two C chunks, TCG * LDS_ each
    const double* W2 = wp + (static_cast<long long>(b) * nsl * ntile + t) * (KB * TCG);
    const int kwr = (kw + 3) & ~3;
    for (int e = threadIdx.x; e < KB * TCG; e += 256) cp_async8(sW + (e % KB) + (e / KB) * LDW, W2 + e, true);
    const int nchunk = (rhi - rlo + CHG - 1) / CHG;
    auto issue = [&](int c) {
        const int r0 = rlo + c * CHG, rc = min(CHG, rhi - r0);
        double* vb = sV0 + (c & 1) * (CHG * LDV);
        double* cb = sC0 + (c & 1) * (TCG * LDS_);
        for (int e = threadIdx.x; e < CHG * kwr; e += 256) {
            const int i = e % CHG, j = e / CHG, r = r0 + i;
            double* dst = vb + j + i * LDV;
            double v;
            if (i >= rc) *dst = 0.0;
            else if (v_direct(r, j, kw, v)) *dst = v;
            else cp_async8(dst, A + (J0 + r) + static_cast<long long>(J0 + j) * ld, true);
        }
        for (int e = threadIdx.x; e < CHG * TCG; e += 256) {
            const int i = e % CHG, j = e / CHG;
            const bool ok = i < rc && j < nc;
            cp_async8(cb + i + j * LDS_, ok ? A + (J0 + r0 + i) + static_cast<long long>(c0 + j) * ld : A, ok);
        }
        cp_commit();
    };
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int rw = wid & 1, cw = wid >> 1;  // warp: rows rw*16..+16, cols cw*16..+16 of the chunk
    issue(0);
    for (int c = 0; c < nchunk; ++c) {
        const int r0 = rlo + c * CHG, rc = min(CHG, rhi - r0);
        if (c + 1 < nchunk) {
            issue(c + 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const double* sV = sV0 + (c & 1) * (CHG * LDV);
        double* sC = sC0 + (c & 1) * (TCG * LDS_);
        double o[2][2][2] = {};
#pragma unroll 4
        for (int k0 = 0; k0 < kwr; k0 += 4) {
            double av[2], bv[2];
#pragma unroll
            for (int i = 0; i < 2; ++i) av[i] = sV[(k0 + t4) + ((rw * 2 + i) * 8 + g) * LDV];
#pragma unroll
            for (int q = 0; q < 2; ++q) bv[q] = sW[(k0 + t4) + ((cw * 2 + q) * 8 + g) * LDW];
#pragma unroll
            for (int i = 0; i < 2; ++i)
#pragma unroll
                for (int q = 0; q < 2; ++q) dmma(o[i][q][0], o[i][q][1], av[i], bv[q]);
        }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int q = 0; q < 2; ++q) {
                const int row = (rw * 2 + i) * 8 + g, col = (cw * 2 + q) * 8 + 2 * t4;
                sC[row + col * LDS_] -= o[i][q][0];
                sC[row + (col + 1) * LDS_] -= o[i][q][1];
            }
        __syncthreads();
        for (int e = threadIdx.x; e < CHG * TCG; e += 256) {
            const int i = e % CHG, j = e / CHG;
            if (i < rc && j < nc) A[(J0 + r0 + i) + static_cast<long long>(c0 + j) * ld] = sC[i + j * LDS_];
        }
        __syncthreads();
    }
}

// C(128-row tile, 64-column tile) -= V(tile rows, 0:kw) W2(0:kw, tile columns):
// a plain GEMM tile with K = kw <= KB.  Warps 4 (rows) x 2 (columns), warp tile
// 32 x 32 (4 x 4 DMMA m8n8k4 tiles: 8 fragment loads per 16 DMMA).  V and W2
// stream through two shared-memory stages of 32 reflectors (cp.async); C is
// read and written straight from/to global memory in the accumulator layout
// (each warp access covers 8 rows x 4 column pairs: whole 32-byte sectors).
constexpr int CM = 128;          // rows per CTA
constexpr int KC = 32;           // reflectors per stage
constexpr int LDM = CM + 4;      // V stage: (row, refl) at row + refl * LDM
constexpr int LDK = KC + 4;      // W2 stage: (refl, col) at refl + col * LDK
template <int KB>
__global__ void __launch_bounds__(256, 2) k_cvw2(double* __restrict__ a, int ld, long long stride, int m, int J0,
                                                 int kw, int cbeg, int cend, const double* __restrict__ wp, int nsl) {
    const int t = blockIdx.x, rtile = blockIdx.y, b = blockIdx.z, ntile = gridDim.x;
    double* A = a + b * stride;
    const int rows = m - J0;
    const int c0 = cbeg + t * TCG, nc = min(TCG, cend - c0);
    const int r0 = rtile * CM;
    const double* W2 = wp + (static_cast<long long>(b) * nsl * ntile + t) * (KB * TCG);
    extern __shared__ double dsm[];
    double* const sV0 = dsm;                  // two stages of CM x KC
    double* const sW0 = dsm + 2 * KC * LDM;   // two stages of KC x TCG
    const int nst = (kw + KC - 1) / KC;
    {  // pull this CTA's C tile into L2 while the stages run (read in the epilogue)
        const int e = threadIdx.x;  // 256 threads: column e / 4, 32-row quarter e % 4
        const int c = e >> 2, rq = (e & 3) * 32;
        if (c < nc && r0 + rq < rows) {
            const double* pc = A + (J0 + r0 + rq) + static_cast<long long>(c0 + c) * ld;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pc));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pc + 16));
        }
    }
    // 16-byte copies below the unit-triangular rows when row pairs are aligned (W2 always is)
    const bool vec = ((ld & 1) == 0) && ((J0 & 1) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
                     r0 >= KB && r0 + CM <= rows;
    auto issue = [&](int s) {
        double* vb = sV0 + (s & 1) * (KC * LDM);
        double* wb = sW0 + (s & 1) * (TCG * LDK);
        const int k0 = s * KC;
        if (vec) {
            for (int e = threadIdx.x; e < CM * KC / 2; e += 256) {
                const int i = 2 * (e % (CM / 2)), j = e / (CM / 2), jj = k0 + j;
                if (jj < kw)
                    cp_async16(vb + i + j * LDM, A + (J0 + r0 + i) + static_cast<long long>(J0 + jj) * ld);
                else
                    vb[i + j * LDM] = vb[i + 1 + j * LDM] = 0.0;
            }
        } else {
            for (int e = threadIdx.x; e < CM * KC; e += 256) {
                const int i = e % CM, j = e / CM, r = r0 + i, jj = k0 + j;
                double* dst = vb + i + j * LDM;
                double v;
                if (r >= rows) *dst = 0.0;
                else if (v_direct(r, jj, kw, v)) *dst = v;
                else cp_async8(dst, A + (J0 + r) + static_cast<long long>(J0 + jj) * ld, true);
            }
        }
        for (int e = threadIdx.x; e < KC * TCG / 2; e += 256) {
            const int j = 2 * (e % (KC / 2)), c = e / (KC / 2);
            cp_async16(wb + j + c * LDK, W2 + (k0 + j) + c * KB);
        }
        cp_commit();
    };
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int mw = wid & 3, nw = wid >> 2;
    double acc[4][4][2] = {};
    issue(0);
    for (int s = 0; s < nst; ++s) {
        if (s + 1 < nst) {
            issue(s + 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const double* sV = sV0 + (s & 1) * (KC * LDM);
        const double* sW = sW0 + (s & 1) * (TCG * LDK);
        const int kend = min(KC, ((kw - s * KC) + 3) & ~3);
#pragma unroll 4
        for (int k0 = 0; k0 < kend; k0 += 4) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = sV[(mw * 32 + i * 8 + g) + (k0 + t4) * LDM];
#pragma unroll
            for (int q = 0; q < 4; ++q) bv[q] = sW[(k0 + t4) + (nw * 32 + q * 8 + g) * LDK];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) dmma(acc[i][q][0], acc[i][q][1], av[i], bv[q]);
        }
        __syncthreads();
    }
    // epilogue: C -= acc, in the accumulator layout (one row tile of 8 at a time)
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = r0 + mw * 32 + i * 8 + g;
        double* crow = A + (J0 + r) + static_cast<long long>(c0) * ld;
        double cv[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = nw * 32 + q * 8 + 2 * t4 + h;
                cv[q][h] = (r < rows && c < nc) ? crow[static_cast<long long>(c) * ld] : 0.0;
            }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = nw * 32 + q * 8 + 2 * t4 + h;
                if (r < rows && c < nc) crow[static_cast<long long>(c) * ld] = cv[q][h] - acc[i][q][h];
            }
    }
}
constexpr size_t kCvw2Smem = sizeof(double) * (2 * KC * LDM + 2 * TCG * LDK);

// k_cvw2 with 64-row tiles, 4-warp CTAs and KCT-reflector stages: four CTAs per SM (38 KB of
// shared memory and 16 K registers each at KCT = 16) instead of two.  Measured on C5 4096x1024:
// 39.2 ms against 40.3 ms with k_cvw2, although a tile moves 18 % more bytes through L2 per flop
// — the barrier-synchronised phases of a CTA (stage wait, DMMA stage, C read-modify-write) leave
// the FP64 tensor pipe idle unless enough INDEPENDENT CTAs share the SM; the opposite change
// (one 16-warp CTA per SM, W2 resident, 40 % fewer bytes per flop) ran 44.1 ms (DESIGN 6).
template <int KB, int KCT>
__global__ void __launch_bounds__(128, 4) k_cvw4(double* __restrict__ a, int ld, long long stride, int m, int J0,
                                                 int kw, int cbeg, int cend, const double* __restrict__ wp, int nsl) {
    constexpr int CMT = 64, LDM4 = CMT + 4, LDK4 = KCT + 4, NT = 128;
    const int t = blockIdx.x, rtile = blockIdx.y, b = blockIdx.z, ntile = gridDim.x;
    double* A = a + b * stride;
    const int rows = m - J0;
    const int c0 = cbeg + t * TCG, nc = min(TCG, cend - c0);
    const int r0 = rtile * CMT;
    const double* W2 = wp + (static_cast<long long>(b) * nsl * ntile + t) * (KB * TCG);
    extern __shared__ double dsm[];
    double* const sV0 = dsm;                    // two stages of CMT x KCT
    double* const sW0 = dsm + 2 * KCT * LDM4;   // two stages of KCT x TCG
    const int nst = (kw + KCT - 1) / KCT;
    {
        const int e = threadIdx.x;  // 128 threads: column e / 2, 32-row half e % 2
        const int c = e >> 1, rq = (e & 1) * 32;
        if (c < nc && r0 + rq < rows) {
            const double* pc = A + (J0 + r0 + rq) + static_cast<long long>(c0 + c) * ld;
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pc));
            asm volatile("prefetch.global.L2 [%0];" ::"l"(pc + 16));
        }
    }
    const bool vec = ((ld & 1) == 0) && ((J0 & 1) == 0) && ((reinterpret_cast<uintptr_t>(A) & 15) == 0) &&
                     r0 >= KB && r0 + CMT <= rows;
    auto issue = [&](int s) {
        double* vb = sV0 + (s & 1) * (KCT * LDM4);
        double* wb = sW0 + (s & 1) * (TCG * LDK4);
        const int k0 = s * KCT;
        if (vec) {
            for (int e = threadIdx.x; e < CMT * KCT / 2; e += NT) {
                const int i = 2 * (e % (CMT / 2)), j = e / (CMT / 2), jj = k0 + j;
                if (jj < kw)
                    cp_async16(vb + i + j * LDM4, A + (J0 + r0 + i) + static_cast<long long>(J0 + jj) * ld);
                else
                    vb[i + j * LDM4] = vb[i + 1 + j * LDM4] = 0.0;
            }
        } else {
            for (int e = threadIdx.x; e < CMT * KCT; e += NT) {
                const int i = e % CMT, j = e / CMT, r = r0 + i, jj = k0 + j;
                double* dst = vb + i + j * LDM4;
                double v;
                if (r >= rows) *dst = 0.0;
                else if (v_direct(r, jj, kw, v)) *dst = v;
                else cp_async8(dst, A + (J0 + r) + static_cast<long long>(J0 + jj) * ld, true);
            }
        }
        for (int e = threadIdx.x; e < KCT * TCG / 2; e += NT) {
            const int j = 2 * (e % (KCT / 2)), c = e / (KCT / 2);
            if (k0 + j < KB)
                cp_async16(wb + j + c * LDK4, W2 + (k0 + j) + c * KB);
            else
                wb[j + c * LDK4] = wb[j + 1 + c * LDK4] = 0.0;
        }
        cp_commit();
    };
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int g = lane >> 2, t4 = lane & 3;
    const int mw = wid & 1, nw = wid >> 1;
    double acc[4][4][2] = {};
    issue(0);
    for (int s = 0; s < nst; ++s) {
        if (s + 1 < nst) {
            issue(s + 1);
            cp_wait<1>();
        } else {
            cp_wait<0>();
        }
        __syncthreads();
        const double* sV = sV0 + (s & 1) * (KCT * LDM4);
        const double* sW = sW0 + (s & 1) * (TCG * LDK4);
        const int kend = min(KCT, ((kw - s * KCT) + 3) & ~3);
#pragma unroll 4
        for (int k0 = 0; k0 < kend; k0 += 4) {
            double av[4], bv[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) av[i] = sV[(mw * 32 + i * 8 + g) + (k0 + t4) * LDM4];
#pragma unroll
            for (int q = 0; q < 4; ++q) bv[q] = sW[(k0 + t4) + (nw * 32 + q * 8 + g) * LDK4];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int q = 0; q < 4; ++q) dmma(acc[i][q][0], acc[i][q][1], av[i], bv[q]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int r = r0 + mw * 32 + i * 8 + g;
        double* crow = A + (J0 + r) + static_cast<long long>(c0) * ld;
        double cv[4][2];
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = nw * 32 + q * 8 + 2 * t4 + h;
                cv[q][h] = (r < rows && c < nc) ? crow[static_cast<long long>(c) * ld] : 0.0;
            }
#pragma unroll
        for (int q = 0; q < 4; ++q)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
                const int c = nw * 32 + q * 8 + 2 * t4 + h;
                if (r < rows && c < nc) crow[static_cast<long long>(c) * ld] = cv[q][h] - acc[i][q][h];
            }
    }
}
template <int KCT>
constexpr size_t cvw4_smem() {
    return sizeof(double) * (2 * KCT * (64 + 4) + 2 * TCG * (KCT + 4));
}
template <int KB, int KCT>
void launch_cvw4(dim3 grid, cudaStream_t st, double* d_a, int ld, long long stride, int m, int J0, int kw, int cbeg,
                 int cend, const double* wp, int nsl) {
    static SmemCfg cfg;
    smem_optin(reinterpret_cast<const void*>(k_cvw4<KB, KCT>), cvw4_smem<KCT>(), cfg);
    k_cvw4<KB, KCT><<<grid, 128, cvw4_smem<KCT>(), st>>>(d_a, ld, stride, m, J0, kw, cbeg, cend, wp, nsl);
}

// Outer T (KO x KO) of an outer block whose four NB-column panels have compact-WY
// factors T_q (written by the panel kernels), composed pairwise:
//   H_A H_B = I - [V_A V_B] [T_A, -T_A (V_A^T V_B) T_B; 0, T_B] [V_A V_B]^T
// first (0,1) and (2,3), then (01, 23).  V_A^T V_B are blocks of the Gram matrix
// V^T V, summed over the row-slice partials of k_vtc in fixed order.  Same
// matrix as accumulate_wy's column recurrence (dense_kernels.cpp:41-53), in
// blocked order.
__global__ void __launch_bounds__(256) k_tmerge(const double* __restrict__ wp, int nsl,
                                                const double* __restrict__ Tin, long long tin_slot, int nq,
                                                double* __restrict__ T_all) {
    constexpr int LDT = KO + 1, ntile = KO / TCG;
    const int b = blockIdx.x;
    extern __shared__ double sm[];
    double* sT = sm;                    // KO x KO, ld LDT
    double* G01 = sT + KO * LDT;        // 32 x 32: G(0:32, 32:64)
    double* G23 = G01 + 32 * 32;        // 32 x 32: G(64:96, 96:128)
    double* GAB = G23 + 32 * 32;        // 64 x 64: G(0:64, 64:128)
    double* X = GAB + 64 * 64;          // 64 x 64 scratch
    const double* G0 = wp + static_cast<long long>(b) * nsl * ntile * (KO * TCG);
    auto gram = [&](int i, int j) {     // G(i, j), partials in fixed order
        double v = 0.0;
        for (int s = 0; s < nsl; ++s) v += G0[(static_cast<long long>(s) * ntile + j / TCG) * (KO * TCG) + i + (j % TCG) * KO];
        return v;
    };
    for (int e = threadIdx.x; e < KO * KO; e += 256) {
        const int i = e % KO, j = e / KO, q = i / NB;
        double v = 0.0;
        if (q == j / NB && q < nq) v = Tin[q * tin_slot + static_cast<long long>(b) * NB * NB + (i % NB) + (j % NB) * NB];
        sT[i + j * LDT] = v;
    }
    for (int e = threadIdx.x; e < 32 * 32; e += 256) {
        const int i = e % 32, j = e / 32;
        G01[e] = gram(i, 32 + j);
        G23[e] = gram(64 + i, 96 + j);
    }
    for (int e = threadIdx.x; e < 64 * 64; e += 256) GAB[e] = gram(e % 64, 64 + e / 64);
    __syncthreads();
    // C = alpha A B (n x n, column-major, shared memory), 4 x 4 register blocks per thread
    auto mm4 = [](double* C, int ldc, const double* A, int lda, const double* B, int ldb, int n, double alpha, int tid,
                  int nthr) {
        const int nb = n / 4;
        for (int blk = tid; blk < nb * nb; blk += nthr) {
            const int i0 = 4 * (blk % nb), j0 = 4 * (blk / nb);
            double acc[4][4] = {};
            for (int l = 0; l < n; ++l) {
                double av[4], bv[4];
#pragma unroll
                for (int r = 0; r < 4; ++r) av[r] = A[(i0 + r) + l * lda];
#pragma unroll
                for (int c = 0; c < 4; ++c) bv[c] = B[l + (j0 + c) * ldb];
#pragma unroll
                for (int r = 0; r < 4; ++r)
#pragma unroll
                    for (int c = 0; c < 4; ++c) acc[r][c] = fma(av[r], bv[c], acc[r][c]);
            }
#pragma unroll
            for (int r = 0; r < 4; ++r)
#pragma unroll
                for (int c = 0; c < 4; ++c) C[(i0 + r) + (j0 + c) * ldc] = alpha * acc[r][c];
        }
    };
    // level 1: T(o, o+32) = -T_o G T_{o+32} for o = 0 (threads 0..127) and o = 64 (128..255)
    {
        const int h = threadIdx.x >> 7, tl = threadIdx.x & 127, o = 64 * h;
        const double* G = h ? G23 : G01;
        double* Xh = X + h * 1024;
        mm4(Xh, 32, G, 32, sT + (o + 32) + (o + 32) * LDT, LDT, 32, 1.0, tl, 128);
        __syncthreads();
        mm4(sT + o + (o + 32) * LDT, LDT, sT + o + o * LDT, LDT, Xh, 32, 32, -1.0, tl, 128);
    }
    __syncthreads();
    // level 2: T(0:64, 64:128) = -T_A (G_AB T_B)
    mm4(X, 64, GAB, 64, sT + 64 + 64 * LDT, LDT, 64, 1.0, threadIdx.x, 256);
    __syncthreads();
    mm4(sT + 64 * LDT, LDT, sT, LDT, X, 64, 64, -1.0, threadIdx.x, 256);
    __syncthreads();
    double* T = T_all + static_cast<long long>(b) * KO * KO;
    for (int e = threadIdx.x; e < KO * KO; e += 256) T[e] = sT[(e % KO) + (e / KO) * LDT];
}
constexpr size_t kTmergeSmem = sizeof(double) * (KO * (KO + 1) + 2 * 32 * 32 + 2 * 64 * 64);

size_t vtc_smem(int kb) { return sizeof(double) * (2 * kb * LDS_ + 2 * TCG * LDS_); }
size_t cvw_smem(int kb) { return sizeof(double) * (TCG * (kb + 4) + 2 * CHG * (kb + 4) + 2 * TCG * LDS_); }

// workspace for the partial W tiles and the outer T (grow-only)
struct BigWs {
    double* p = nullptr;
    size_t cap = 0;
    double* get(size_t n) {
        if (n > cap) {
            if (p) cudaFree(p);  // synchronises: no kernel still uses the old buffer
            p = nullptr;
            cap = 0;
            const cudaError_t e = cudaMalloc(&p, sizeof(double) * n);
            if (e != cudaSuccess) {
                p = nullptr;
                throw CudaError(std::string("blocked QR workspace: ") + cudaGetErrorString(e));
            }
            cap = n;
        }
        return p;
    }
};
// Per-device state of the blocked path: workspaces ([0] trailing updates on the caller's
// stream, [1] panel phase on the look-ahead side stream), the side stream and its events.
// Calls on one device are serialised on the host (mutex) and on the GPU (each call's stream
// waits for the previous call's completion event), so concurrent handles never share a
// workspace in flight; every device gets its own buffers and stream.
struct MbqrDev {
    std::mutex mu;
    BigWs ws_w[2], ws_t[2];
    cudaStream_t side = nullptr;
    cudaEvent_t ev_a = nullptr, ev_b = nullptr, done = nullptr;
    bool used = false;
};
MbqrDev& mbqr_dev() {
    static MbqrDev s[kMaxDevices];
    int d = 0;
    cudaGetDevice(&d);
    return s[(d >= 0 && d < kMaxDevices) ? d : 0];
}

// block reflector (KB columns at J0, kw valid, T in T_all with ld KB) applied
// to columns [cbeg, cend) of every problem; gram != 0 computes V^T V instead
template <int KB>
void apply_block(BigWs& ws, int nbatch, int m, int ld, long long stride, double* d_a, int J0, int kw, int cbeg,
                 int cend, const double* T_all, cudaStream_t st, int* nsl_out = nullptr, int gram = 0) {
    const int rows = m - J0;
    const int ntile = (cend - cbeg + TCG - 1) / TCG;
    if (ntile <= 0 || rows <= 0) return;
    const int sms = sm_count();
    // row slices: minimise (waves of resident CTAs) x (chunks per slice), two
    // k_vtc CTAs per SM; fewer slices on ties (less partial-sum traffic)
    const long long resident = 2LL * sms;
    const int nchunks = (rows + CHG - 1) / CHG;
    int nsl = 1;
    long long best = -1;
    for (int cand = 1; cand <= std::min(64, std::max(1, nchunks / 2)); ++cand) {
        const int per = (nchunks + cand - 1) / cand;
        const long long waves = (static_cast<long long>(gram ? 1 : ntile) * cand * nbatch + resident - 1) / resident;
        const long long cost = waves * (per + 2);  // +2: fixed cost per CTA (prologue, partial write)
        if (best < 0 || cost < best) {
            best = cost;
            nsl = cand;
        }
    }
    const int rs = ((nchunks + nsl - 1) / nsl) * CHG;
    nsl = (rows + rs - 1) / rs;
    double* wp = ws.get(static_cast<size_t>(nbatch) * nsl * ntile * KB * TCG);
    {
        static SmemCfg cfg;
        smem_optin(reinterpret_cast<const void*>(k_vtc<KB>), vtc_smem(KB), cfg);
        k_vtc<KB><<<dim3(gram ? 1 : ntile, nsl, nbatch), 256, vtc_smem(KB), st>>>(d_a, ld, stride, m, J0, kw, cbeg, cend, rs, gram,
                                                                         wp, (nsl == 1 && !gram) ? T_all : nullptr);
    }
    if (gram) {
        *nsl_out = nsl;
        return;
    }
    if (nsl > 1) {  // (one slice: fused into k_vtc)
        static SmemCfg cfg;
        const size_t sm = sizeof(double) * KB * 0 + sizeof(double) * (KB + 4) * TCG;
        smem_optin(reinterpret_cast<const void*>(k_tw<KB>), sm, cfg);
        k_tw<KB><<<dim3(ntile, nbatch), 256, sm, st>>>(wp, nsl, T_all, kw);
    }
    // k_cvw4 (64-row tiles, 4-warp CTAs) for the KO-wide block reflectors and the NB-wide inner
    // updates; SPQR_CVW4=0 keeps k_cvw2, =32 takes 32-reflector stages, SPQR_CVW4_INNER=0 leaves the
    // inner updates on k_cvw2 (comparisons)
    static const int cvw4 = std::getenv("SPQR_CVW4") ? std::atoi(std::getenv("SPQR_CVW4")) : 16;
    static const bool cvw4_inner = !std::getenv("SPQR_CVW4_INNER") || std::atoi(std::getenv("SPQR_CVW4_INNER")) != 0;
    if (cvw4 && (KB > NB || cvw4_inner)) {
        const dim3 grid(ntile, (rows + 63) / 64, nbatch);
        if (cvw4 == 16)
            launch_cvw4<KB, 16>(grid, st, d_a, ld, stride, m, J0, kw, cbeg, cend, wp, nsl);
        else
            launch_cvw4<KB, 32>(grid, st, d_a, ld, stride, m, J0, kw, cbeg, cend, wp, nsl);
    } else if (!std::getenv("SPQR_CVW1")) {
        static SmemCfg cfg;
        smem_optin(reinterpret_cast<const void*>(k_cvw2<KB>), kCvw2Smem, cfg);
        k_cvw2<KB><<<dim3(ntile, (rows + CM - 1) / CM, nbatch), 256, kCvw2Smem, st>>>(d_a, ld, stride, m, J0, kw, cbeg,
                                                                                   cend, wp, nsl);
    } else {
        const int rt = rows <= 512 ? ((rows + 1) / 2 + CHG - 1) / CHG * CHG : 256;
        const int nrt = (rows + rt - 1) / rt;
        static SmemCfg cfg;
        smem_optin(reinterpret_cast<const void*>(k_cvw<KB>), cvw_smem(KB), cfg);
        k_cvw<KB><<<dim3(ntile, nrt, nbatch), 256, cvw_smem(KB), st>>>(d_a, ld, stride, m, J0, kw, cbeg, cend,
                                                                         std::max(rt, CHG), wp, nsl);
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
    MbqrDev& D = mbqr_dev();
    std::lock_guard<std::mutex> lk(D.mu);
    if (!D.done) CK(cudaEventCreateWithFlags(&D.done, cudaEventDisableTiming));
    if (D.used) CK(cudaStreamWaitEvent(st, D.done, 0));  // previous call (any stream) has finished
    BigWs* g_ws_w = D.ws_w;
    BigWs* g_ws_t = D.ws_t;
    const int ldA = ld_in > 0 ? ld_in : m;
    const long long stride = static_cast<long long>(ldA) * ntot;
    const size_t smem_cap = 160 * 1024;
    // panel j0..j0+w: V, tau, and the panel's T (NB x NB per problem) in d_T
    auto panel = [&](int j0, int w, double* d_T, cudaStream_t st) {
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
            static SmemCfg cfg;
            smem_optin(reinterpret_cast<const void*>(k_panel_cluster), csmem, cfg);
            k_panel_cluster<<<nbatch * kCS, 256, csmem, st>>>(d_a, ldA, stride, m, j0, w, d_tau, n, d_T, Rc);
        } else if (rows <= 512) {
            static SmemCfg cfg;
            smem_optin(reinterpret_cast<const void*>(k_panel2<8>), smem, cfg);
            k_panel2<8><<<nbatch, 256, smem, st>>>(d_a, ldA, stride, m, j0, w, d_tau, n, d_T, smem_rows);
        } else {
            static SmemCfg cfg;
            smem_optin(reinterpret_cast<const void*>(k_panel2<16>), smem, cfg);
            k_panel2<16><<<nbatch, 512, smem, st>>>(d_a, ldA, stride, m, j0, w, d_tau, n, d_T, smem_rows);
        }
    };
    // one level (SPQR_QR_L1=1, kept for comparison): every NB panel updates all
    // trailing columns in one CTA per column tile (k_wy)
    const bool one_level = std::getenv("SPQR_QR_L1") != nullptr;
    if (one_level || n <= NB) {
        for (int j0 = 0; j0 < n; j0 += NB) {
            const int w = std::min(NB, n - j0);
            panel(j0, w, d_T, st);
            const int trail = ntot - (j0 + w);
            if (trail > 0) {
                dim3 grid((trail + TC2 - 1) / TC2, nbatch);
                const size_t vsz = std::max(NB * LDV, CH * LDVT);
                const size_t wsm = sizeof(double) * (2 * vsz + 2 * TC2 * LDC + TC2 * LDW + NB * LDW);
                static SmemCfg cfg;
                smem_optin(reinterpret_cast<const void*>(k_wy<16>), wsm, cfg);
                k_wy<16><<<grid, 512, wsm, st>>>(d_a, ldA, stride, m, ntot, j0, w, d_T);
            }
        }
    } else {
        // two levels: NB panels inside KO-wide outer blocks, one KO-wide block
        // reflector per outer block for the trailing columns.  Look-ahead: once
        // block J has updated block J+1's columns, block J+1's panel phase runs on
        // a side stream (high priority) while block J updates the columns beyond.
        const long long slot = static_cast<long long>(nbatch) * NB * NB;
        const size_t tsz = static_cast<size_t>(nbatch) * (KO * KO + (KO / NB) * NB * NB);
        double* Tb[2] = {g_ws_t[0].get(tsz), g_ws_t[1].get(tsz)};
        const bool reg_panel = !std::getenv("SPQR_SMEM_PANEL");
        const bool lookahead = !std::getenv("SPQR_NO_LOOKAHEAD");
        if (lookahead && !D.side) {
            int lo = 0, hi = 0;
            CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
            CK(cudaStreamCreateWithPriority(&D.side, cudaStreamNonBlocking, hi));
            CK(cudaEventCreateWithFlags(&D.ev_a, cudaEventDisableTiming));
            CK(cudaEventCreateWithFlags(&D.ev_b, cudaEventDisableTiming));
        }
        cudaStream_t side = D.side;
        cudaEvent_t ev_a = D.ev_a, ev_b = D.ev_b;
        // panels + inner updates of block J0, its Gram matrix and merged T into Tout
        auto panel_phase = [&](int J0, double* Tout, cudaStream_t s) {
            const int kw2 = std::min(KO, n - J0);
            double* T_in = Tout + static_cast<size_t>(nbatch) * KO * KO;
            for (int j0 = J0; j0 < J0 + kw2; j0 += NB) {
                const int w = std::min(NB, J0 + kw2 - j0);
                double* Tq = T_in + ((j0 - J0) / NB) * slot;
                if (!(reg_panel && launch_panel_reg(nbatch, m, ldA, stride, d_a, j0, w, d_tau, n, Tq, s)))
                    panel(j0, w, Tq, s);
                if (j0 + w < J0 + kw2)
                    apply_block<NB>(g_ws_w[1], nbatch, m, ldA, stride, d_a, j0, w, j0 + w, J0 + kw2, Tq, s);
            }
            if (kw2 <= NB || J0 + kw2 >= ntot) return;
            int nsl = 1;
            apply_block<KO>(g_ws_w[1], nbatch, m, ldA, stride, d_a, J0, kw2, J0, J0 + KO, nullptr, s, &nsl, 1);
            static SmemCfg cfg;
            smem_optin(reinterpret_cast<const void*>(k_tmerge), kTmergeSmem, cfg);
            k_tmerge<<<nbatch, 256, kTmergeSmem, s>>>(g_ws_w[1].p, nsl, T_in, slot, (kw2 + NB - 1) / NB, Tout);
        };
        // block J0's reflectors applied to columns [c0, c1)
        auto update = [&](int J0, const double* Tout, int c0, int c1) {
            const int kw2 = std::min(KO, n - J0);
            if (c1 <= c0) return;
            if (kw2 <= NB)
                apply_block<NB>(g_ws_w[0], nbatch, m, ldA, stride, d_a, J0, kw2, c0, c1,
                                Tout + static_cast<size_t>(nbatch) * KO * KO, st);
            else
                apply_block<KO>(g_ws_w[0], nbatch, m, ldA, stride, d_a, J0, kw2, c0, c1, Tout, st);
        };
        panel_phase(0, Tb[0], st);
        for (int bi = 0, J0 = 0; J0 < n; ++bi, J0 += KO) {
            const int kw2 = std::min(KO, n - J0);
            double* Tcur = Tb[bi & 1];
            const int nJ = J0 + KO;  // next block
            if (nJ >= n) {
                update(J0, Tcur, J0 + kw2, ntot);
                break;
            }
            const int nend = std::min(nJ + KO, n);
            update(J0, Tcur, nJ, nend);  // the next block's columns first
            if (lookahead) {
                cudaEventRecord(ev_a, st);
                cudaStreamWaitEvent(side, ev_a, 0);
                panel_phase(nJ, Tb[(bi + 1) & 1], side);
                cudaEventRecord(ev_b, side);
                update(J0, Tcur, nend, ntot);
                cudaStreamWaitEvent(st, ev_b, 0);
            } else {
                update(J0, Tcur, nend, ntot);
                panel_phase(nJ, Tb[(bi + 1) & 1], st);
            }
        }
    }
    if (n > kFlipMaxN) throw std::runtime_error("blocked_qr_apply: n above the flip kernel's limit");
    dim3 g2((ntot + kFlipCols - 1) / kFlipCols, nbatch);
    k_flip<<<g2, 256, 0, st>>>(d_a, ldA, stride, n, ntot, d_sign, d_info);
    k_flip_diag<<<nbatch, 256, 0, st>>>(d_a, ldA, stride, n);
    CK(cudaEventRecord(D.done, st));
    D.used = true;
}

}  // namespace spqr
