// Column-tiled batched Householder QR + Q^T apply for small and medium fronts.
//
// Reference semantics: block_householder_qr (Eigen makeHouseholder convention,
// nonnegative-diagonal flip) + apply_reflectors_left_t on the neighbour block
// (proj/src/dense_kernels.cpp:11-35, 89-99); identical results to qr_body in
// kernels.cu up to floating-point summation order.
//
// Work unit = (front, tile of trailing columns).  Every CTA of a front stages
// the m x n panel in shared memory and factors it redundantly (the panel is
// small next to the trailing block, and redundancy removes every inter-CTA
// dependency); then each warp streams its tile columns through registers,
// applies all n reflectors from shared memory (no block barriers), flips the
// rows of negative R diagonals and stores the column once.  The CTA holding
// the first tile also writes the factored panel (R / V / [I;0]), the R copy,
// the signs and the singular-pivot flag.
//
// Panel factorisation: one barrier per reflector.  Warp (j mod 8) owns panel
// column j; after applying reflector k the owner of column k+1 immediately
// forms reflector k+1 (look-ahead), so the next step can start after a single
// __syncthreads.
#include <cfloat>
#include <climits>
#include <cmath>
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "dev.h"

namespace spqr {

namespace {

// warps per CTA by row class: 4 for panels of up to 128 rows (four CTAs per SM), 8 above
template <int TPC>
constexpr int nw_of() { return TPC <= 8 ? 4 : 8; }

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Eigen makeHouseholder on panel column k (rows k..m-1), warp-cooperative.
__device__ __forceinline__ void make_reflector(double* P, int ldp, int m, int k, double* s_tau) {
    const int lane = threadIdx.x & 31;
    double* pk = P + static_cast<long long>(k) * ldp;
    double s = 0.0;
    for (int i = k + 1 + lane; i < m; i += 32) s = fma(pk[i], pk[i], s);
    const double tail2 = wsum(s);
    const double c0 = pk[k];
    double tau = 0.0, den = 0.0;
    if (!(tail2 <= DBL_MIN)) {
        double beta = sqrt(c0 * c0 + tail2);
        if (hh_beta_negative(c0, tail2)) beta = -beta;
        den = c0 - beta;
        tau = (beta - c0) / beta;
        if (lane == 0) pk[k] = beta;
    }
    for (int i = k + 1 + lane; i < m; i += 32) pk[i] = (tau == 0.0) ? 0.0 : pk[i] / den;
    if (lane == 0) s_tau[k] = tau;
    __syncwarp();
}

// reflector k applied to panel column j (warp-cooperative, shared memory)
__device__ __forceinline__ void apply_panel(double* P, int ldp, int m, int k, int j, double tau) {
    const int lane = threadIdx.x & 31;
    const double* pk = P + static_cast<long long>(k) * ldp;
    double* pj = P + static_cast<long long>(j) * ldp;
    double s = 0.0;
    for (int i = k + 1 + lane; i < m; i += 32) s = fma(pk[i], pj[i], s);
    const double tw = tau * (wsum(s) + pj[k]);
    for (int i = k + 1 + lane; i < m; i += 32) pj[i] = fma(-tw, pk[i], pj[i]);
    __syncwarp();
    if (lane == 0) pj[k] -= tw;
    __syncwarp();
}

// Panel factorisation with the panel in registers (n <= 32, MP <= 256): warp
// g holds rows [g*RPT, (g+1)*RPT) and lane j holds column j.  Per reflector:
// the owners of column k reduce its tail norm across warps (barrier), every
// thread forms the same Householder scalars, the owners publish v (barrier),
// every column reduces its dot product with v across warps (barrier) and
// updates its rows.  The factored panel is written back to P.
template <int MP, int kNW>
__device__ void panel_regs(double* P, int m, int n, int kmax, double* s_tau) {
    constexpr int RPT = MP / kNW;
    __shared__ double red[kNW], vsh[MP], part[kNW][32];
    __shared__ double s_c0;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    const int r0 = wid * RPT;
    double x[RPT];
#pragma unroll
    for (int i = 0; i < RPT; ++i) x[i] = lane < n ? P[(r0 + i) + lane * MP] : 0.0;
    for (int i = threadIdx.x; i < MP; i += blockDim.x) vsh[i] = 0.0;
    // Row conditions are warp-uniform except in the one warp holding row k,
    // so the common paths below are branch-free loops over all RPT rows.
    for (int k = 0; k < kmax; ++k) {
        const bool below = r0 > k, holds = !below && r0 + RPT > k;
        if (lane == k) {
            double s = 0.0;
            if (below) {
#pragma unroll
                for (int i = 0; i < RPT; ++i) s = fma(x[i], x[i], s);
            } else if (holds) {
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    if (r0 + i > k) s = fma(x[i], x[i], s);
                    if (r0 + i == k) s_c0 = x[i];
                }
            }
            red[wid] = s;
        }
        __syncthreads();
        double tail2 = 0.0;
#pragma unroll
        for (int g = 0; g < kNW; ++g) tail2 += red[g];
        const double c0 = s_c0;
        double tau = 0.0, den = 0.0, beta = c0;
        if (!(tail2 <= DBL_MIN)) {  // Eigen makeHouseholder
            beta = sqrt(c0 * c0 + tail2);
            if (hh_beta_negative(c0, tail2)) beta = -beta;
            den = c0 - beta;
            tau = (beta - c0) / beta;
        }
        // v = tail / (c0 - beta): one reciprocal instead of RPT divisions in a
        // single lane (results differ from the division by at most 1 ulp)
        const double rden = (tau == 0.0) ? 0.0 : 1.0 / den;
        if (lane == k) {
            if (below) {
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    x[i] *= rden;
                    vsh[r0 + i] = x[i];
                }
            } else if (holds) {
#pragma unroll
                for (int i = 0; i < RPT; ++i) {
                    const int row = r0 + i;
                    if (row > k) x[i] *= rden;
                    if (row == k) x[i] = beta;
                    if (row >= k) vsh[row] = row > k ? x[i] : 1.0;
                }
            }
            if (r0 <= k - 1 && k - 1 < r0 + RPT) vsh[k - 1] = 0.0;  // previous unit entry
            if (wid == 0) s_tau[k] = tau;
        }
        __syncthreads();
        if (tau != 0.0) {  // rows above k hold v = 0 in vsh: no row conditions
            double p0 = 0.0, p1 = 0.0;
#pragma unroll
            for (int i = 0; i < RPT; i += 2) {
                p0 = fma(vsh[r0 + i], x[i], p0);
                p1 = fma(vsh[r0 + i + 1], x[i + 1], p1);
            }
            part[wid][lane] = p0 + p1;
            __syncthreads();
            if (lane > k && lane < n) {
                double w = 0.0;
#pragma unroll
                for (int g = 0; g < kNW; ++g) w += part[g][lane];
                const double tw = -tau * w;
#pragma unroll
                for (int i = 0; i < RPT; ++i) x[i] = fma(tw, vsh[r0 + i], x[i]);
            }
        }
    }
    __syncthreads();
    if (lane < n) {
#pragma unroll
        for (int i = 0; i < RPT; ++i) P[(r0 + i) + lane * MP] = x[i];
    }
    __syncthreads();
}

// Panel factorisation without block barriers inside a reflector (n <= 32, MP <= 128):
// the panel is swept in sub-panels of eight columns.  One warp factors a sub-panel
// entirely in registers - lane l holds rows l, l + 32, ... of the eight columns, so
// the tail norm of the pivot column and its dot products with the columns to its
// right are one shuffle butterfly, and the pivot row is one shuffle broadcast; no
// shared memory and no barrier per reflector.  Then every warp applies the eight
// new reflectors to one of the eight-column chunks to the right (reflector vectors
// from shared memory, the chunk in registers).  Two block barriers per sub-panel
// instead of three per reflector.  With v = tail / (c0 - beta) the products
// v^T x_j are formed as (tail^T x_j) / (c0 - beta): same arithmetic as
// make_reflector / apply_panel up to rounding.
template <int N>
__device__ __forceinline__ void wsum_n(double (&p)[8], int first) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
        for (int j = 0; j < N; ++j)
            if (j >= first) p[j] += __shfl_xor_sync(0xffffffffu, p[j], o);
    }
}

// XOR swizzle of the row index per column used by k_qr_wy's shared-memory panel (see there)
__device__ __forceinline__ int wy_swz(int j) { return (((j >> 1) & 3) ^ ((j & 1) << 1)) << 2; }

// One warp factors the eight panel columns c0..c0+7 in registers (straight-line code:
// reflectors beyond kmax and zero reflectors run as no-ops).  SWZ: rows stored at
// (row ^ wy_swz(column)); vtop (optional, SWZ only): the explicit reflectors' top 32 rows
// (unit diagonal, zeros above, zero columns beyond kmax), ld 32, same swizzle.
template <int MP, bool SWZ>
__device__ __forceinline__ void subpanel_factor(double* P, int c0, int n, int kmax, double* s_tau, int lane, double* vtop) {
    constexpr int RPL = MP / 32;  // rows per lane
    double x[RPL][8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int sw = SWZ ? wy_swz(c0 + j) : 0;
#pragma unroll
        for (int i = 0; i < RPL; ++i) x[i][j] = (c0 + j < n) ? P[((lane + 32 * i) ^ sw) + (c0 + j) * MP] : 0.0;
    }
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
        const int k = c0 + kk;
        const bool act = k < kmax;
        const bool t0 = lane > k;  // row `lane` lies below the pivot row (k < 32)
        double p[8], rk[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j < kk) continue;
            double a = t0 ? x[0][kk] * x[0][j] : 0.0;
#pragma unroll
            for (int i = 1; i < RPL; ++i) a = fma(x[i][kk], x[i][j], a);
            p[j] = a;
            rk[j] = __shfl_sync(0xffffffffu, x[0][j], k);  // pivot row
        }
        wsum_n<8>(p, kk);
        const double c = rk[kk], tail2 = p[kk];
        const bool nz = act && !(tail2 <= DBL_MIN);  // Eigen makeHouseholder
        double bt = sqrt(fma(c, c, tail2));
        if (hh_beta_negative(c, tail2)) bt = -bt;
        const double beta = nz ? bt : c;
        const double tau = nz ? (bt - c) / bt : 0.0;
        const double rden = nz ? 1.0 / (c - bt) : 0.0;
        const double sc = act ? rden : 1.0;  // tau == 0: the tail is cleared
#pragma unroll
        for (int i = 1; i < RPL; ++i) x[i][kk] *= sc;
        x[0][kk] = t0 ? x[0][kk] * sc : ((lane == k && act) ? beta : x[0][kk]);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            if (j <= kk) continue;
            const double w = tau * fma(p[j], rden, rk[j]);
#pragma unroll
            for (int i = 1; i < RPL; ++i) x[i][j] = fma(-w, x[i][kk], x[i][j]);
            x[0][j] = t0 ? fma(-w, x[0][kk], x[0][j]) : (lane == k ? x[0][j] - w : x[0][j]);
        }
        if (lane == 0 && act) s_tau[k] = tau;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
        const int sw = SWZ ? wy_swz(c0 + j) : 0;
#pragma unroll
        for (int i = 0; i < RPL; ++i)
            if (c0 + j < n) P[((lane + 32 * i) ^ sw) + (c0 + j) * MP] = x[i][j];
        if (SWZ && vtop) {
            const int k = c0 + j;
            vtop[(lane ^ sw) + k * 32] = k < kmax ? (lane > k ? x[0][j] : (lane == k ? 1.0 : 0.0)) : 0.0;
        }
    }
}

template <int MP, int kNW>
__device__ void panel_warp(double* P, int m_, int n_, int kmax_, double* s_tau) {
    constexpr int RPL = MP / 32;  // rows per lane
    // warp-uniform values are broadcast from lane 0 so that the compiler sees every branch
    // around the shuffles as convergent (plain SHFL instead of per-shuffle warp collectives)
    const int lane = threadIdx.x & 31;
    const int wid = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    const int n = __shfl_sync(0xffffffffu, n_, 0), kmax = __shfl_sync(0xffffffffu, kmax_, 0);
    (void)m_;
    const int nchunks = (n + 7) >> 3;
    for (int s = 0; 8 * s < kmax; ++s) {
        const int c0 = 8 * s;
        if (wid == 0) subpanel_factor<MP, false>(P, c0, n, kmax, s_tau, lane, nullptr);
        __syncthreads();
        if (s + 1 >= nchunks) break;  // uniform
        for (int q = s + 1 + wid; q < nchunks; q += kNW) {
            const int d0 = 8 * q;
            double y[RPL][8];
#pragma unroll
            for (int j = 0; j < 8; ++j)
#pragma unroll
                for (int i = 0; i < RPL; ++i) y[i][j] = (d0 + j < n) ? P[lane + 32 * i + (d0 + j) * MP] : 0.0;
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                const int k = c0 + kk;
                const double tau = k < kmax ? s_tau[k] : 0.0;
                const int kc = min(k, n - 1);  // a column that exists (its values are unused when tau = 0)
                double v[RPL], p[8];
                {
                    const double t = P[lane + kc * MP];
                    v[0] = lane > k ? t : (lane == k ? 1.0 : 0.0);
                }
#pragma unroll
                for (int i = 1; i < RPL; ++i) v[i] = P[lane + 32 * i + kc * MP];
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    double a = v[0] * y[0][j];
#pragma unroll
                    for (int i = 1; i < RPL; ++i) a = fma(v[i], y[i][j], a);
                    p[j] = a;
                }
                wsum_n<8>(p, 0);
#pragma unroll
                for (int j = 0; j < 8; ++j) {
                    const double w = -tau * p[j];
#pragma unroll
                    for (int i = 0; i < RPL; ++i) y[i][j] = fma(w, v[i], y[i][j]);
                }
            }
#pragma unroll
            for (int j = 0; j < 8; ++j)
#pragma unroll
                for (int i = 0; i < RPL; ++i)
                    if (d0 + j < n) P[lane + 32 * i + (d0 + j) * MP] = y[i][j];
        }
        __syncthreads();
    }
    __syncthreads();
}

__device__ __forceinline__ void dmma884(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// shared memory of the DMMA tile phase (doubles): X tile (MP x 32, ld MP+4; the
// staged panel aliases it), explicit V (MP x 32, ld MP+4), T and W (32 x 32, ld 36)
__host__ __device__ constexpr int dmma_tile_doubles(int MP) { return 2 * (MP + 4) * 32 + 2 * 36 * 32; }

// Tile phase on FP64 tensor cores (n <= 32, MP <= 256): the panel's reflectors in
// compact-WY form, H = I - V T V^T (T by accumulate_wy, dense_kernels.cpp:41-53),
// applied to 32-column tiles as three DMMA m8n8k4 products: W = V^T X,
// W = T^T W, X -= V W (apply_raw's blocked branch, dense_kernels.cpp:61-69).
// Leading dimensions are = 4 (mod 16) doubles so every fragment load is two
// conflict-free wavefronts.
template <int MP, int kNW>
__device__ void tile_dmma(const QrDesc& d, const int4& wk, double* sm, int kmax, const double* s_tau,
                          const unsigned char* s_neg) {
    constexpr int LV = MP + 4, LT = 36;
    const double* P = sm;  // factored panel (ld MP), consumed before sX is written
    double* sX = sm;
    double* sV = sm + LV * 32;
    double* sT = sV + LV * 32;
    double* sW = sT + LT * 32;
    const int m = d.m;
    const long long ld = d.ld;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, g = lane >> 2, t4 = lane & 3;
    for (int e = threadIdx.x; e < MP * 32; e += blockDim.x) {
        const int j = e / MP, r = e - j * MP;
        double v = 0.0;
        if (j < kmax) v = r < j ? 0.0 : (r == j ? 1.0 : P[r + j * MP]);
        sV[r + j * LV] = v;
    }
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) sT[(e & 31) + (e >> 5) * LT] = 0.0;
    __syncthreads();
    // Gram matrix V^T V (strict upper part) into sW, then T column by column
    for (int e = threadIdx.x; e < 32 * 32; e += blockDim.x) {
        const int i = e & 31, j = e >> 5;
        double s = 0.0;
        if (i < j && j < kmax) {
            const double* vi = sV + i * LV;
            const double* vj = sV + j * LV;
            double s1 = 0.0, s2 = 0.0, s3 = 0.0;
            int r = j;  // v_j is zero above row j
            for (; r + 3 < MP; r += 4) {
                s = fma(vi[r], vj[r], s);
                s1 = fma(vi[r + 1], vj[r + 1], s1);
                s2 = fma(vi[r + 2], vj[r + 2], s2);
                s3 = fma(vi[r + 3], vj[r + 3], s3);
            }
            for (; r < MP; ++r) s = fma(vi[r], vj[r], s);
            s = (s + s1) + (s2 + s3);
        }
        sW[i + j * LT] = s;
    }
    __syncthreads();
    if (wid == 0) {
        for (int j = 0; j < kmax; ++j) {
            const double tj = s_tau[j];
            if (tj == 0.0) continue;
            double s = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
            if (lane < j) {
                int q = lane;
                for (; q + 3 < j; q += 4) {
                    s = fma(sT[lane + q * LT], sW[q + j * LT], s);
                    s1 = fma(sT[lane + (q + 1) * LT], sW[q + 1 + j * LT], s1);
                    s2 = fma(sT[lane + (q + 2) * LT], sW[q + 2 + j * LT], s2);
                    s3 = fma(sT[lane + (q + 3) * LT], sW[q + 3 + j * LT], s3);
                }
                for (; q < j; ++q) s = fma(sT[lane + q * LT], sW[q + j * LT], s);
                s = (s + s1) + (s2 + s3);
            }
            __syncwarp();
            if (lane < j) sT[lane + j * LT] = -tj * s;
            if (lane == 0) sT[j + j * LT] = tj;
            __syncwarp();
        }
    }
    constexpr int NQ = 16 / kNW;  // W column tiles per warp (W is 4 x 4 tiles of 8 x 8)
    const int mt = wid & 3, nt = (wid >> 2) * NQ;
    for (int c0 = wk.y; c0 < wk.z; c0 += 32) {
        const int nc = min(32, wk.z - c0);
        __syncthreads();  // T ready / previous tile stored
        {  // all loads of the tile in flight at once
            constexpr int NL = MP * 32 / (32 * kNW);
            double xv[NL];
#pragma unroll
            for (int u = 0; u < NL; ++u) {
                const int e = threadIdx.x + u * 32 * kNW;
                const int c = e / MP, r = e - c * MP;
                xv[u] = (r < m && c < nc) ? d.a[r + static_cast<long long>(c0 + c) * ld] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < NL; ++u) {
                const int e = threadIdx.x + u * 32 * kNW;
                const int c = e / MP, r = e - c * MP;
                sX[r + c * LV] = xv[u];
            }
        }
        __syncthreads();
        // W = V^T X  (32 x 32): warp -> W rows 8 mt.., columns 8 nt.. (two tiles)
        double acc[NQ][2] = {};
#pragma unroll 8
        for (int k0 = 0; k0 < MP; k0 += 4) {
            const double a = sV[(k0 + t4) + (8 * mt + g) * LV];
#pragma unroll
            for (int q = 0; q < NQ; ++q) dmma884(acc[q][0], acc[q][1], a, sX[(k0 + t4) + (8 * (nt + q) + g) * LV]);
        }
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            sW[(8 * mt + g) + (8 * (nt + q) + 2 * t4) * LT] = acc[q][0];
            sW[(8 * mt + g) + (8 * (nt + q) + 2 * t4 + 1) * LT] = acc[q][1];
        }
        __syncthreads();
        // W = T^T W
        double acc2[NQ][2] = {};
#pragma unroll
        for (int k0 = 0; k0 < 32; k0 += 4) {
            const double a = sT[(k0 + t4) + (8 * mt + g) * LT];
#pragma unroll
            for (int q = 0; q < NQ; ++q) dmma884(acc2[q][0], acc2[q][1], a, sW[(k0 + t4) + (8 * (nt + q) + g) * LT]);
        }
        __syncthreads();
#pragma unroll
        for (int q = 0; q < NQ; ++q) {
            sW[(8 * mt + g) + (8 * (nt + q) + 2 * t4) * LT] = acc2[q][0];
            sW[(8 * mt + g) + (8 * (nt + q) + 2 * t4 + 1) * LT] = acc2[q][1];
        }
        __syncthreads();
        // X -= V W: warp -> row tiles wid, wid + 8, ..., all four column tiles
        for (int m8 = wid; m8 < MP / 8; m8 += kNW) {
            double o[4][2] = {{0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
            for (int k0 = 0; k0 < 32; k0 += 4) {
                const double a = sV[(8 * m8 + g) + (k0 + t4) * LV];
#pragma unroll
                for (int q = 0; q < 4; ++q) dmma884(o[q][0], o[q][1], a, sW[(k0 + t4) + (8 * q + g) * LT]);
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
                sX[(8 * m8 + g) + (8 * q + 2 * t4) * LV] -= o[q][0];
                sX[(8 * m8 + g) + (8 * q + 2 * t4 + 1) * LV] -= o[q][1];
            }
        }
        __syncthreads();
        for (int e = threadIdx.x; e < MP * 32; e += blockDim.x) {
            const int c = e / MP, r = e - c * MP;
            if (r < m && c < nc) {
                const double v = sX[r + c * LV];
                d.a[r + static_cast<long long>(c0 + c) * ld] = (r < kmax && s_neg[r]) ? -v : v;
            }
        }
    }
}

// work.x = descriptor, [work.y, work.z) = trailing columns, work.w = tiles of this front.
// count[desc] (zero on entry, zero again on exit) elects the panel writer: the
// last CTA of the front to finish staging, so no CTA can still be reading the
// unfactored panel from global memory when it is overwritten.
//
// Tile phase layout: TPC threads per column (consecutive lanes), each holding
// 8 row pairs {2(i*TPC + r), +1} in registers (16*TPC rows per column); one
// reflector costs 8 shared-memory pair loads, 16 FMAs for the dot product,
// log2(TPC) shuffles and 16 FMAs for the update, with no block barriers.
// ~120 registers; 4-warp CTAs, so four share an SM and their panel
// factorisations overlap the others' tile sweeps.
template <int TPC, bool WY, int kNW = nw_of<TPC>()>
__global__ void __launch_bounds__(32 * kNW, 16 / kNW) k_qr_tile(const QrDesc* __restrict__ ds, const int4* __restrict__ work,
                                                      int* __restrict__ count, int panel_regs_only) {
    constexpr int MP = 16 * TPC;  // padded rows (panel leading dimension)
    const int4 wk = work[blockIdx.x];
    const QrDesc d = ds[wk.x];
    const int m = d.m, n = d.n, kmax = min(m, n);
    const long long ld = d.ld;
    extern __shared__ double P[];  // MP x n panel, column-major; rows >= m are zero
    __shared__ double s_tau[kQrTileMaxN];
    __shared__ unsigned char s_neg[kQrTileMaxN];
    __shared__ int s_writer;
    const int wid = threadIdx.x >> 5;

    // ---- stage the panel (4 loads in flight per thread), zero padding rows
    {
        const int tot = MP * n;
        for (int e0 = threadIdx.x; e0 < tot; e0 += 4 * 32 * kNW) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * 32 * kNW;
                const int j = e / MP, i = e - j * MP;
                v[u] = (e < tot && i < m) ? d.a[i + j * ld] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const int e = e0 + u * 32 * kNW;
                if (e < tot) P[e] = v[u];
            }
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int writer = 1;
        if (wk.w > 1) {
            writer = atomicAdd(count + wk.x, 1) == wk.w - 1;
            if (writer) count[wk.x] = 0;  // every other CTA of this front has already counted
        }
        s_writer = writer;
    }
    // ---- panel factorisation
    if (MP <= 256 && n <= 32) {
        __syncthreads();
        if (panel_regs_only == 2) {  // timing probe: no factorisation
            for (int i = threadIdx.x; i < kmax; i += blockDim.x) s_tau[i] = 0.5;
        } else if (MP <= 128 && !panel_regs_only)
            panel_warp<(MP <= 128 ? MP : 128), kNW>(P, m, n, kmax, s_tau);
        else
            panel_regs<(MP <= 256 ? MP : 256), kNW>(P, m, n, kmax, s_tau);
    } else {  // smem panel, warp per column, one barrier per reflector (look-ahead)
        if (kmax > 0 && wid == 0) make_reflector(P, MP, m, 0, s_tau);
        __syncthreads();
        for (int k = 0; k < kmax; ++k) {
            const double tau = s_tau[k];
            int j = k + 1;
            j += (wid - j % kNW + kNW) % kNW;  // first owned column > k
            for (; j < n; j += kNW) {
                if (tau != 0.0) apply_panel(P, MP, m, k, j, tau);
                if (j == k + 1 && j < kmax) make_reflector(P, MP, m, j, s_tau);
            }
            __syncthreads();
        }
    }
    for (int i = threadIdx.x; i < kmax; i += blockDim.x) s_neg[i] = P[i + i * MP] < 0.0;
    __syncthreads();

    // ---- elected CTA: factored panel, R copy, signs, flag, tau
    if (s_writer) {
        const int tot = m * n;
        for (int e = threadIdx.x; e < tot; e += blockDim.x) {
            const int j = e / m, i = e - j * m;
            double v = P[i + j * MP];
            if (i <= j && i < kmax && s_neg[i]) v = -v;
            if (d.rout && i < n) d.rout[i + static_cast<long long>(j) * n] = (i <= j) ? v : 0.0;
            if (d.set_identity)
                v = (i == j) ? 1.0 : 0.0;
            else if (d.zero_lower && i > j)
                v = 0.0;
            d.a[i + j * ld] = v;
        }
        for (int i = threadIdx.x; i < kmax; i += blockDim.x) {
            const double r = fabs(P[i + i * MP]);
            if (d.sign) d.sign[i] = s_neg[i] ? -1.0 : 1.0;
            if (d.tau) d.tau[i] = s_tau[i];
            if (d.flag && !(r >= DBL_MIN)) atomicMin(d.flag, i);
        }
    }
    if (wk.z <= wk.y) return;
    __syncthreads();
    if (WY && MP <= 256 && n <= 32) {  // compact-WY tile phase on DMMA (SPQR_TILE_DMMA=1)
        tile_dmma<(MP <= 256 ? MP : 256), kNW>(d, wk, P, kmax, s_tau, s_neg);
        return;
    }
    // ---- explicit reflectors: V(:, k) = [0; 1; v], zero rows >= m
    for (int e = threadIdx.x; e < MP * kmax; e += blockDim.x) {
        const int k = e / MP, i = e - k * MP;
        if (i <= k) P[e] = (i == k) ? 1.0 : 0.0;
    }
    __syncthreads();

    // ---- tile columns: registers, all reflectors, no barriers.  Each thread
    // carries two columns (j and j + HALF) so every shared-memory load of v
    // feeds four FMAs.
    const int r = threadIdx.x % TPC;
    constexpr int HALF = 32 * kNW / TPC;  // column pairs per pass
    for (int base = wk.y; base < wk.z; base += 2 * HALF) {
        const int ja = base + static_cast<int>(threadIdx.x) / TPC, jb = ja + HALF;
        const bool acta = ja < wk.z, actb = jb < wk.z;
        const double* pa = d.a + static_cast<long long>(acta ? ja : wk.y) * ld;
        const double* pb = d.a + static_cast<long long>(actb ? jb : wk.y) * ld;
        double x[16], y[16];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = 2 * (i * TPC + r);
            x[2 * i] = (acta && row < m) ? pa[row] : 0.0;
            x[2 * i + 1] = (acta && row + 1 < m) ? pa[row + 1] : 0.0;
            y[2 * i] = (actb && row < m) ? pb[row] : 0.0;
            y[2 * i + 1] = (actb && row + 1 < m) ? pb[row + 1] : 0.0;
        }
        for (int k = 0; k < kmax; ++k) {
            const double tau = s_tau[k];
            if (tau == 0.0) continue;
            const double2* vk = reinterpret_cast<const double2*>(P + k * MP) + r;
            double sa0 = 0.0, sa1 = 0.0, sb0 = 0.0, sb1 = 0.0;
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double2 v = vk[i * TPC];
                sa0 = fma(v.x, x[2 * i], sa0);
                sa1 = fma(v.y, x[2 * i + 1], sa1);
                sb0 = fma(v.x, y[2 * i], sb0);
                sb1 = fma(v.y, y[2 * i + 1], sb1);
            }
            double sa = sa0 + sa1, sb = sb0 + sb1;
#pragma unroll
            for (int o = 1; o < TPC; o <<= 1) {
                sa += __shfl_xor_sync(0xffffffffu, sa, o);
                sb += __shfl_xor_sync(0xffffffffu, sb, o);
            }
            const double ta = -tau * sa, tb = -tau * sb;
            asm volatile("" ::: "memory");  // reload v below instead of keeping it live
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                const double2 v = vk[i * TPC];
                x[2 * i] = fma(ta, v.x, x[2 * i]);
                x[2 * i + 1] = fma(ta, v.y, x[2 * i + 1]);
                y[2 * i] = fma(tb, v.x, y[2 * i]);
                y[2 * i + 1] = fma(tb, v.y, y[2 * i + 1]);
            }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const int row = 2 * (i * TPC + r);
            const double fa = (row < kmax && s_neg[row]) ? -1.0 : 1.0;
            const double fb = (row + 1 < kmax && s_neg[row + 1]) ? -1.0 : 1.0;
            if (acta) {
                double* out = d.a + static_cast<long long>(ja) * ld;
                if (row < m) out[row] = fa * x[2 * i];
                if (row + 1 < m) out[row + 1] = fb * x[2 * i + 1];
            }
            if (actb) {
                double* out = d.a + static_cast<long long>(jb) * ld;
                if (row < m) out[row] = fa * y[2 * i];
                if (row + 1 < m) out[row + 1] = fb * y[2 * i + 1];
            }
        }
    }
}

// ---------------------------------------------------------------------------------------
// Fronts of 65..128 rows with panels of up to 32 columns and a wide trailing block (the
// C5 128x32+256 shape).  The panel is swept in sub-panels of eight columns; a sub-panel's
// reflectors are kept in compact-WY form H_7..H_0 = I - V_s T_s^T V_s^T (T_s 8 x 8, from the
// Gram matrix V_s^T V_s as accumulate_wy, dense_kernels.cpp:41-53) and applied on the FP64
// tensor cores (m8n8k4) to the panel's own later columns and to the trailing block, both held
// in REGISTERS.  A warp owns eight columns at a time; lane (g, t4) holds rows
// {8b + 2 t4, 8b + 2 t4 + 1}, b = 0..15, of column g, which is at once
//   * the A fragment of  W^T  = X^T V_s  (contraction over rows: k-lane t4 carries row
//     8b + 2 t4 + e in step (b, e) - a permutation of the contraction index that A and B share),
//   * and the C fragment of  X^T -= W'^T V_s^T  (C columns 2 t4, 2 t4 + 1 = those same rows).
// W^T leaves product 1 as a C fragment (reflectors 2 t4 + e), which is the A fragment of
// W'^T = W^T T_s under the same index permutation, and W'^T likewise feeds product 3.  So
// applying a block reflector needs no shuffles, no barriers and no shared-memory traffic for
// X or W; shared memory only serves the V and T_s operands.  The panel (R and raw reflectors)
// is stored 128 x 32 unpadded with the row index XOR-swizzled per column (wy_swz), so that both
// operand patterns are conflict-free: row pairs {8b + 2 t4, +1} of columns g, g + 1 as 16-byte
// loads (product 1, Gram matrix) and rows 8b + g of columns 2 t4 + e as 8-byte loads (product
// 3); the explicit form of the top 32 rows (unit diagonal, zeros above) is a second 32 x 32
// block.  The sub-panels themselves are factored by one warp in registers (subpanel_factor).
// 43 KB of shared memory and 128 registers: four 4-warp CTAs per SM, so the latency-bound
// sub-panel sweeps of some fronts overlap the tensor-core phase of others.
constexpr int kWyP = 128 * 32, kWyTop = 32 * 32;
constexpr int kWyLT = 10, kWyT = 8 * kWyLT;  // T_s row-major with padded rows: the (2 t4 + e, g) loads are conflict-free
constexpr size_t kWySmem = sizeof(double) * (kWyP + kWyTop + 4 * kWyT + 64);

// global-memory accesses of the trailing block (the pointer comes out of a descriptor, so the
// compiler would otherwise emit generic loads and stores)
__device__ __forceinline__ double2 wy_ldg2(const double* p) {
    double2 v;
    asm("ld.global.v2.f64 {%0, %1}, [%2];" : "=d"(v.x), "=d"(v.y) : "l"(p));
    return v;
}
__device__ __forceinline__ double wy_ldg(const double* p) {
    double v;
    asm("ld.global.f64 %0, [%1];" : "=d"(v) : "l"(p));
    return v;
}
__device__ __forceinline__ void wy_stg2(double* p, double2 v) {
    asm volatile("st.global.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}
__device__ __forceinline__ void wy_stg(double* p, double v) { asm volatile("st.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory"); }

// x (eight columns in the register layout above) <- H_7..H_0 of sub-panel S applied.
// Operand addresses: the swizzle only touches bits 2 and 3 of the row index, so
// (8b + r) ^ s = (r ^ (s & 4)) + 8 (b ^ (s >> 3 & 1)): one base pointer for even b and one
// for odd b per operand, and every load is base + constant.
template <int S>
__device__ __forceinline__ void wy_apply(double2 (&x)[16], const double* P, const double* vtop, const double* sTs, int g, int t4,
                                         int sg) {
    // product 1: W^T = X^T V_s (rows above 8 S are zero in V_s); four accumulation chains
    const int o1 = ((2 * t4) ^ (sg & 4)), h1 = 8 * ((sg >> 3) & 1);
    const double* p1e = P + (8 * S + g) * 128 + o1 + h1;
    const double* p1o = P + (8 * S + g) * 128 + o1 - h1;
    const double* q1e = vtop + (8 * S + g) * 32 + o1 + h1;
    const double* q1o = vtop + (8 * S + g) * 32 + o1 - h1;
    double w[4][2] = {};
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        if (b < S) continue;
        const double* src = (b < 4) ? ((b & 1) ? q1o : q1e) : ((b & 1) ? p1o : p1e);
        const double2 v = *reinterpret_cast<const double2*>(src + 8 * b);
        dmma884(w[2 * (b & 1)][0], w[2 * (b & 1)][1], x[b].x, v.x);
        dmma884(w[2 * (b & 1) + 1][0], w[2 * (b & 1) + 1][1], x[b].y, v.y);
    }
    const double w0 = (w[0][0] + w[1][0]) + (w[2][0] + w[3][0]);
    const double w1 = (w[0][1] + w[1][1]) + (w[2][1] + w[3][1]);
    // product 2: W'^T = W^T T_s, negated for product 3
    double u0 = 0.0, u1 = 0.0;
    dmma884(u0, u1, w0, sTs[S * kWyT + (2 * t4) * kWyLT + g]);
    dmma884(u0, u1, w1, sTs[S * kWyT + (2 * t4 + 1) * kWyLT + g]);
    u0 = -u0;
    u1 = -u1;
    // product 3: X^T -= W'^T V_s^T; columns ca = 8 S + 2 t4 and ca + 1 (swizzles t4 << 2, (t4 ^ 2) << 2)
    const int ca = 8 * S + 2 * t4;
    const int oa = g ^ ((t4 << 2) & 4), ha = 8 * ((t4 >> 1) & 1);
    const int ob = g ^ (((t4 ^ 2) << 2) & 4), hb = 8 * (((t4 ^ 2) >> 1) & 1);
    const double* p3a[2] = {P + ca * 128 + oa + ha, P + ca * 128 + oa - ha};
    const double* q3a[2] = {vtop + ca * 32 + oa + ha, vtop + ca * 32 + oa - ha};
    const double* p3b[2] = {P + (ca + 1) * 128 + ob + hb, P + (ca + 1) * 128 + ob - hb};
    const double* q3b[2] = {vtop + (ca + 1) * 32 + ob + hb, vtop + (ca + 1) * 32 + ob - hb};
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        if (b < S) continue;
        const double va = (b < 4) ? q3a[b & 1][8 * b] : p3a[b & 1][8 * b];
        dmma884(x[b].x, x[b].y, u0, va);
    }
#pragma unroll
    for (int b = 0; b < 16; ++b) {
        if (b < S) continue;
        const double vb = (b < 4) ? q3b[b & 1][8 * b] : p3b[b & 1][8 * b];
        dmma884(x[b].x, x[b].y, u1, vb);
    }
}

// T_s of sub-panel S by one warp: Gram matrix on DMMA, then row i of T_s by lane i
// (T(i, j) = -tau_j sum_{q = i..j-1} T(i, q) G(q, j): a row only needs its own earlier entries)
__device__ __forceinline__ void wy_subpanel_t(int S, const double* P, const double* vtop, double* sTs, double* Gs,
                                              const double* s_tau, int lane) {
    const int g = lane >> 2, t4 = lane & 3, sg = wy_swz(g);
    double c[2][2] = {};
    for (int b = S; b < 16; ++b) {  // V_s is zero above row 8 S
        double2 v;
        if (b < 4)
            v = *reinterpret_cast<const double2*>(vtop + (8 * S + g) * 32 + ((8 * b + 2 * t4) ^ sg));
        else
            v = *reinterpret_cast<const double2*>(P + (8 * S + g) * 128 + ((8 * b + 2 * t4) ^ sg));
        dmma884(c[0][0], c[0][1], v.x, v.x);
        dmma884(c[1][0], c[1][1], v.y, v.y);
    }
    Gs[g * 8 + 2 * t4] = c[0][0] + c[1][0];
    Gs[g * 8 + 2 * t4 + 1] = c[0][1] + c[1][1];
    __syncwarp();
    if (lane < 8) {
        double t[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const double tj = s_tau[8 * S + j];
            double acc = 0.0;
#pragma unroll
            for (int q = 0; q < j; ++q)
                if (q >= lane) acc = fma(t[q], Gs[q * 8 + j], acc);
            t[j] = j < lane ? 0.0 : (j == lane ? tj : -tj * acc);
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) sTs[S * kWyT + lane * kWyLT + j] = t[j];
    }
    __syncwarp();
}

template <int kNW>
__global__ void __launch_bounds__(32 * kNW, 16 / kNW) k_qr_wy(const QrDesc* __restrict__ ds, const int4* __restrict__ work,
                                                              int* __restrict__ count, long long* __restrict__ prof, int dbg) {
    constexpr int MP = 128;
    const int4 wk = work[blockIdx.x];
    const QrDesc d = ds[wk.x];
    const int m = d.m, n = d.n;  // 64 < m <= 128, n <= 32 < m: every column carries a reflector
    const long long ld = d.ld;
    extern __shared__ double sm[];
    double* P = sm;  // panel, swizzled: (r, j) at j * 128 + (r ^ wy_swz(j))
    double* vtop = sm + kWyP;
    double* sTs = vtop + kWyTop;
    double* Gs = sTs + 4 * kWyT;
    __shared__ double s_tau[32];
    __shared__ unsigned char s_neg[32];
    __shared__ int s_writer;
    const int lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
    const int wid = __shfl_sync(0xffffffffu, static_cast<int>(threadIdx.x >> 5), 0);
    long long tc[4];
    tc[0] = prof ? clock64() : 0;

    {  // stage the panel (zero padding rows and columns)
        constexpr int NE = MP * 32 / (32 * kNW);
        double v[NE];
#pragma unroll
        for (int u = 0; u < NE; ++u) {
            const int e = threadIdx.x + u * 32 * kNW;
            const int j = e >> 7, i = e & 127;
            v[u] = (j < n && i < m) ? d.a[i + j * ld] : 0.0;
        }
#pragma unroll
        for (int u = 0; u < NE; ++u) {
            const int e = threadIdx.x + u * 32 * kNW;
            const int j = e >> 7, i = e & 127;
            P[j * MP + (i ^ wy_swz(j))] = v[u];
        }
    }
    if (threadIdx.x < 32) s_tau[threadIdx.x] = 0.0;
    for (int e = threadIdx.x; e < kWyTop + 4 * kWyT; e += blockDim.x) vtop[e] = 0.0;  // vtop and T_s
    __syncthreads();
    if (threadIdx.x == 0) {  // the last CTA of the front to finish staging writes the panel
        int writer = 1;
        if (wk.w > 1) {
            writer = atomicAdd(count + wk.x, 1) == wk.w - 1;
            if (writer) count[wk.x] = 0;
        }
        s_writer = writer;
    }
    tc[1] = prof ? clock64() : 0;
    // ---- panel: factor sub-panel S (warp 0), T_s, block-apply to the later chunks (one per warp)
    const int nchunks = __shfl_sync(0xffffffffu, (n + 7) >> 3, 0);
    const int sg = wy_swz(g);  // swizzle of columns 8 q + g
    for (int S = 0; S < nchunks; ++S) {
        if (wid == 0 && !(dbg & 1)) {
            subpanel_factor<MP, true>(P, 8 * S, n, n, s_tau, lane, vtop);
            __syncwarp();
            wy_subpanel_t(S, P, vtop, sTs, Gs, s_tau, lane);
        }
        __syncthreads();
        if (S + 1 >= nchunks) break;
        for (int q = S + 1 + wid; q < nchunks; q += kNW) {
            double* yp = P + (8 * q + g) * MP;
            double2 y[16];
#pragma unroll
            for (int b = 0; b < 16; ++b) y[b] = *reinterpret_cast<const double2*>(yp + ((8 * b + 2 * t4) ^ sg));
            if (S == 0)
                wy_apply<0>(y, P, vtop, sTs, g, t4, sg);
            else if (S == 1)
                wy_apply<1>(y, P, vtop, sTs, g, t4, sg);
            else
                wy_apply<2>(y, P, vtop, sTs, g, t4, sg);
#pragma unroll
            for (int b = 0; b < 16; ++b) *reinterpret_cast<double2*>(yp + ((8 * b + 2 * t4) ^ sg)) = y[b];
        }
        // no barrier here: warp 0 has just updated chunk S + 1 itself and goes on to factor it
        // while the other warps finish theirs (they touch neither that chunk nor T_{S+1}); the
        // barrier after the next factorisation orders their updates before the next round
        __syncwarp();
    }
    __syncthreads();
    tc[2] = prof ? clock64() : 0;
    for (int i = threadIdx.x; i < 32; i += blockDim.x) s_neg[i] = i < n && P[i * MP + (i ^ wy_swz(i))] < 0.0;
    __syncthreads();
    if (s_writer) {
        const int tot = m * n;
        for (int e = threadIdx.x; e < tot; e += blockDim.x) {
            const int j = e / m, i = e - j * m;
            double v = P[j * MP + (i ^ wy_swz(j))];
            if (i <= j && s_neg[i]) v = -v;
            if (d.rout && i < n) d.rout[i + static_cast<long long>(j) * n] = (i <= j) ? v : 0.0;
            if (d.set_identity)
                v = (i == j) ? 1.0 : 0.0;
            else if (d.zero_lower && i > j)
                v = 0.0;
            d.a[i + j * ld] = v;
        }
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const double r = fabs(P[i * MP + (i ^ wy_swz(i))]);
            if (d.sign) d.sign[i] = s_neg[i] ? -1.0 : 1.0;
            if (d.tau) d.tau[i] = s_tau[i];
            if (d.flag && !(r >= DBL_MIN)) atomicMin(d.flag, i);
        }
    }
    // ---- trailing block: eight columns per warp pass, the four block reflectors in turn
    const bool vec_ok = ((reinterpret_cast<uintptr_t>(d.a) | static_cast<uintptr_t>(ld * 8)) & 15) == 0;
    for (int n0 = wk.y + 8 * wid; n0 < wk.z; n0 += 8 * kNW) {
        const int col = n0 + g;
        const bool cok = col < wk.z;
        double* xp = d.a + static_cast<long long>(cok ? col : wk.y) * ld;
        double2 x[16];
#pragma unroll
        for (int b = 0; b < 16; ++b) {
            const int row = 8 * b + 2 * t4;
            if (dbg & 2) {
                x[b] = make_double2(1.0, 2.0);
            } else if (cok && vec_ok && row + 1 < m) {
                x[b] = wy_ldg2(xp + row);
            } else {
                x[b].x = (cok && row < m) ? wy_ldg(xp + row) : 0.0;
                x[b].y = (cok && row + 1 < m) ? wy_ldg(xp + row + 1) : 0.0;
            }
        }
        wy_apply<0>(x, P, vtop, sTs, g, t4, sg);
        if (nchunks > 1) wy_apply<1>(x, P, vtop, sTs, g, t4, sg);
        if (nchunks > 2) wy_apply<2>(x, P, vtop, sTs, g, t4, sg);
        if (nchunks > 3) wy_apply<3>(x, P, vtop, sTs, g, t4, sg);
        if (cok && !((dbg & 2) && x[0].x != 12345.0)) {
#pragma unroll
            for (int b = 0; b < 16; ++b) {
                const int row = 8 * b + 2 * t4;
                if (b < 4) {  // rows of negative R diagonals are flipped
                    if (s_neg[row]) x[b].x = -x[b].x;
                    if (s_neg[row + 1]) x[b].y = -x[b].y;
                }
                if (vec_ok && row + 1 < m) {
                    wy_stg2(xp + row, x[b]);
                } else {
                    if (row < m) wy_stg(xp + row, x[b].x);
                    if (row + 1 < m) wy_stg(xp + row + 1, x[b].y);
                }
            }
        }
    }
    if (prof) {
        tc[3] = clock64();
        if (threadIdx.x == 0) {
            for (int i = 0; i < 3; ++i) atomicAdd(reinterpret_cast<unsigned long long*>(prof) + i, static_cast<unsigned long long>(tc[i + 1] - tc[i]));
            atomicAdd(reinterpret_cast<unsigned long long*>(prof) + 3, 1ull);
        }
    }
}

// The register/FMA tile phase is the default: measured on C5 128x32+256 x 4096 it
// takes 1.85 ms against 2.16 ms for the DMMA compact-WY variant (32-column
// passes, five barriers each); SPQR_TILE_DMMA=1 selects the latter.
bool tile_dmma_enabled() { return std::getenv("SPQR_TILE_DMMA") != nullptr; }
// SPQR_PANEL_REGS=1: the barrier-per-reflector register panel for every row class
// (comparisons); default is the warp-local sub-panel sweep up to 128 rows.
static int panel_regs_only() {
    static const int v = std::getenv("SPQR_PANEL_REGS") ? std::atoi(std::getenv("SPQR_PANEL_REGS")) : 0;
    return v;
}

template <int TPC>
void launch_tile(const QrDesc* dd, const int4* dw, int nwork, size_t smem, int* count, cudaStream_t st) {
    if (tile_dmma_enabled()) {
        static SmemCfg configured;
        smem_optin(reinterpret_cast<const void*>(k_qr_tile<TPC, true>), smem, configured);
        k_qr_tile<TPC, true><<<nwork, 32 * nw_of<TPC>(), smem, st>>>(dd, dw, count, panel_regs_only());
    } else {
        static SmemCfg configured;
        smem_optin(reinterpret_cast<const void*>(k_qr_tile<TPC, false>), smem, configured);
        k_qr_tile<TPC, false><<<nwork, 32 * nw_of<TPC>(), smem, st>>>(dd, dw, count, panel_regs_only());
    }
}

}  // namespace

bool qr_wy_ok(int m, int n, int ntot) { return m > 64 && m <= 128 && n >= 1 && n <= 32 && ntot - n >= 64; }
bool qr_wy_enabled() { return std::getenv("SPQR_NO_WY") == nullptr; }

void launch_qr_wy(const QrDesc* d_desc, const int4* d_work, int nwork, int* d_count, cudaStream_t st) {
    if (nwork <= 0) return;
    static SmemCfg configured;
    smem_optin(reinterpret_cast<const void*>(k_qr_wy<4>), kWySmem, configured);
    // SPQR_WY_PROF=1: per-phase clock64 totals of thread 0 of every CTA (stage, panel, output + tiles), printed after the launch (diagnostic; synchronises)
    static const bool prof = std::getenv("SPQR_WY_PROF") != nullptr;
    long long* dp = nullptr;
    if (prof) {
        cudaMalloc(&dp, 8 * sizeof(long long));
        cudaMemsetAsync(dp, 0, 8 * sizeof(long long), st);
    }
    // SPQR_WY_DBG (timing probes, wrong results): 1 = no sub-panel factorisation, 2 = no trailing loads / stores
    static const int dbg = std::getenv("SPQR_WY_DBG") ? std::atoi(std::getenv("SPQR_WY_DBG")) : 0;
    k_qr_wy<4><<<nwork, 128, kWySmem, st>>>(d_desc, d_work, d_count, dp, dbg);
    if (prof) {
        long long h[8];
        cudaStreamSynchronize(st);
        cudaMemcpy(h, dp, sizeof(h), cudaMemcpyDeviceToHost);
        cudaFree(dp);
        const double c = h[3] ? double(h[3]) : 1.0;
        std::fprintf(stderr, "[wy prof] %lld CTAs, mean cycles: stage %.0f panel %.0f output+tiles %.0f\n", h[3], h[0] / c,
                     h[1] / c, h[2] / c);
    }
}

int qr_tile_class(int m, int n) {
    static const int maxm = std::getenv("SPQR_TILE_MAXM") ? std::atoi(std::getenv("SPQR_TILE_MAXM")) : 512;
    if (n > kQrTileMaxN || m < 1 || m > maxm) return -1;
    int cls = 0;
    while ((32 << cls) < m) ++cls;
    if (cls > 4 || qr_tile_smem(cls, n) > kQrTileSmem) return -1;
    return cls;
}

size_t qr_tile_smem(int cls, int n) {
    const int MP = 32 << cls;
    if (tile_dmma_enabled() && MP <= 256 && n <= 32) return sizeof(double) * static_cast<size_t>(dmma_tile_doubles(MP));
    return sizeof(double) * static_cast<size_t>(MP) * n;
}

std::vector<int4> qr_tile_plan(const QrDesc* hq, const int* idx, int cnt, int sms) {
    long long trail = 0;
    for (int t = 0; t < cnt; ++t) trail += std::max(0, hq[idx[t]].ntot - hq[idx[t]].n);
    long long tc = (trail + 2LL * sms - 1) / (2LL * sms);
    tc = std::min<long long>(512, std::max<long long>(16, (tc + 15) / 16 * 16));
    if (const char* f = std::getenv("SPQR_TILE_TC")) tc = std::atoll(f);
    std::vector<int4> wk;
    for (int t = 0; t < cnt; ++t) {
        const int i = idx[t], n = hq[i].n, nt = hq[i].ntot;
        if (nt <= n) {
            wk.push_back(int4{i, n, n, 1});
            continue;
        }
        const int tiles = static_cast<int>((nt - n + tc - 1) / tc);
        for (int c0 = n; c0 < nt; c0 += static_cast<int>(tc))
            wk.push_back(int4{i, c0, std::min(nt, c0 + static_cast<int>(tc)), tiles});
    }
    return wk;
}

void launch_qr_tile(int cls, const QrDesc* d_desc, const int4* d_work, int nwork, size_t smem, int* d_count,
                    cudaStream_t st) {
    if (nwork <= 0) return;
    switch (cls) {
        case 0: launch_tile<2>(d_desc, d_work, nwork, smem, d_count, st); break;
        case 1: launch_tile<4>(d_desc, d_work, nwork, smem, d_count, st); break;
        case 2: launch_tile<8>(d_desc, d_work, nwork, smem, d_count, st); break;
        case 3: launch_tile<16>(d_desc, d_work, nwork, smem, d_count, st); break;
        default: launch_tile<32>(d_desc, d_work, nwork, smem, d_count, st); break;
    }
}

}  // namespace spqr
