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
                                                      int* __restrict__ count) {
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

// The register/FMA tile phase is the default: measured on C5 128x32+256 x 4096 it
// takes 1.85 ms against 2.16 ms for the DMMA compact-WY variant (32-column
// passes, five barriers each); SPQR_TILE_DMMA=1 selects the latter.
bool tile_dmma_enabled() { return std::getenv("SPQR_TILE_DMMA") != nullptr; }

template <int TPC>
void launch_tile(const QrDesc* dd, const int4* dw, int nwork, size_t smem, int* count, cudaStream_t st) {
    if (tile_dmma_enabled()) {
        static SmemCfg configured;
        smem_optin(reinterpret_cast<const void*>(k_qr_tile<TPC, true>), smem, configured);
        k_qr_tile<TPC, true><<<nwork, 32 * nw_of<TPC>(), smem, st>>>(dd, dw, count);
    } else {
        static SmemCfg configured;
        smem_optin(reinterpret_cast<const void*>(k_qr_tile<TPC, false>), smem, configured);
        k_qr_tile<TPC, false><<<nwork, 32 * nw_of<TPC>(), smem, st>>>(dd, dw, count);
    }
}

}  // namespace

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
