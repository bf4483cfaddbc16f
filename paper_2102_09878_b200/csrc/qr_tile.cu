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

constexpr int kNW = 8;  // warps per CTA

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
        if (c0 >= 0.0) beta = -beta;
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
template <int MP>
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
            if (c0 >= 0.0) beta = -beta;
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

// work.x = descriptor, [work.y, work.z) = trailing columns, work.w = tiles of this front.
// count[desc] (zero on entry, zero again on exit) elects the panel writer: the
// last CTA of the front to finish staging, so no CTA can still be reading the
// unfactored panel from global memory when it is overwritten.
//
// Tile phase layout: TPC threads per column (consecutive lanes), each holding
// 8 row pairs {2(i*TPC + r), +1} in registers (16*TPC rows per column); one
// reflector costs 8 shared-memory pair loads, 16 FMAs for the dot product,
// log2(TPC) shuffles and 16 FMAs for the update, with no block barriers.
// ~100 registers, so two CTAs share an SM and one's panel factorisation
// overlaps the other's tile sweep.
template <int TPC>
__global__ void __launch_bounds__(32 * kNW, 2) k_qr_tile(const QrDesc* __restrict__ ds, const int4* __restrict__ work,
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
        panel_regs<(MP <= 256 ? MP : 256)>(P, m, n, kmax, s_tau);
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

template <int TPC>
void launch_tile(const QrDesc* dd, const int4* dw, int nwork, size_t smem, int* count, cudaStream_t st) {
    static size_t configured = 0;
    smem_optin(reinterpret_cast<const void*>(k_qr_tile<TPC>), smem, configured);
    k_qr_tile<TPC><<<nwork, 32 * kNW, smem, st>>>(dd, dw, count);
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

size_t qr_tile_smem(int cls, int n) { return sizeof(double) * (32u << cls) * static_cast<size_t>(n); }

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
