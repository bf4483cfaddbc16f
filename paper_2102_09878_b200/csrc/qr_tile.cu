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
__device__ __forceinline__ void make_reflector(double* P, int m, int k, double* s_tau) {
    const int lane = threadIdx.x & 31;
    double* pk = P + static_cast<long long>(k) * m;
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
__device__ __forceinline__ void apply_panel(double* P, int m, int k, int j, double tau) {
    const int lane = threadIdx.x & 31;
    const double* pk = P + static_cast<long long>(k) * m;
    double* pj = P + static_cast<long long>(j) * m;
    double s = 0.0;
    for (int i = k + 1 + lane; i < m; i += 32) s = fma(pk[i], pj[i], s);
    const double tw = tau * (wsum(s) + pj[k]);
    for (int i = k + 1 + lane; i < m; i += 32) pj[i] = fma(-tw, pk[i], pj[i]);
    __syncwarp();
    if (lane == 0) pj[k] -= tw;
    __syncwarp();
}

// work.x = descriptor, [work.y, work.z) = trailing columns, work.w = tiles of this front.
// count[desc] (zero on entry, zero again on exit) elects the panel writer: the
// last CTA of the front to finish staging, so no CTA can still be reading the
// unfactored panel from global memory when it is overwritten.
template <int RPL, int CPW>
__global__ void __launch_bounds__(32 * kNW) k_qr_tile(const QrDesc* __restrict__ ds, const int4* __restrict__ work,
                                                      int* __restrict__ count) {
    const int4 wk = work[blockIdx.x];
    const QrDesc d = ds[wk.x];
    const int m = d.m, n = d.n, kmax = min(m, n);
    const long long ld = d.ld;
    extern __shared__ double P[];  // m x n panel, column-major, ld m
    __shared__ double s_tau[kQrTileMaxN];
    __shared__ unsigned char s_neg[kQrTileMaxN];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;

    // ---- stage the panel (4 loads in flight per thread)
    {
        const long long tot = static_cast<long long>(m) * n;
        for (long long e0 = threadIdx.x; e0 < tot; e0 += 4 * 32 * kNW) {
            double v[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long e = e0 + u * 32 * kNW;
                v[u] = 0.0;
                if (e < tot) {
                    const int j = static_cast<int>(e / m), i = static_cast<int>(e - static_cast<long long>(j) * m);
                    v[u] = d.a[i + j * ld];
                }
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const long long e = e0 + u * 32 * kNW;
                if (e < tot) P[e] = v[u];
            }
        }
    }
    __shared__ int s_writer;
    __syncthreads();
    if (threadIdx.x == 0) {
        int writer = 1;
        if (wk.w > 1) {
            writer = atomicAdd(count + wk.x, 1) == wk.w - 1;
            if (writer) count[wk.x] = 0;  // every other CTA of this front has already counted
        }
        s_writer = writer;
    }
    // ---- panel factorisation, one barrier per reflector
    if (kmax > 0 && wid == 0) make_reflector(P, m, 0, s_tau);
    __syncthreads();
    for (int k = 0; k < kmax; ++k) {
        const double tau = s_tau[k];
        int j = k + 1;
        j += (wid - j % kNW + kNW) % kNW;  // first owned column > k
        for (; j < n; j += kNW) {
            if (tau != 0.0) apply_panel(P, m, k, j, tau);
            if (j == k + 1 && j < kmax) make_reflector(P, m, j, s_tau);
        }
        __syncthreads();
    }
    for (int i = threadIdx.x; i < kmax; i += blockDim.x) s_neg[i] = P[i + static_cast<long long>(i) * m] < 0.0;
    __syncthreads();

    // ---- tile columns: registers, all reflectors, no barriers
    for (int j0 = wk.y + wid * CPW; j0 < wk.z; j0 += kNW * CPW) {
        double x[CPW][RPL];
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
            const int j = j0 + c;
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int i = lane + 32 * q;
                x[c][q] = (j < wk.z && i < m) ? d.a[i + j * ld] : 0.0;
            }
        }
        for (int k = 0; k < kmax; ++k) {
            const double tau = s_tau[k];
            if (tau == 0.0) continue;
            const double* pk = P + static_cast<long long>(k) * m;
            double vk[RPL];
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int i = lane + 32 * q;
                vk[q] = (i > k && i < m) ? pk[i] : (i == k ? 1.0 : 0.0);
            }
            double w[CPW];
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < RPL; ++q) s = fma(vk[q], x[c][q], s);
                w[c] = s;
            }
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int c = 0; c < CPW; ++c) w[c] += __shfl_xor_sync(0xffffffffu, w[c], o);
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const double tw = tau * w[c];
#pragma unroll
                for (int q = 0; q < RPL; ++q) x[c][q] = fma(-tw, vk[q], x[c][q]);
            }
        }
#pragma unroll
        for (int c = 0; c < CPW; ++c) {
            const int j = j0 + c;
            if (j >= wk.z) continue;
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int i = lane + 32 * q;
                if (i < m) d.a[i + j * ld] = (i < kmax && s_neg[i]) ? -x[c][q] : x[c][q];
            }
        }
    }

    // ---- first tile: factored panel, R copy, signs, flag, tau
    if (!s_writer) return;
    const long long tot = static_cast<long long>(m) * n;
    for (long long e = threadIdx.x; e < tot; e += blockDim.x) {
        const int j = static_cast<int>(e / m), i = static_cast<int>(e - static_cast<long long>(j) * m);
        double v = P[e];
        if (i <= j && i < kmax && s_neg[i]) v = -v;
        if (d.rout && i < n) d.rout[i + static_cast<long long>(j) * n] = (i <= j) ? v : 0.0;
        if (d.set_identity)
            v = (i == j) ? 1.0 : 0.0;
        else if (d.zero_lower && i > j)
            v = 0.0;
        d.a[i + j * ld] = v;
    }
    for (int i = threadIdx.x; i < kmax; i += blockDim.x) {
        const double r = fabs(P[i + static_cast<long long>(i) * m]);
        if (d.sign) d.sign[i] = s_neg[i] ? -1.0 : 1.0;
        if (d.tau) d.tau[i] = s_tau[i];
        if (d.flag && !(r >= DBL_MIN)) atomicMin(d.flag, i);
    }
}

template <int RPL, int CPW>
void launch_tile(const QrDesc* dd, const int4* dw, int nwork, size_t smem, int* count, cudaStream_t st) {
    static size_t configured = 0;
    smem_optin(reinterpret_cast<const void*>(k_qr_tile<RPL, CPW>), smem, configured);
    k_qr_tile<RPL, CPW><<<nwork, 32 * kNW, smem, st>>>(dd, dw, count);
}

}  // namespace

int qr_tile_class(int m, int n) {
    if (n > kQrTileMaxN || m < 1 || 8ull * m * n > kQrTileSmem) return -1;
    static const int maxm = std::getenv("SPQR_TILE_MAXM") ? std::atoi(std::getenv("SPQR_TILE_MAXM")) : 512;
    if (m > maxm) return -1;
    if (m <= 32) return 0;
    if (m <= 64) return 1;
    if (m <= 128) return 2;
    if (m <= 256) return 3;
    if (m <= 512) return 4;
    return -1;
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
        case 0: launch_tile<1, 4>(d_desc, d_work, nwork, smem, d_count, st); break;
        case 1: launch_tile<2, 4>(d_desc, d_work, nwork, smem, d_count, st); break;
        case 2: launch_tile<4, 2>(d_desc, d_work, nwork, smem, d_count, st); break;
        case 3: launch_tile<8, 2>(d_desc, d_work, nwork, smem, d_count, st); break;
        default: launch_tile<16, 1>(d_desc, d_work, nwork, smem, d_count, st); break;
    }
}

}  // namespace spqr
