// W sweeps and CGLS vector kernels (proj/src/transforms.cpp:40-111,
// proj/src/solve.cpp:24-76) for B200.
//
// A sweep runs W's level schedule (solve.cpp build_solve_plan): the factors of one
// level touch disjoint column sets and no factor's cols meet another's coupled set,
// so a level is one launch with one warp per factor (one CTA per wide factor).
// wt_solve's coupled updates (z[coupled] -= C^T zs) may hit the same column from
// several factors of a level: each factor writes its contribution to a scratch
// vector and a second kernel subtracts them per column in walk order, which is the
// reference's sequential order and keeps the result deterministic.
#include <algorithm>
#include <cfloat>
#include <cmath>

#include "dev.h"

namespace spqr {

namespace {

constexpr int kWarpsPerBlock = 4;

// mode: 0 w_solve (z <- F^{-1} z), 1 wt_solve (F^{-T}), 2 w_apply (F), 3 wt_apply (F^T)
__global__ void k_wsweep(const WFac* __restrict__ fs, int nf, double* __restrict__ z, double* __restrict__ contrib,
                         int mode, int maxc) {
    extern __shared__ double smem[];
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
    const int fi = blockIdx.x * kWarpsPerBlock + wl;
    if (fi >= nf) return;
    const WFac f = fs[fi];
    double* x = smem + static_cast<long long>(wl) * maxc;
    const int c = f.c;
    for (int i = lane; i < c; i += 32) x[i] = z[f.cols[i]];
    __syncwarp();
    if (f.kind == 0) {
        const double* R = f.a;
        const double* C = f.a + static_cast<long long>(c) * c;
        if (mode == 0) {  // zs = z[cols] - C z[coupled]; zs = R^{-1} zs
            if (f.k > 0)
                for (int i = lane; i < c; i += 32) {
                    double s = 0.0;
                    for (int j = 0; j < f.k; ++j) s = fma(C[i + static_cast<long long>(j) * c], z[f.coupled[j]], s);
                    x[i] -= s;
                }
            __syncwarp();
            for (int i = c - 1; i >= 0; --i) {
                const double xi = x[i] / R[i + static_cast<long long>(i) * c];
                __syncwarp();
                for (int l = lane; l < i; l += 32) x[l] = fma(-R[l + static_cast<long long>(i) * c], xi, x[l]);
                if (lane == 0) x[i] = xi;
                __syncwarp();
            }
        } else if (mode == 1) {  // zs = R^{-T} z[cols]; contributions C^T zs
            for (int i = 0; i < c; ++i) {
                const double xi = x[i] / R[i + static_cast<long long>(i) * c];
                __syncwarp();
                for (int l = i + 1 + lane; l < c; l += 32) x[l] = fma(-R[i + static_cast<long long>(l) * c], xi, x[l]);
                if (lane == 0) x[i] = xi;
                __syncwarp();
            }
            for (int j = lane; j < f.k; j += 32) {
                double s = 0.0;
                const double* cj = C + static_cast<long long>(j) * c;
                for (int i = 0; i < c; ++i) s = fma(cj[i], x[i], s);
                contrib[f.contrib_off + j] = s;
            }
        } else if (mode == 2) {  // out = R zs + C z[coupled]
            for (int i = lane; i < c; i += 32) {
                double s = 0.0;
                for (int j = i; j < c; ++j) s = fma(R[i + static_cast<long long>(j) * c], x[j], s);
                double t = 0.0;
                for (int j = 0; j < f.k; ++j) t = fma(C[i + static_cast<long long>(j) * c], z[f.coupled[j]], t);
                z[f.cols[i]] = s + t;
            }
            return;
        } else {  // mode 3: contributions C^T zs (+), out = R^T zs
            for (int j = lane; j < f.k; j += 32) {
                double s = 0.0;
                const double* cj = C + static_cast<long long>(j) * c;
                for (int i = 0; i < c; ++i) s = fma(cj[i], x[i], s);
                contrib[f.contrib_off + j] = s;
            }
            for (int i = lane; i < c; i += 32) {
                double s = 0.0;
                for (int j = 0; j <= i; ++j) s = fma(R[j + static_cast<long long>(i) * c], x[j], s);
                z[f.cols[i]] = s;
            }
            return;
        }
    } else {
        // rotation factor Q^T on cols: w_apply / wt_solve apply H^T (reflectors then flip);
        // w_solve / wt_apply apply H (flip then reflectors), dense_kernels.cpp:96-104
        const double* V = f.a;
        const bool transpose = (mode == 1 || mode == 2);
        auto reflect = [&](int j) {
            const double tj = f.tau[j];
            if (tj == 0.0) return;
            const double* v = V + static_cast<long long>(j) * c;
            double w = 0.0;
            for (int i = j + lane; i < c; i += 32) w = fma(x[i], v[i], w);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1) w += __shfl_xor_sync(0xffffffffu, w, o);
            const double tw = tj * w;
            __syncwarp();
            for (int i = j + lane; i < c; i += 32) x[i] = fma(-tw, v[i], x[i]);
            __syncwarp();
        };
        if (transpose) {
            for (int j = 0; j < f.k; ++j) reflect(j);
            for (int i = lane; i < f.k; i += 32)
                if (f.sign[i] < 0.0) x[i] = -x[i];
        } else {
            for (int i = lane; i < f.k; i += 32)
                if (f.sign[i] < 0.0) x[i] = -x[i];
            __syncwarp();
            for (int j = f.k - 1; j >= 0; --j) reflect(j);
        }
    }
    __syncwarp();
    for (int i = lane; i < c; i += 32) z[f.cols[i]] = x[i];
}

// One large factor per CTA (the top-level separators of the 3D and kNN
// problems have factors thousands of columns wide; a warp per factor would
// serialise them).  Same semantics as k_wsweep (transforms.cpp:40-111), work
// spread over the CTA: products are thread-per-row GEMVs over the column-major
// blocks (coalesced), triangular solves are blocked by 32 (one warp solves the
// diagonal block, the CTA updates the rest), reflector dot products are block
// reductions.
constexpr int kBigThreads = 512;
constexpr int kBigWarps = kBigThreads / 32;

__device__ __forceinline__ double block_reduce(double v, double* red) {
    const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    __syncthreads();
    if (lane == 0) red[wl] = v;
    __syncthreads();
    double t = 0.0;
#pragma unroll
    for (int w = 0; w < kBigWarps; ++w) t += red[w];
    return t;
}

__global__ void __launch_bounds__(kBigThreads) k_wsweep_big(const WFac* __restrict__ fs, double* __restrict__ z,
                                                          double* __restrict__ contrib, int mode) {
    extern __shared__ double x[];
    __shared__ double red[kBigWarps];
    const WFac f = fs[blockIdx.x];
    const int c = f.c, tid = threadIdx.x, lane = tid & 31, wl = tid >> 5;
    for (int i = tid; i < c; i += kBigThreads) x[i] = z[f.cols[i]];
    __syncthreads();
    if (f.kind == 0) {
        const double* R = f.a;
        const double* C = f.a + static_cast<long long>(c) * c;
        // C^T x -> contributions, warp per coupled column (modes 1 and 3)
        auto ctx = [&]() {
            for (int j = wl; j < f.k; j += kBigWarps) {
                const double* cj = C + static_cast<long long>(j) * c;
                double s = 0.0;
                for (int i = lane; i < c; i += 32) s = fma(cj[i], x[i], s);
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
                if (lane == 0) contrib[f.contrib_off + j] = s;
            }
        };
        if (mode == 0) {  // zs = z[cols] - C z[coupled]; zs = R^{-1} zs
            if (f.k > 0) {
                for (int i = tid; i < c; i += kBigThreads) {
                    double s = 0.0;
                    for (int j = 0; j < f.k; ++j) s = fma(C[i + static_cast<long long>(j) * c], z[f.coupled[j]], s);
                    x[i] -= s;
                }
                __syncthreads();
            }
            for (int i1 = c; i1 > 0; i1 -= 32) {  // backward, 32-row blocks
                const int i0 = max(0, i1 - 32);
                if (wl == 0) {
                    for (int i = i1 - 1; i >= i0; --i) {
                        const double xi = x[i] / R[i + static_cast<long long>(i) * c];
                        __syncwarp();
                        const int l = i0 + lane;
                        if (l < i) x[l] = fma(-R[l + static_cast<long long>(i) * c], xi, x[l]);
                        if (lane == 0) x[i] = xi;
                        __syncwarp();
                    }
                }
                __syncthreads();
                for (int r = tid; r < i0; r += kBigThreads) {
                    double s = 0.0;
                    for (int i = i0; i < i1; ++i) s = fma(R[r + static_cast<long long>(i) * c], x[i], s);
                    x[r] -= s;
                }
                __syncthreads();
            }
        } else if (mode == 1) {  // zs = R^{-T} z[cols]; contributions C^T zs
            for (int i0 = 0; i0 < c; i0 += 32) {  // forward, 32-row blocks
                const int i1 = min(c, i0 + 32);
                if (wl == 0) {
                    for (int i = i0; i < i1; ++i) {
                        const double xi = x[i] / R[i + static_cast<long long>(i) * c];
                        __syncwarp();
                        const int l = i0 + lane;
                        if (l > i && l < i1) x[l] = fma(-R[i + static_cast<long long>(l) * c], xi, x[l]);
                        if (lane == 0) x[i] = xi;
                        __syncwarp();
                    }
                }
                __syncthreads();
                for (int r = i1 + tid; r < c; r += kBigThreads) {
                    const double* rr = R + static_cast<long long>(r) * c;  // column r: R(i0:i1, r) contiguous
                    double s = 0.0;
                    for (int i = i0; i < i1; ++i) s = fma(rr[i], x[i], s);
                    x[r] -= s;
                }
                __syncthreads();
            }
            ctx();
        } else if (mode == 2) {  // out = R zs + C z[coupled]
            for (int i = tid; i < c; i += kBigThreads) {
                double s = 0.0;
                for (int j = i; j < c; ++j) s = fma(R[i + static_cast<long long>(j) * c], x[j], s);
                double t = 0.0;
                for (int j = 0; j < f.k; ++j) t = fma(C[i + static_cast<long long>(j) * c], z[f.coupled[j]], t);
                z[f.cols[i]] = s + t;
            }
            return;
        } else {  // mode 3: contributions C^T zs, out = R^T zs
            ctx();
            for (int i = tid; i < c; i += kBigThreads) {
                const double* ri = R + static_cast<long long>(i) * c;
                double s = 0.0;
                for (int j = 0; j <= i; ++j) s = fma(ri[j], x[j], s);
                z[f.cols[i]] = s;
            }
            return;
        }
    } else {
        const double* V = f.a;
        const bool transpose = (mode == 1 || mode == 2);
        auto reflect = [&](int j) {
            const double tj = f.tau[j];
            if (tj == 0.0) return;
            const double* v = V + static_cast<long long>(j) * c;
            double w = 0.0;
            for (int i = j + tid; i < c; i += kBigThreads) w = fma(x[i], v[i], w);
            const double tw = tj * block_reduce(w, red);
            for (int i = j + tid; i < c; i += kBigThreads) x[i] = fma(-tw, v[i], x[i]);
            __syncthreads();
        };
        if (transpose) {
            for (int j = 0; j < f.k; ++j) reflect(j);
            for (int i = tid; i < f.k; i += kBigThreads)
                if (f.sign[i] < 0.0) x[i] = -x[i];
        } else {
            for (int i = tid; i < f.k; i += kBigThreads)
                if (f.sign[i] < 0.0) x[i] = -x[i];
            __syncthreads();
            for (int j = f.k - 1; j >= 0; --j) reflect(j);
        }
    }
    __syncthreads();
    for (int i = tid; i < c; i += kBigThreads) z[f.cols[i]] = x[i];
}

__global__ void k_wreduce(const int* __restrict__ ptr, const int* __restrict__ idx, const int* __restrict__ col, int ncol,
                          const double* __restrict__ contrib, double* __restrict__ z, double sgn) {
    const int t = blockIdx.x * blockDim.x + threadIdx.x;
    if (t >= ncol) return;
    double v = z[col[t]];
    for (int q = ptr[t]; q < ptr[t + 1]; ++q) v = (sgn < 0) ? v - contrib[idx[q]] : v + contrib[idx[q]];
    z[col[t]] = v;
}

__global__ void k_spmv_csr(int m, const int* __restrict__ ptr, const int* __restrict__ idx, const double* __restrict__ val,
                           const double* __restrict__ x, double* __restrict__ y) {
    const int r = blockIdx.x * blockDim.x + threadIdx.x;
    if (r >= m) return;
    double s = 0.0;
    for (int k = ptr[r]; k < ptr[r + 1]; ++k) s = fma(val[k], x[idx[k]], s);
    y[r] = s;
}

constexpr int kDotThreads = 256;

// partial[b] = sum over the block's slice of (a*b) or (a*w)^2 when w != null (weighted norm^2)
__global__ void k_dot_partial(int n, const double* __restrict__ a, const double* __restrict__ b,
                              const double* __restrict__ w, double* __restrict__ partial) {
    __shared__ double red[kDotThreads / 32];
    double s = 0.0;
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
        if (w) {
            const double t = a[i] * w[i];
            s = fma(t, t, s);
        } else {
            s = fma(a[i], b[i], s);
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < kDotThreads / 32; ++q) t += red[q];
        partial[blockIdx.x] = t;
    }
}

__global__ void k_finish_sum(const double* __restrict__ partial, int nb, double* __restrict__ out) {
    __shared__ double red[32];
    double s = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) s += partial[i];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
    __syncthreads();
    if (threadIdx.x == 0) {
        double t = 0.0;
        for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) t += red[q];
        *out = t;
    }
}

__global__ void k_cgls_alpha(const double* gamma, const double* qq, double* alpha, int* brk) {
    const double g = *gamma, q = *qq;
    if (q == 0.0 || g == 0.0) {  // solve.cpp:54 breakdown
        *brk = 1;
        *alpha = 0.0;
    } else {
        *brk = 0;
        *alpha = g / q;
    }
}

__global__ void k_axpy_dev(int n, const double* __restrict__ alpha, double sgn, const double* __restrict__ x,
                           double* __restrict__ y) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) y[i] = fma(sgn * *alpha, x[i], y[i]);
}

__global__ void k_p_update(int n, const double* __restrict__ s, const double* gnew, const double* gold, double* __restrict__ p) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) p[i] = fma(*gnew / *gold, p[i], s[i]);
}

__global__ void k_copy(int n, const double* __restrict__ a, double* __restrict__ b) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) b[i] = a[i];
}

}  // namespace

namespace {
SmemCfg g_wsweep_cfg, g_wsweep_big_cfg;  // dynamic smem opted in so far (see prepare_wsweep)
}

void prepare_wsweep(int maxc, int bmaxc) {
    smem_optin(reinterpret_cast<const void*>(k_wsweep), sizeof(double) * static_cast<size_t>(std::max(maxc, 1)) * kWarpsPerBlock,
               g_wsweep_cfg);
    smem_optin(reinterpret_cast<const void*>(k_wsweep_big), sizeof(double) * static_cast<size_t>(std::max(bmaxc, 1)),
               g_wsweep_big_cfg);
}

static void wsweep(const WFac* f, int nf, double* z, double* contrib, int mode, int maxc, cudaStream_t st) {
    if (nf <= 0) return;
    const size_t smem = sizeof(double) * static_cast<size_t>(maxc > 0 ? maxc : 1) * kWarpsPerBlock;
    smem_optin(reinterpret_cast<const void*>(k_wsweep), smem, g_wsweep_cfg);
    k_wsweep<<<(nf + kWarpsPerBlock - 1) / kWarpsPerBlock, 32 * kWarpsPerBlock, smem, st>>>(f, nf, z, contrib, mode, maxc);
}

void launch_wsweep(const WFac* f, int nf, double* z, double* contrib, int mode, int maxc, cudaStream_t st) {
    wsweep(f, nf, z, contrib, mode, maxc, st);
}

void launch_wsweep_big(const WFac* f, int nf, double* z, double* contrib, int mode, int maxc, cudaStream_t st) {
    if (nf <= 0) return;
    const size_t smem = sizeof(double) * static_cast<size_t>(maxc > 0 ? maxc : 1);
    smem_optin(reinterpret_cast<const void*>(k_wsweep_big), smem, g_wsweep_big_cfg);
    k_wsweep_big<<<nf, kBigThreads, smem, st>>>(f, z, contrib, mode);
}

void launch_wreduce(const int* ptr, const int* idx, const int* col, int ncol, const double* contrib, double* z, double sgn,
                    cudaStream_t st) {
    if (ncol <= 0) return;
    k_wreduce<<<(ncol + 127) / 128, 128, 0, st>>>(ptr, idx, col, ncol, contrib, z, sgn);
}

void launch_spmv_csr(int m, const int* ptr, const int* idx, const double* val, const double* x, double* y, cudaStream_t st) {
    if (m <= 0) return;
    k_spmv_csr<<<(m + 255) / 256, 256, 0, st>>>(m, ptr, idx, val, x, y);
}

void launch_dot_partial(int n, const double* a, const double* b, const double* w, double* partial, int nblocks,
                        cudaStream_t st) {
    k_dot_partial<<<nblocks, kDotThreads, 0, st>>>(n, a, b, w, partial);
}

void launch_finish_sum(const double* partial, int nblocks, double* out, cudaStream_t st) {
    k_finish_sum<<<1, 256, 0, st>>>(partial, nblocks, out);
}

void launch_cgls_alpha(const double* gamma, const double* qq, double* alpha, int* brk, cudaStream_t st) {
    k_cgls_alpha<<<1, 1, 0, st>>>(gamma, qq, alpha, brk);
}

void launch_axpy_dev(int n, const double* alpha, double sgn, const double* x, double* y, cudaStream_t st) {
    if (n <= 0) return;
    k_axpy_dev<<<(n + 255) / 256, 256, 0, st>>>(n, alpha, sgn, x, y);
}

void launch_cgls_p_update(int n, const double* s, const double* gnew, const double* gold, double* p, cudaStream_t st) {
    if (n <= 0) return;
    k_p_update<<<(n + 255) / 256, 256, 0, st>>>(n, s, gnew, gold, p);
}

void launch_copy(int n, const double* a, double* b, cudaStream_t st) {
    if (n <= 0) return;
    k_copy<<<(n + 255) / 256, 256, 0, st>>>(n, a, b);
}

}  // namespace spqr
