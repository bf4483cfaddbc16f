// Batched FP64 front kernels for the spaQR factorization on B200 (sm_100a).
//
// One launch per engine phase covers every front of a stage.  The fronts at
// the BASELINE configs are tiny (median width 1-2 columns, tens of rows), so
// these kernels are latency/HBM bound: one CTA per problem, warp-per-column
// Householder updates with warp-shuffle reductions, columns addressed in
// place in HBM (L1/L2 resident at these sizes).  Reference semantics per
// kernel are cited next to each one (proj/src/dense_kernels.cpp).
#include <cfloat>
#include <cmath>
#include <cstdio>

#include "dev.h"

namespace spqr {

namespace {

constexpr int kQrThreads = 128;
constexpr int kCpqrThreads = 256;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

// Block-wide sum; every thread gets the result.  red must hold 32 doubles.
__device__ double block_sum(double v, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    v = warp_sum(v);
    __syncthreads();
    if (lane == 0) red[wid] = v;
    __syncthreads();
    double s = 0.0;
    for (int w = 0; w < nw; ++w) s += red[w];
    return s;
}

// ------------------------------------------------------------------ assemble
__global__ void k_assemble(const AsmDst* __restrict__ dst, int ndst, long long total, const int4* __restrict__ rowref,
                           const int* __restrict__ cmap, const AsmSrc* __restrict__ src) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= total) return;
    int lo = 0, hi = ndst - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (dst[mid].elem_off <= e)
            lo = mid;
        else
            hi = mid - 1;
    }
    const AsmDst d = dst[lo];
    const long long loc = e - d.elem_off;
    const int i = static_cast<int>(loc % d.nrows);
    const int j = static_cast<int>(loc / d.nrows);
    const int4 rr = rowref[d.row_off + i];
    const int* cm = cmap + d.cmap_off + static_cast<long long>(j) * d.nsrc;
    double v = 0.0;
    if (rr.x == -2) {  // scan mode: first slot with a mapping for column j, row rr.y in every slot
        for (int t = 0; t < d.nsrc; ++t) {
            const int c = cm[t];
            if (c >= 0) {
                const AsmSrc s = src[d.src_off + t];
                v = s.p[rr.y * s.rs + c * s.cs];
                break;
            }
            if (c <= -2) {  // identity column: 1 on row (-c-2)
                v = (i == -c - 2) ? 1.0 : 0.0;
                break;
            }
        }
    } else {
        int c = -1, t = -1, r = 0;
        if (rr.x >= 0 && cm[rr.x] != -1) {
            t = rr.x;
            r = rr.y;
        } else if (rr.z >= 0 && cm[rr.z] != -1) {
            t = rr.z;
            r = rr.w;
        }
        if (t >= 0) {
            c = cm[t];
            if (c >= 0) {
                const AsmSrc s = src[d.src_off + t];
                v = s.p[r * s.rs + c * s.cs];
            } else {
                v = (i == -c - 2) ? 1.0 : 0.0;
            }
        }
    }
    if (d.trans)
        d.p[j + static_cast<long long>(i) * d.ld] = v;
    else
        d.p[i + static_cast<long long>(j) * d.ld] = v;
}

// init scatter of A's values into the leaf fronts (factorize.cpp:77-81)
__global__ void k_scatter(const long long* __restrict__ off, const double* __restrict__ val, long long n, double* base) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e < n) base[off[e]] = val[e];
}

// --------------------------------------------------------------------- stats
__global__ void k_stats(const StatDesc* __restrict__ ds, int nd, long long total, double* __restrict__ out_sq,
                        unsigned char* __restrict__ out_nz) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= total) return;
    int lo = 0, hi = nd - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ds[mid].work_off <= e)
            lo = mid;
        else
            hi = mid - 1;
    }
    const StatDesc d = ds[lo];
    if (d.mode == 0) {
        const int i = static_cast<int>(e - d.work_off);
        const double* a = d.p + (d.r0 + i) + static_cast<long long>(d.c0) * d.ld;
        double s = 0.0;
        unsigned char nz = 0;
        for (int j = 0; j < d.ncols; ++j) {
            const double x = a[static_cast<long long>(j) * d.ld];
            s = fma(x, x, s);
            nz |= (x != 0.0);
        }
        out_sq[d.out_off + i] = s;
        out_nz[d.out_off + i] = nz;
    } else if (d.mode == 2) {  // exactly [I; 0]?  (Eigen isIdentity(0) / isZero(0), factorize.cpp:435)
        unsigned char ok = 1;
        for (int j = 0; j < d.ncols && ok; ++j)
            for (int i = 0; i < d.nrows; ++i)
                if (d.p[(d.r0 + i) + static_cast<long long>(d.c0 + j) * d.ld] != (i == j ? 1.0 : 0.0)) {
                    ok = 0;
                    break;
                }
        out_sq[d.out_off] = 0.0;
        out_nz[d.out_off] = ok;
    } else {
        double mx = 0.0;
        unsigned char nz = 0;
        for (int j = 0; j < d.ncols; ++j)
            for (int i = 0; i < d.nrows; ++i) {
                const double x = d.p[(d.r0 + i) + static_cast<long long>(d.c0 + j) * d.ld];
                mx = fmax(mx, fabs(x));
                nz |= (x != 0.0);
            }
        out_sq[d.out_off] = mx;
        out_nz[d.out_off] = nz;
    }
}

// ------------------------------------------------------------------------ QR
// dense_kernels.cpp:11-35 + apply_reflectors_left_t (:96-99) on the trailing
// columns, fused: reflector k is applied to every column right of k (the QR
// trailing columns and the neighbour block X) in one right-looking sweep.
__global__ void __launch_bounds__(kQrThreads) k_qr(const QrDesc* __restrict__ ds) {
    const QrDesc d = ds[blockIdx.x];
    __shared__ double red[32];
    __shared__ double s_tau, s_den;
    __shared__ signed char s_neg[1024];
    const int m = d.m, n = d.n, nt = d.ntot, ld = d.ld;
    double* A = d.a;
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int k = 0; k < n; ++k) {
        double* ak = A + static_cast<long long>(k) * ld;
        double part = 0.0;
        for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) part = fma(ak[i], ak[i], part);
        const double tail2 = block_sum(part, red);
        if (threadIdx.x == 0) {
            const double c0 = ak[k];
            if (tail2 <= DBL_MIN) {  // Eigen makeHouseholder: tau = 0, beta = c0
                s_tau = 0.0;
                s_den = 0.0;
            } else {
                double beta = sqrt(c0 * c0 + tail2);
                if (c0 >= 0.0) beta = -beta;
                s_den = c0 - beta;
                s_tau = (beta - c0) / beta;
                ak[k] = beta;
            }
        }
        __syncthreads();
        const double tau = s_tau, den = s_den;
        for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) ak[i] = (tau == 0.0) ? 0.0 : ak[i] / den;
        __syncthreads();
        if (tau != 0.0) {
            for (int j = k + 1 + wid; j < nt; j += nw) {
                double* aj = A + static_cast<long long>(j) * ld;
                double w = 0.0;
                for (int i = k + 1 + lane; i < m; i += 32) w = fma(ak[i], aj[i], w);
                w = warp_sum(w) + aj[k];
                const double tw = tau * w;
                for (int i = k + 1 + lane; i < m; i += 32) aj[i] = fma(-tw, ak[i], aj[i]);
                if (lane == 0) aj[k] -= tw;
            }
        }
        if (threadIdx.x == 0 && d.tau) d.tau[k] = tau;
        __syncthreads();
    }
    // nonnegative diagonal: flip row i of R and of the updated neighbour block
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double r = A[i + static_cast<long long>(i) * ld];
        s_neg[i] = (r < 0.0);
        if (d.sign) d.sign[i] = (r < 0.0) ? -1.0 : 1.0;
        if (d.flag && !(fabs(r) >= DBL_MIN)) atomicMin(d.flag, i);  // first singular pivot
    }
    __syncthreads();
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
        double* aj = A + static_cast<long long>(j) * ld;
        const int top = j < n ? j + 1 : n;
        for (int i = 0; i < top; ++i)
            if (s_neg[i]) aj[i] = -aj[i];
    }
    __syncthreads();
    if (d.rout)
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
            const int i = e % n, j = e / n;
            d.rout[e] = (i <= j) ? A[i + static_cast<long long>(j) * ld] : 0.0;
        }
    if (d.zero_lower && !d.set_identity) {
        __syncthreads();
        for (int j = 0; j < n; ++j)
            for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) A[i + static_cast<long long>(j) * ld] = 0.0;
    }
    if (d.set_identity) {
        __syncthreads();
        for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
            const int i = e % m, j = e / m;
            A[i + static_cast<long long>(j) * ld] = (i == j) ? 1.0 : 0.0;
        }
    }
}

// ---------------------------------------------------------------------- TRSM
__global__ void k_trsm(const TrsmDesc* __restrict__ ds, int nd, long long total) {
    const long long e = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
    if (e >= total) return;
    int lo = 0, hi = nd - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (ds[mid].work_off <= e)
            lo = mid;
        else
            hi = mid - 1;
    }
    const TrsmDesc d = ds[lo];
    double* b = d.b + (e - d.work_off);
    for (int j = 0; j < d.n; ++j) {  // x U = b, dense_kernels.cpp:242-257 (Right, no transpose)
        double s = b[static_cast<long long>(j) * d.ldb];
        for (int i = 0; i < j; ++i) s = fma(-b[static_cast<long long>(i) * d.ldb], d.r[i + static_cast<long long>(j) * d.ldr], s);
        b[static_cast<long long>(j) * d.ldb] = s / d.r[j + static_cast<long long>(j) * d.ldr];
    }
}

// ---------------------------------------------------------------------- CPQR
__device__ double col_norm_from(const double* a, int r0, int m) {  // per warp
    double s = 0.0;
    for (int i = r0 + (threadIdx.x & 31); i < m; i += 32) s = fma(a[i], a[i], s);
    return sqrt(warp_sum(s));
}

// dense_kernels.cpp:124-232.  Logical column order is kept in ph[] (no data
// swaps); physical column = original column, so rows [0, rank) are R in the
// original order on exit.  First-max argmax (strict >) reproduces the
// reference's lowest-index tie break.
__global__ void __launch_bounds__(kCpqrThreads) k_cpqr(const CpqrDesc* __restrict__ ds) {
    const CpqrDesc d = ds[blockIdx.x];
    extern __shared__ double sv[];  // reflector vector, m entries
    __shared__ double red[32];
    __shared__ int redi[32];
    __shared__ double s_r11, s_exact;
    __shared__ int s_piv, s_stop;
    const int m = d.m, n = d.n, ld = d.ld, kmax = min(m, n);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double* A = d.a;
    double* vn1 = d.work;
    double* vn2 = d.work + n;
    int* ph = reinterpret_cast<int*>(d.work + 2 * n);
    if (kmax == 0) {
        if (threadIdx.x == 0) {
            *d.rank = 0;
            *d.r11 = 0.0;
        }
        return;
    }
    const double tol3z = sqrt(DBL_EPSILON);
    for (int j = wid; j < n; j += nw) {
        const double nr = col_norm_from(A + static_cast<long long>(j) * ld, 0, m);
        if (lane == 0) {
            vn1[j] = vn2[j] = nr;
            ph[j] = j;
        }
    }
    if (threadIdx.x == 0) s_r11 = 0.0;
    __syncthreads();

    auto argmax_from = [&](int k) {  // first maximum of vn1[k..n)
        double bv = -1.0;
        int bj = n;
        for (int j = k + threadIdx.x; j < n; j += blockDim.x) {
            const double v = vn1[j];
            if (v > bv || (v == bv && j < bj)) {
                bv = v;
                bj = j;
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            if (ov > bv || (ov == bv && oj < bj)) {
                bv = ov;
                bj = oj;
            }
        }
        __syncthreads();
        if (lane == 0) {
            red[wid] = bv;
            redi[wid] = bj;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            double b = -1.0;
            int jj = n;
            for (int w = 0; w < nw; ++w)
                if (red[w] > b || (red[w] == b && redi[w] < jj)) {
                    b = red[w];
                    jj = redi[w];
                }
            s_piv = jj;
        }
        __syncthreads();
        return s_piv;
    };

    int k = 0;
    while (k < kmax) {
        int piv = argmax_from(k);
        if (wid == 0) {
            const double ex = col_norm_from(A + static_cast<long long>(ph[piv]) * ld, k, m);
            if (lane == 0) {
                s_exact = ex;
                s_stop = (k == 0) ? !(ex > 0.0) : (d.eps > 0.0 && ex < d.eps * s_r11);
            }
        }
        __syncthreads();
        if (s_stop && k > 0) {  // refresh every trailing norm and retry once
            for (int j = k + wid; j < n; j += nw) {
                const double nr = col_norm_from(A + static_cast<long long>(ph[j]) * ld, k, m);
                if (lane == 0) vn1[j] = vn2[j] = nr;
            }
            __syncthreads();
            piv = argmax_from(k);
            if (threadIdx.x == 0) {
                s_exact = vn1[piv];
                s_stop = d.eps > 0.0 && s_exact < d.eps * s_r11;
            }
            __syncthreads();
        }
        if (s_stop) break;
        if (threadIdx.x == 0 && piv != k) {
            const int t = ph[piv];
            ph[piv] = ph[k];
            ph[k] = t;
            double x = vn1[piv];
            vn1[piv] = vn1[k];
            vn1[k] = x;
            x = vn2[piv];
            vn2[piv] = vn2[k];
            vn2[k] = x;
        }
        __syncthreads();
        const int pc = ph[k];
        double* ap = A + static_cast<long long>(pc) * ld;
        const int len = m - k;
        // Householder: alpha = -sign+(x0)||x||, v = x - alpha e1, tau = 2/||v||^2
        double alpha = s_exact;
        const double x0 = ap[k];
        if (x0 > 0.0) alpha = -alpha;
        double part = 0.0;
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            const double vi = (i == 0) ? x0 - alpha : ap[k + i];
            sv[i] = vi;
            part = fma(vi, vi, part);
        }
        const double vns = block_sum(part, red);  // syncs: sv visible
        const double v0 = sv[0];
        if (d.V) {
            double* vk = d.V + static_cast<long long>(k) * d.ldv;
            for (int i = threadIdx.x; i < m; i += blockDim.x)
                vk[i] = (i < k) ? 0.0 : (i == k ? 1.0 : (vns > 0.0 ? sv[i - k] / v0 : 0.0));
        }
        if (vns > 0.0) {
            const double t = 2.0 / vns;
            for (int jl = k + 1 + wid; jl < n; jl += nw) {
                double* aj = A + static_cast<long long>(ph[jl]) * ld + k;
                double w = 0.0;
                for (int i = lane; i < len; i += 32) w = fma(aj[i], sv[i], w);
                const double tw = t * warp_sum(w);
                for (int i = lane; i < len; i += 32) aj[i] = fma(-tw, sv[i], aj[i]);
            }
            __syncthreads();
            for (int i = threadIdx.x; i < len; i += blockDim.x) ap[k + i] = (i == 0) ? alpha : 0.0;
            if (threadIdx.x == 0 && d.tau) d.tau[k] = t * v0 * v0;
        } else if (threadIdx.x == 0 && d.tau) {
            d.tau[k] = 0.0;
        }
        __syncthreads();
        const bool neg = ap[k] < 0.0;
        if (neg)
            for (int jl = k + threadIdx.x; jl < n; jl += blockDim.x) {
                double* x = A + static_cast<long long>(ph[jl]) * ld + k;
                *x = -*x;
            }
        __syncthreads();
        if (threadIdx.x == 0) {
            if (d.sign) d.sign[k] = neg ? -1.0 : 1.0;
            if (k == 0) s_r11 = ap[0];
            if (d.perm) d.perm[k] = pc;
        }
        ++k;
        __syncthreads();
        if (k < kmax) {  // LAPACK-style downdate, recompute on cancellation
            for (int jl = k + wid; jl < n; jl += nw) {
                const double v1 = vn1[jl];
                if (v1 == 0.0) continue;
                double* aj = A + static_cast<long long>(ph[jl]) * ld;
                double tt = fabs(aj[k - 1]) / v1;
                tt = fmax(0.0, (1.0 - tt) * (1.0 + tt));
                const double ratio = v1 / vn2[jl];
                if (tt * ratio * ratio <= tol3z) {
                    const double nr = col_norm_from(aj, k, m);
                    if (lane == 0) vn1[jl] = vn2[jl] = nr;
                } else if (lane == 0) {
                    vn1[jl] = v1 * sqrt(tt);
                }
            }
            __syncthreads();
        }
    }
    if (threadIdx.x == 0) {
        *d.rank = k;
        *d.r11 = s_r11;
    }
}

}  // namespace

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
        if (n <= 0) n = 148;
    }
    return n;
}

void launch_assemble(const AsmDst* d_dst, int ndst, long long total, const int4* d_rowref, const int* d_cmap,
                     const AsmSrc* d_src, cudaStream_t st) {
    if (total <= 0 || ndst <= 0) return;
    const int bs = 256;
    k_assemble<<<static_cast<unsigned>((total + bs - 1) / bs), bs, 0, st>>>(d_dst, ndst, total, d_rowref, d_cmap, d_src);
}

void launch_scatter_values(const long long* off, const double* val, long long n, double* base, cudaStream_t st) {
    if (n <= 0) return;
    k_scatter<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(off, val, n, base);
}

void launch_stats(const StatDesc* d, int nd, long long total, double* out_sq, unsigned char* out_nz, cudaStream_t st) {
    if (total <= 0 || nd <= 0) return;
    const int bs = 128;
    k_stats<<<static_cast<unsigned>((total + bs - 1) / bs), bs, 0, st>>>(d, nd, total, out_sq, out_nz);
}

void launch_qr(const QrDesc* d, int nd, int /*max_m*/, cudaStream_t st) {
    if (nd <= 0) return;
    k_qr<<<nd, kQrThreads, 0, st>>>(d);
}

void launch_trsm(const TrsmDesc* d, int nd, long long total, cudaStream_t st) {
    if (total <= 0 || nd <= 0) return;
    const int bs = 128;
    k_trsm<<<static_cast<unsigned>((total + bs - 1) / bs), bs, 0, st>>>(d, nd, total);
}

void launch_cpqr(const CpqrDesc* d, int nd, int max_m, cudaStream_t st) {
    if (nd <= 0) return;
    const size_t smem = sizeof(double) * static_cast<size_t>(max_m > 0 ? max_m : 1);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_cpqr, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    k_cpqr<<<nd, kCpqrThreads, smem, st>>>(d);
}

}  // namespace spqr
