// Batched FP64 front kernels for the spaQR factorization on B200 (sm_100a).
//
// One launch per engine phase covers every front of a stage.  The fronts at
// the BASELINE configs are tiny (median width 1-2 columns, tens of rows), so
// these kernels are latency/HBM bound: one CTA per problem, warp-per-column
// Householder updates with warp-shuffle reductions, columns addressed in
// place in HBM (L1/L2 resident at these sizes).  Reference semantics per
// kernel are cited next to each one (proj/src/dense_kernels.cpp).
#include <cfloat>
#include <climits>
#include <cmath>
#include <cstdio>

#include "dev.h"

namespace spqr {

namespace {

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
                           const int* __restrict__ segoff, const int* __restrict__ kmap, const AsmSrc* __restrict__ src) {
    // the destinations this block's elements fall in, found once per block; each thread then
    // searches only that (usually short) range
    __shared__ int s_lo, s_hi;
    const long long b0 = blockIdx.x * static_cast<long long>(blockDim.x);
    if (threadIdx.x < 2) {
        const long long t = threadIdx.x == 0 ? b0 : min(total - 1, b0 + blockDim.x - 1);
        int lo = 0, hi = ndst - 1;
        while (lo < hi) {
            const int mid = (lo + hi + 1) >> 1;
            if (dst[mid].elem_off <= t)
                lo = mid;
            else
                hi = mid - 1;
        }
        if (threadIdx.x == 0)
            s_lo = lo;
        else
            s_hi = lo;
    }
    __syncthreads();
    const long long e = b0 + threadIdx.x;
    if (e >= total) return;
    int lo = s_lo, hi = s_hi;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (dst[mid].elem_off <= e)
            lo = mid;
        else
            hi = mid - 1;
    }
    const AsmDst d = dst[lo];
    // 32-bit index arithmetic: one destination holds fewer than 2^31 elements
    const unsigned loc = static_cast<unsigned>(e - d.elem_off), nr = static_cast<unsigned>(d.nrows);
    const int j = static_cast<int>(loc / nr);
    const int i = static_cast<int>(loc - static_cast<unsigned>(j) * nr);
    const int* so = segoff + d.seg_off;
    int q = 0, qh = d.nseg - 1;
    while (q < qh) {
        const int mid = (q + qh + 1) >> 1;
        if (so[mid] <= j)
            q = mid;
        else
            qh = mid - 1;
    }
    const int o = j - so[q];
    const int* km = kmap + d.kmap_off + static_cast<long long>(q) * d.nsrc;
    const int4 rr = rowref[d.row_off + i];
    int t = -1, r = 0;
    if (rr.x == -2) {  // scan mode
        for (int s = 0; s < d.nsrc; ++s)
            if (km[s] != -1) {
                t = s;
                r = rr.y;
                break;
            }
    } else if (rr.x >= 0 && km[rr.x] != -1) {
        t = rr.x;
        r = rr.y;
    } else if (rr.z >= 0 && km[rr.z] != -1) {
        t = rr.z;
        r = rr.w;
    }
    double v = 0.0;
    if (t >= 0) {
        const int c = km[t];
        if (c >= 0) {
            const AsmSrc s = src[d.src_off + t];
            v = s.p[r * s.rs + static_cast<long long>(c + o) * s.cs];
        } else {
            v = (i == o) ? 1.0 : 0.0;  // identity segment
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
__global__ void k_stats_init(const StatDesc* __restrict__ ds, int nd, double* __restrict__ out_sq,
                             unsigned char* __restrict__ out_nz) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nd || ds[i].mode == 0) return;
    out_sq[ds[i].out_off] = 0.0;
    out_nz[ds[i].out_off] = ds[i].mode == 2 ? 1 : 0;
}

// byte-wide atomic OR / AND-NOT through the containing 32-bit word
__device__ __forceinline__ void byte_or(unsigned char* p, unsigned v) {
    const size_t a = reinterpret_cast<size_t>(p);
    atomicOr(reinterpret_cast<unsigned*>(a & ~size_t(3)), v << (8 * (a & 3)));
}
__device__ __forceinline__ void byte_clear(unsigned char* p) {
    const size_t a = reinterpret_cast<size_t>(p);
    atomicAnd(reinterpret_cast<unsigned*>(a & ~size_t(3)), ~(0xFFu << (8 * (a & 3))));
}

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
        const long long i = e - d.work_off;
        if (i >= d.nrows) return;  // alignment padding of a following warp-mode descriptor
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
        return;
    }
    // modes 1/2: the warp owns 256 consecutive elements (column-major in the block)
    const long long u = e - d.work_off;
    const long long nel = static_cast<long long>(d.nrows) * d.ncols;
    const long long base = (u >> 5) * 256;
    const int lane = static_cast<int>(u & 31);
    double mx = 0.0;
    bool nz = false, bad = false;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
        const long long t = base + lane + 32 * q;
        if (t >= nel) break;
        const int j = static_cast<int>(t / d.nrows), i = static_cast<int>(t - static_cast<long long>(j) * d.nrows);
        const double x = d.p[(d.r0 + i) + static_cast<long long>(d.c0 + j) * d.ld];
        mx = fmax(mx, fabs(x));
        nz |= (x != 0.0);
        bad |= (x != (i == j ? 1.0 : 0.0));  // exactly [I; 0]?  (Eigen isIdentity(0) / isZero(0), factorize.cpp:435)
    }
    // the whole warp belongs to this descriptor (32-aligned work_off)
    for (int o = 16; o > 0; o >>= 1) {
        mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    }
    nz = __any_sync(0xffffffffu, nz);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) {
        if (d.mode == 1) {
            if (mx > 0.0)
                atomicMax(reinterpret_cast<unsigned long long*>(out_sq + d.out_off), __double_as_longlong(mx));
            if (nz) byte_or(out_nz + d.out_off, 1u);
        } else if (bad) {
            byte_clear(out_nz + d.out_off);
        }
    }
}

// ------------------------------------------------------------------------ QR
// dense_kernels.cpp:11-35 + apply_reflectors_left_t (:96-99) on the trailing
// columns, fused: reflector k is applied to every column right of k (the QR
// trailing columns and the neighbour block X) in one right-looking sweep.
// The body runs on a block that is either staged in shared memory (most
// fronts: the whole m x ntot block fits) or addressed in place in HBM.
// Column updates are warp-per-column when m >= 32, else thread-per-column.
__device__ void qr_body(double* A, int ld, int m, int n, int nt, double* tau_out, double* s_neg_f, double* red,
                        double* s_sc) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool wide = m < 32;
    for (int k = 0; k < n; ++k) {
        double* ak = A + static_cast<long long>(k) * ld;
        double part = 0.0;
        for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) part = fma(ak[i], ak[i], part);
        const double tail2 = block_sum(part, red);
        if (threadIdx.x == 0) {
            const double c0 = ak[k];
            if (tail2 <= DBL_MIN) {  // Eigen makeHouseholder: tau = 0, beta = c0
                s_sc[0] = 0.0;
                s_sc[1] = 0.0;
            } else {
                double beta = sqrt(c0 * c0 + tail2);
                if (hh_beta_negative(c0, tail2)) beta = -beta;
                s_sc[1] = c0 - beta;
                s_sc[0] = (beta - c0) / beta;
                ak[k] = beta;
            }
        }
        __syncthreads();
        const double tau = s_sc[0], den = s_sc[1];
        for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) ak[i] = (tau == 0.0) ? 0.0 : ak[i] / den;
        __syncthreads();
        if (tau != 0.0) {
            if (wide) {
                for (int j = k + 1 + threadIdx.x; j < nt; j += blockDim.x) {
                    double* aj = A + static_cast<long long>(j) * ld;
                    double w = aj[k];
                    for (int i = k + 1; i < m; ++i) w = fma(ak[i], aj[i], w);
                    const double tw = tau * w;
                    aj[k] -= tw;
                    for (int i = k + 1; i < m; ++i) aj[i] = fma(-tw, ak[i], aj[i]);
                }
            } else {
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
        }
        if (threadIdx.x == 0 && tau_out) tau_out[k] = tau;
        __syncthreads();
    }
    // nonnegative diagonal: flip row i of R and of the updated neighbour block
    for (int i = threadIdx.x; i < n; i += blockDim.x) s_neg_f[i] = (A[i + static_cast<long long>(i) * ld] < 0.0) ? -1.0 : 1.0;
    __syncthreads();
    for (int j = threadIdx.x; j < nt; j += blockDim.x) {
        double* aj = A + static_cast<long long>(j) * ld;
        const int top = j < n ? j + 1 : n;
        for (int i = 0; i < top; ++i)
            if (s_neg_f[i] < 0.0) aj[i] = -aj[i];
    }
    __syncthreads();
}

__device__ void qr_epilogue(const QrDesc& d, double* A, int ld, const double* s_neg_f) {
    const int m = d.m, n = d.n;
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        const double r = A[i + static_cast<long long>(i) * ld];
        if (d.sign) d.sign[i] = s_neg_f[i];
        if (d.flag && !(fabs(r) >= DBL_MIN)) atomicMin(d.flag, i);  // first singular pivot
    }
    if (d.rout)
        for (int e = threadIdx.x; e < n * n; e += blockDim.x) {
            const int i = e % n, j = e / n;
            d.rout[e] = (i <= j) ? A[i + static_cast<long long>(j) * ld] : 0.0;
        }
    __syncthreads();
    if (d.zero_lower && !d.set_identity)
        for (int j = 0; j < n; ++j)
            for (int i = j + 1 + threadIdx.x; i < m; i += blockDim.x) A[i + static_cast<long long>(j) * ld] = 0.0;
    if (d.set_identity)
        for (int e = threadIdx.x; e < m * n; e += blockDim.x) {
            const int i = e % m, j = e / m;
            A[i + static_cast<long long>(j) * ld] = (i == j) ? 1.0 : 0.0;
        }
    __syncthreads();
}

constexpr int kQrMaxN = 1024;


__global__ void __launch_bounds__(256) k_qr_idx(const QrDesc* __restrict__ ds, const int* __restrict__ idx) {
    const QrDesc d = ds[idx[blockIdx.x]];
    __shared__ double red[32];
    __shared__ double s_sc[2];
    __shared__ double s_neg[kQrMaxN];
    qr_body(d.a, d.ld, d.m, d.n, d.ntot, d.tau, s_neg, red, s_sc);
    qr_epilogue(d, d.a, d.ld, s_neg);
}

// staged in shared memory (block + sign buffer), written back once
__global__ void __launch_bounds__(256) k_qr_smem(const QrDesc* __restrict__ ds, const int* __restrict__ idx) {
    const QrDesc d = ds[idx[blockIdx.x]];
    extern __shared__ double sm[];
    __shared__ double red[32];
    __shared__ double s_sc[2];
    const int m = d.m, nt = d.ntot;
    double* A = sm;
    double* s_neg = sm + static_cast<long long>(m) * nt;
    for (long long e = threadIdx.x; e < static_cast<long long>(m) * nt; e += blockDim.x) {
        const int i = static_cast<int>(e % m), j = static_cast<int>(e / m);
        A[e] = d.a[i + static_cast<long long>(j) * d.ld];
    }
    __syncthreads();
    qr_body(A, m, m, d.n, nt, d.tau, s_neg, red, s_sc);
    qr_epilogue(d, A, m, s_neg);
    for (long long e = threadIdx.x; e < static_cast<long long>(m) * nt; e += blockDim.x) {
        const int i = static_cast<int>(e % m), j = static_cast<int>(e / m);
        d.a[i + static_cast<long long>(j) * d.ld] = A[e];
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
// dense_kernels.cpp:124-232.  Logical column order is kept in ph[] (no data
// swaps); physical column = original column, so rows [0, rank) are R in the
// original order on exit.  First-max argmax (strict >) reproduces the
// reference's lowest-index tie break.  Column norms and updates are
// thread-per-column when m < 32 (interfaces are a few rows tall), else
// warp-per-column.
struct CpqrShared {
    double red[32];
    int redi[32];
    double r11, exact;
    int piv, stop;
};

__device__ double colnorm_seq(const double* a, int r0, int m) {
    double s = 0.0;
    for (int i = r0; i < m; ++i) s = fma(a[i], a[i], s);
    return sqrt(s);
}
__device__ double colnorm_warp(const double* a, int r0, int m) {
    double s = 0.0;
    for (int i = r0 + (threadIdx.x & 31); i < m; i += 32) s = fma(a[i], a[i], s);
    return sqrt(warp_sum(s));
}

__device__ int cpqr_argmax(const double* vn1, int k, int n, CpqrShared& S) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    double bv = -1.0;
    int bj = n;
    for (int j = k + threadIdx.x; j < n; j += blockDim.x) {
        const double v = vn1[j];
        if (v > bv) {
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
        S.red[wid] = bv;
        S.redi[wid] = bj;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double b = -1.0;
        int jj = n;
        for (int w = 0; w < nw; ++w)
            if (S.red[w] > b || (S.red[w] == b && S.redi[w] < jj)) {
                b = S.red[w];
                jj = S.redi[w];
            }
        S.piv = jj;
    }
    __syncthreads();
    return S.piv;
}

// A: m x n (ld), vn1/vn2/ph: n, sv: m.  Returns rank; R in rows [0, rank).
__device__ int cpqr_body(const CpqrDesc& d, double* A, int ld, double* vn1, double* vn2, int* ph, double* sv,
                         CpqrShared& S) {
    const int m = d.m, n = d.n, kmax = min(m, n);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    const bool wide = m < 32;
    const double tol3z = sqrt(DBL_EPSILON);
    if (wide) {
        for (int j = threadIdx.x; j < n; j += blockDim.x) {
            vn1[j] = vn2[j] = colnorm_seq(A + static_cast<long long>(j) * ld, 0, m);
            ph[j] = j;
        }
    } else {
        for (int j = wid; j < n; j += nw) {
            const double nr = colnorm_warp(A + static_cast<long long>(j) * ld, 0, m);
            if (lane == 0) {
                vn1[j] = vn2[j] = nr;
                ph[j] = j;
            }
        }
    }
    if (threadIdx.x == 0) S.r11 = 0.0;
    __syncthreads();
    int k = 0;
    while (k < kmax) {
        int piv = cpqr_argmax(vn1, k, n, S);
        if (threadIdx.x < 32) {
            const double* ap = A + static_cast<long long>(ph[piv]) * ld;
            const double ex = wide ? colnorm_seq(ap, k, m) : colnorm_warp(ap, k, m);
            if (threadIdx.x == 0) {
                S.exact = ex;
                S.stop = (k == 0) ? !(ex > 0.0) : (d.eps > 0.0 && ex < d.eps * S.r11);
            }
        }
        __syncthreads();
        if (S.stop && k > 0) {  // refresh every trailing norm and retry once
            if (wide) {
                for (int j = k + threadIdx.x; j < n; j += blockDim.x)
                    vn1[j] = vn2[j] = colnorm_seq(A + static_cast<long long>(ph[j]) * ld, k, m);
            } else {
                for (int j = k + wid; j < n; j += nw) {
                    const double nr = colnorm_warp(A + static_cast<long long>(ph[j]) * ld, k, m);
                    if (lane == 0) vn1[j] = vn2[j] = nr;
                }
            }
            __syncthreads();
            piv = cpqr_argmax(vn1, k, n, S);
            if (threadIdx.x == 0) {
                S.exact = vn1[piv];
                S.stop = d.eps > 0.0 && S.exact < d.eps * S.r11;
            }
            __syncthreads();
        }
        if (S.stop) break;
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
        double alpha = S.exact;
        const double x0 = ap[k];
        if (x0 > 0.0) alpha = -alpha;
        double part = 0.0;
        for (int i = threadIdx.x; i < len; i += blockDim.x) {
            const double vi = (i == 0) ? x0 - alpha : ap[k + i];
            sv[i] = vi;
            part = fma(vi, vi, part);
        }
        const double vns = block_sum(part, S.red);
        const double v0 = sv[0];
        if (d.V) {
            double* vk = d.V + static_cast<long long>(k) * d.ldv;
            for (int i = threadIdx.x; i < m; i += blockDim.x)
                vk[i] = (i < k) ? 0.0 : (i == k ? 1.0 : (vns > 0.0 ? sv[i - k] / v0 : 0.0));
        }
        if (vns > 0.0) {
            const double t = 2.0 / vns;
            if (wide) {
                for (int jl = k + 1 + threadIdx.x; jl < n; jl += blockDim.x) {
                    double* aj = A + static_cast<long long>(ph[jl]) * ld + k;
                    double w = 0.0;
                    for (int i = 0; i < len; ++i) w = fma(aj[i], sv[i], w);
                    const double tw = t * w;
                    for (int i = 0; i < len; ++i) aj[i] = fma(-tw, sv[i], aj[i]);
                }
            } else {
                for (int jl = k + 1 + wid; jl < n; jl += nw) {
                    double* aj = A + static_cast<long long>(ph[jl]) * ld + k;
                    double w = 0.0;
                    for (int i = lane; i < len; i += 32) w = fma(aj[i], sv[i], w);
                    const double tw = t * warp_sum(w);
                    for (int i = lane; i < len; i += 32) aj[i] = fma(-tw, sv[i], aj[i]);
                }
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
            if (k == 0) S.r11 = ap[0];
            if (d.perm) d.perm[k] = pc;
        }
        ++k;
        __syncthreads();
        if (k < kmax) {  // LAPACK-style downdate, recompute on cancellation
            if (wide) {
                for (int jl = k + threadIdx.x; jl < n; jl += blockDim.x) {
                    const double v1 = vn1[jl];
                    if (v1 == 0.0) continue;
                    const double* aj = A + static_cast<long long>(ph[jl]) * ld;
                    double tt = fabs(aj[k - 1]) / v1;
                    tt = fmax(0.0, (1.0 - tt) * (1.0 + tt));
                    const double ratio = v1 / vn2[jl];
                    if (tt * ratio * ratio <= tol3z)
                        vn1[jl] = vn2[jl] = colnorm_seq(aj, k, m);
                    else
                        vn1[jl] = v1 * sqrt(tt);
                }
            } else {
                for (int jl = k + wid; jl < n; jl += nw) {
                    const double v1 = vn1[jl];
                    if (v1 == 0.0) continue;
                    const double* aj = A + static_cast<long long>(ph[jl]) * ld;
                    double tt = fabs(aj[k - 1]) / v1;
                    tt = fmax(0.0, (1.0 - tt) * (1.0 + tt));
                    const double ratio = v1 / vn2[jl];
                    if (tt * ratio * ratio <= tol3z) {
                        const double nr = colnorm_warp(aj, k, m);
                        if (lane == 0) vn1[jl] = vn2[jl] = nr;
                    } else if (lane == 0) {
                        vn1[jl] = v1 * sqrt(tt);
                    }
                }
            }
            __syncthreads();
        }
    }
    return k;
}

// in place in HBM; scratch from d.work, reflector vector in dynamic smem
__global__ void __launch_bounds__(kCpqrThreads) k_cpqr(const CpqrDesc* __restrict__ ds, const int* __restrict__ idx) {
    const CpqrDesc d = ds[idx[blockIdx.x]];
    extern __shared__ double sv[];
    __shared__ CpqrShared S;
    const int n = d.n;
    if (min(d.m, n) == 0) {
        if (threadIdx.x == 0) {
            *d.rank = 0;
            *d.r11 = 0.0;
        }
        return;
    }
    const int r = cpqr_body(d, d.a, d.ld, d.work, d.work + n, reinterpret_cast<int*>(d.work + 2 * n), sv, S);
    if (threadIdx.x == 0) {
        *d.rank = r;
        *d.r11 = S.r11;
    }
}

// staged: A (m x n), vn1, vn2 (n), ph (n ints), v (m) all in shared memory;
// rows [0, rank) written back (the rest is never read by the engine)
__global__ void __launch_bounds__(kCpqrThreads) k_cpqr_smem(const CpqrDesc* __restrict__ ds, const int* __restrict__ idx) {
    const CpqrDesc d = ds[idx[blockIdx.x]];
    extern __shared__ double sm[];
    __shared__ CpqrShared S;
    const int m = d.m, n = d.n;
    if (min(m, n) == 0) {
        if (threadIdx.x == 0) {
            *d.rank = 0;
            *d.r11 = 0.0;
        }
        return;
    }
    double* A = sm;
    double* vn1 = A + static_cast<long long>(m) * n;
    double* vn2 = vn1 + n;
    double* sv = vn2 + n;
    int* ph = reinterpret_cast<int*>(sv + m);
    for (long long e = threadIdx.x; e < static_cast<long long>(m) * n; e += blockDim.x) {
        const int i = static_cast<int>(e % m), j = static_cast<int>(e / m);
        A[e] = d.a[i + static_cast<long long>(j) * d.ld];
    }
    __syncthreads();
    const int r = cpqr_body(d, A, m, vn1, vn2, ph, sv, S);
    for (long long e = threadIdx.x; e < static_cast<long long>(r) * n; e += blockDim.x) {
        const int i = static_cast<int>(e % r), j = static_cast<int>(e / r);
        d.a[i + static_cast<long long>(j) * d.ld] = A[i + static_cast<long long>(j) * m];
    }
    if (threadIdx.x == 0) {
        *d.rank = r;
        *d.r11 = S.r11;
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

void launch_assemble(const AsmDst* d_dst, int ndst, long long total, const int4* d_rowref, const int* d_segoff,
                     const int* d_kmap, const AsmSrc* d_src, cudaStream_t st) {
    if (total <= 0 || ndst <= 0) return;
    const int bs = 256;
    k_assemble<<<static_cast<unsigned>((total + bs - 1) / bs), bs, 0, st>>>(d_dst, ndst, total, d_rowref, d_segoff, d_kmap,
                                                                          d_src);
}

void launch_scatter_values(const long long* off, const double* val, long long n, double* base, cudaStream_t st) {
    if (n <= 0) return;
    k_scatter<<<static_cast<unsigned>((n + 255) / 256), 256, 0, st>>>(off, val, n, base);
}

void launch_stats(const StatDesc* d, int nd, long long total, double* out_sq, unsigned char* out_nz, cudaStream_t st) {
    if (total <= 0 || nd <= 0) return;
    const int bs = 128;
    k_stats_init<<<(nd + 255) / 256, 256, 0, st>>>(d, nd, out_sq, out_nz);
    k_stats<<<static_cast<unsigned>((total + bs - 1) / bs), bs, 0, st>>>(d, nd, total, out_sq, out_nz);
}


void launch_qr_split(const QrDesc* d_desc, const int* d_small, int n_small, size_t smem_small, const int* d_large,
                     int n_large, cudaStream_t st) {
    if (n_small > 0) {
        static SmemCfg cfg;
        smem_optin(reinterpret_cast<const void*>(k_qr_smem), smem_small, cfg);
        k_qr_smem<<<n_small, 256, smem_small, st>>>(d_desc, d_small);
    }
    if (n_large > 0) k_qr_idx<<<n_large, 256, 0, st>>>(d_desc, d_large);
}

void launch_trsm(const TrsmDesc* d, int nd, long long total, cudaStream_t st) {
    if (total <= 0 || nd <= 0) return;
    const int bs = 128;
    k_trsm<<<static_cast<unsigned>((total + bs - 1) / bs), bs, 0, st>>>(d, nd, total);
}

void launch_cpqr_split(const CpqrDesc* d_desc, const int* d_small, int n_small, size_t smem_small, const int* d_large,
                       int n_large, int max_m_large, cudaStream_t st) {
    if (n_small > 0) {
        static SmemCfg cfg;
        smem_optin(reinterpret_cast<const void*>(k_cpqr_smem), smem_small, cfg);
        k_cpqr_smem<<<n_small, kCpqrThreads, smem_small, st>>>(d_desc, d_small);
    }
    if (n_large > 0) {
        const size_t smem = sizeof(double) * static_cast<size_t>(max_m_large > 0 ? max_m_large : 1);
        static SmemCfg cfg;
        smem_optin(reinterpret_cast<const void*>(k_cpqr), smem, cfg);
        k_cpqr<<<n_large, kCpqrThreads, smem, st>>>(d_desc, d_large);
    }
}

namespace {
__global__ void k_info_fixup(int* info, int n) {
    const int i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n && info[i] == INT_MAX) info[i] = -1;
}
}  // namespace

// QR flags are atomicMin'd from INT_MAX: map "no singular pivot" to the C ABI's -1
void launch_info_fixup(int* info, int n, cudaStream_t st) {
    if (n > 0) k_info_fixup<<<(n + 255) / 256, 256, 0, st>>>(info, n);
}

namespace {
// store_q (factorize.cpp:324-330, :483, :514-519): copy the reflectors a QR left below the
// diagonal of src(:, :n) into dst (m x n, ld m, explicit unit diagonal, zeros above — the
// layout the rotation sweeps read), then restore what the non-store_q launch would have left:
// the lower part cleared (VCOPY_ZERO_LOWER) or the block set to [I; 0] (VCOPY_SET_IDENTITY).
// One CTA per block; each element is read, copied and rewritten by one thread.
__global__ void k_vcopy(const VCopyDesc* __restrict__ ds) {
    const VCopyDesc d = ds[blockIdx.x];
    const long long total = static_cast<long long>(d.m) * d.n;
    for (long long e = threadIdx.x; e < total; e += blockDim.x) {
        const int j = static_cast<int>(e / d.m), i = static_cast<int>(e - static_cast<long long>(j) * d.m);
        double* sp = d.src + static_cast<long long>(j) * d.lds + i;
        d.dst[static_cast<long long>(j) * d.m + i] = i > j ? *sp : (i == j ? 1.0 : 0.0);
        if ((d.mode & VCOPY_ZERO_LOWER) && i > j) *sp = 0.0;
        if (d.mode & VCOPY_SET_IDENTITY) *sp = (i == j) ? 1.0 : 0.0;
    }
}
}  // namespace

void launch_vcopy(const VCopyDesc* d, int nd, cudaStream_t st) {
    if (nd > 0) k_vcopy<<<nd, 256, 0, st>>>(d);
}

}  // namespace spqr
