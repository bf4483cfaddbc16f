// Truncated CPQR for short-wide interface blocks (m <= 128 rows, n <= 2048).
//
// Semantics: truncated_cpqr (proj/src/dense_kernels.cpp:124-232), exactly as
// cpqr_body in kernels.cu — greedy column-norm pivoting (first maximum by
// logical position), exact-norm stop rule with one refresh and retry,
// Householder alpha = -sign+(x0)||x||, nonnegative diagonal flip, LAPACK-style
// norm downdate with recompute below sqrt(eps).
//
// The sparsify_cols blocks G = [B^T | own rows] are a few interface columns
// tall and hundreds of rows wide; one CTA per problem, the block staged in
// shared memory (odd leading dimension: conflict-free column walks).  Thread t
// owns physical columns t, t+256, ...; their logical positions and downdated
// norms live in registers.  Per pivot step there is one block barrier (argmax
// partials, double-buffered); every warp then recomputes the same pivot norm
// and Householder vector from shared memory with warp shuffles (lane = row),
// so no further block synchronisation is needed.  Each thread updates its own
// trailing columns serially over the m rows.  The pivot column is finalised
// by its owner one step later, after the barrier that proves every warp has
// read it.
#include <cfloat>
#include <climits>
#include <cmath>

#include "dev.h"

namespace spqr {

namespace {

constexpr int kThreads = 256;
constexpr int kNW = kThreads / 32;
constexpr size_t kNarrowSmem = 216 * 1024;  // dynamic smem cap (227 KB minus up to 9 KB of static arrays)

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

__device__ __forceinline__ bool better(double v, int j, double bv, int bj) { return v > bv || (v == bv && j < bj); }

// GLB: the block stays in place in global memory (L1/L2 serve the per-thread
// column walks) when it is too large to stage in shared memory.
// NC: owned columns per thread (n <= 256 NC)
template <int RPL, bool GLB, int NC>
__global__ void __launch_bounds__(kThreads) k_cpqr_narrow(const CpqrDesc* __restrict__ ds, const int* __restrict__ idx) {
    const CpqrDesc d = ds[idx[blockIdx.x]];
    const int m = d.m, n = d.n, kmax = min(m, n);
    const long long ldm = GLB ? d.ld : (m | 1);
    extern __shared__ double sA[];  // ldm x n when staged
    double* A = GLB ? d.a : sA;
    __shared__ double vbuf[kNW][32 * RPL];
    __shared__ double pv[2][kNW];
    __shared__ int pj[2][kNW], pp[2][kNW];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (kmax == 0) {
        if (tid == 0) {
            *d.rank = 0;
            *d.r11 = 0.0;
        }
        return;
    }
    if (!GLB) {  // stage the block, eight loads in flight per thread
        const int tot = m * n;
        for (int e0 = tid; e0 < tot; e0 += 8 * kThreads) {
            double v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * kThreads;
                const int j = e / m, i = e - j * m;
                v[u] = e < tot ? d.a[i + static_cast<long long>(j) * d.ld] : 0.0;
            }
#pragma unroll
            for (int u = 0; u < 8; ++u) {
                const int e = e0 + u * kThreads;
                const int j = e / m, i = e - j * m;
                if (e < tot) A[i + j * ldm] = v[u];
            }
        }
        __syncthreads();
    }
    const double tol3z = sqrt(DBL_EPSILON);
    double vn1[NC], vn2[NC];
    int lpos[NC];
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int p = tid + kThreads * c;
        lpos[c] = p < n ? p : INT_MAX;
        double s = 0.0;
        if (p < n)
            for (int i = 0; i < m; ++i) s = fma(A[i + p * ldm], A[i + p * ldm], s);
        vn1[c] = vn2[c] = p < n ? sqrt(s) : -1.0;
    }
    int buf = 0;
    // grid of the CTA: first max of vn1 over logical positions >= k0 -> (value, position, physical)
    auto argmax = [&](int k0, double& bv, int& bj, int& bp) {
        bv = -1.0;
        bj = INT_MAX;
        bp = -1;
#pragma unroll
        for (int c = 0; c < NC; ++c)
            if (lpos[c] >= k0 && lpos[c] != INT_MAX && better(vn1[c], lpos[c], bv, bj)) {
                bv = vn1[c];
                bj = lpos[c];
                bp = tid + kThreads * c;
            }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            const int op = __shfl_xor_sync(0xffffffffu, bp, o);
            if (better(ov, oj, bv, bj)) {
                bv = ov;
                bj = oj;
                bp = op;
            }
        }
        if (lane == 0) {
            pv[buf][wid] = bv;
            pj[buf][wid] = bj;
            pp[buf][wid] = bp;
        }
        __syncthreads();
        bv = -1.0;
        bj = INT_MAX;
        bp = -1;
#pragma unroll
        for (int w = 0; w < kNW; ++w)
            if (better(pv[buf][w], pj[buf][w], bv, bj)) {
                bv = pv[buf][w];
                bj = pj[buf][w];
                bp = pp[buf][w];
            }
        buf ^= 1;
    };
    // sum over rows [r0, m) of column p squared, lane = row (every warp the same)
    auto tail_sumsq = [&](int p, int r0) {
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            const int i = lane + 32 * q;
            if (i >= r0 && i < m) s = fma(A[i + p * ldm], A[i + p * ldm], s);
        }
        return wsum(s);
    };

    double r11 = 0.0;
    int k = 0;
    int prev_pc = -1, prev_k = -1;
    double prev_alpha = 0.0;
    bool prev_reflect = false, prev_flip = false;
    auto finalise = [&]() {  // owner thread writes alpha e1 into the previous pivot column
        if (prev_pc >= 0 && prev_pc % kThreads == tid) {
            double* ap = A + prev_pc * ldm;
            if (prev_reflect) {
                ap[prev_k] = prev_flip ? -prev_alpha : prev_alpha;
                for (int i = prev_k + 1; i < m; ++i) ap[i] = 0.0;
            } else if (prev_flip) {
                ap[prev_k] = -ap[prev_k];
            }
        }
        prev_pc = -1;
    };
    while (k < kmax) {
        double bv;
        int piv, pc;
        argmax(k, bv, piv, pc);
        finalise();
        double x0 = A[k + pc * ldm];
        double tail = tail_sumsq(pc, k + 1);
        double exact = sqrt(fma(x0, x0, tail));
        bool stop = (k == 0) ? !(exact > 0.0) : (d.eps > 0.0 && exact < d.eps * r11);
        if (stop && k > 0) {  // refresh every trailing norm and retry once
#pragma unroll
            for (int c = 0; c < NC; ++c) {
                if (lpos[c] == INT_MAX || lpos[c] < k) continue;
                const double* a = A + (tid + kThreads * c) * ldm;
                double s = 0.0;
                for (int i = k; i < m; ++i) s = fma(a[i], a[i], s);
                vn1[c] = vn2[c] = sqrt(s);
            }
            argmax(k, bv, piv, pc);
            exact = bv;
            stop = d.eps > 0.0 && exact < d.eps * r11;
            if (!stop) {
                x0 = A[k + pc * ldm];
                tail = tail_sumsq(pc, k + 1);
            }
        }
        if (stop) break;
        // Householder on rows [k, m) of the pivot column (every warp, lane = row)
        double alpha = sqrt(fma(x0, x0, tail));
        if (x0 > 0.0) alpha = -alpha;
        const double v0 = x0 - alpha;
        const double vns = fma(v0, v0, tail);
        const bool reflect = vns > 0.0;
        const double t = reflect ? 2.0 / vns : 0.0;
        const bool flip = (reflect ? alpha : x0) < 0.0;
        __syncwarp();
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            const int i = lane + 32 * q;
            vbuf[wid][i] = (i < k || i >= m) ? 0.0 : (i == k ? v0 : A[i + pc * ldm]);
        }
        __syncwarp();
        if (wid == 0 && d.V) {
            double* vk = d.V + static_cast<long long>(k) * d.ldv;
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int i = lane + 32 * q;
                if (i < m) vk[i] = i < k ? 0.0 : (i == k ? 1.0 : (reflect ? vbuf[0][i] / v0 : 0.0));
            }
        }
        if (tid == 0) {
            if (d.tau) d.tau[k] = reflect ? t * v0 * v0 : 0.0;
            if (d.sign) d.sign[k] = flip ? -1.0 : 1.0;
            if (d.perm) d.perm[k] = pc;
        }
        if (k == 0) r11 = fabs(reflect ? alpha : x0);
        // logical swap k <-> piv, then the owned trailing columns
        const double* v = vbuf[wid];
#pragma unroll
        for (int c = 0; c < NC; ++c) {
            const int p = tid + kThreads * c;
            if (lpos[c] == INT_MAX) continue;
            lpos[c] = p == pc ? k : (lpos[c] == k ? piv : lpos[c]);
            if (lpos[c] <= k) continue;
            double* a = A + p * ldm;
            if (reflect) {  // four independent chains: latency, not issue, bounds one thread
                double w0 = 0.0, w1 = 0.0, w2 = 0.0, w3 = 0.0;
                int i = k;
                for (; i + 3 < m; i += 4) {
                    w0 = fma(v[i], a[i], w0);
                    w1 = fma(v[i + 1], a[i + 1], w1);
                    w2 = fma(v[i + 2], a[i + 2], w2);
                    w3 = fma(v[i + 3], a[i + 3], w3);
                }
                for (; i < m; ++i) w0 = fma(v[i], a[i], w0);
                const double tw = -t * ((w0 + w1) + (w2 + w3));
#pragma unroll 4
                for (i = k; i < m; ++i) a[i] = fma(tw, v[i], a[i]);
            }
            double akk = a[k];
            if (flip) a[k] = akk = -akk;
            if (k + 1 < kmax && vn1[c] != 0.0) {
                double qq = fabs(akk) / vn1[c];
                qq = fmax(0.0, (1.0 - qq) * (1.0 + qq));
                const double ratio = vn1[c] / vn2[c];
                if (qq * ratio * ratio <= tol3z) {
                    double s = 0.0;
                    for (int i = k + 1; i < m; ++i) s = fma(a[i], a[i], s);
                    vn1[c] = vn2[c] = sqrt(s);
                } else {
                    vn1[c] *= sqrt(qq);
                }
            }
        }
        prev_pc = pc;
        prev_k = k;
        prev_alpha = alpha;
        prev_reflect = reflect;
        prev_flip = flip;
        ++k;
    }
    __syncthreads();  // every warp has read the last pivot column
    finalise();
    __syncthreads();
    if (!GLB)
        for (int e = tid; e < k * n; e += kThreads) {
            const int j = e / k, i = e - j * k;
            d.a[i + static_cast<long long>(j) * d.ld] = A[i + j * ldm];
        }
    if (tid == 0) {
        *d.rank = k;
        *d.r11 = r11;
    }
}

// Truncated CPQR for taller blocks (128 < m <= 32 RPL, n <= 2048), in place in
// global memory, one CTA per problem, warp per column.  Same semantics as
// k_cpqr_narrow (first maximum by logical position, exact-norm stop rule with
// one refresh and retry, Householder alpha = -sign+(x0)||x||, row flip, LAPACK
// norm downdate with recompute below sqrt(eps)).  Column state (downdated
// norms, logical positions) lives in shared memory; every warp recomputes the
// pivot's Householder vector from the (L1-resident) pivot column with lane =
// row, keeps v in registers, and sweeps columns w, w + 8, ...: coalesced
// loads of the column, warp-shuffle dot product, update, store.  Two block
// barriers per pivot (argmax partials; column data and state visible to the
// next step).
constexpr int kTallMaxN = 2048;
template <int RPL, int CPW>
__global__ void __launch_bounds__(kThreads, 2) k_cpqr_tall(const CpqrDesc* __restrict__ ds, const int* __restrict__ idx) {
    const CpqrDesc d = ds[idx[blockIdx.x]];
    const int m = d.m, n = d.n, kmax = min(m, n);
    const long long ld = d.ld;
    double* A = d.a;
    __shared__ double s_vn1[kTallMaxN], s_vn2[kTallMaxN];
    __shared__ int s_lpos[kTallMaxN];
    __shared__ double pv[2][kNW];
    __shared__ int pj[2][kNW], pp[2][kNW];
    __shared__ double s_akk[kNW];
    const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
    if (kmax == 0) {
        if (tid == 0) {
            *d.rank = 0;
            *d.r11 = 0.0;
        }
        return;
    }
    const double tol3z = sqrt(DBL_EPSILON);
    // exact column norms, warp per column
    for (int p = wid; p < n; p += kNW) {
        const double* a = A + p * ld;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            const int i = lane + 32 * q;
            if (i < m) s = fma(a[i], a[i], s);
        }
        s = wsum(s);
        if (lane == 0) {
            s_vn1[p] = s_vn2[p] = sqrt(s);
            s_lpos[p] = p;
        }
    }
    __syncthreads();
    int buf = 0;
    auto argmax = [&](int k0, double& bv, int& bj, int& bp) {
        bv = -1.0;
        bj = INT_MAX;
        bp = -1;
        for (int p = tid; p < n; p += kThreads) {
            const int lp = s_lpos[p];
            if (lp >= k0 && better(s_vn1[p], lp, bv, bj)) {
                bv = s_vn1[p];
                bj = lp;
                bp = p;
            }
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            const double ov = __shfl_xor_sync(0xffffffffu, bv, o);
            const int oj = __shfl_xor_sync(0xffffffffu, bj, o);
            const int op = __shfl_xor_sync(0xffffffffu, bp, o);
            if (better(ov, oj, bv, bj)) {
                bv = ov;
                bj = oj;
                bp = op;
            }
        }
        if (lane == 0) {
            pv[buf][wid] = bv;
            pj[buf][wid] = bj;
            pp[buf][wid] = bp;
        }
        __syncthreads();
        bv = -1.0;
        bj = INT_MAX;
        bp = -1;
#pragma unroll
        for (int g = 0; g < kNW; ++g)
            if (better(pv[buf][g], pj[buf][g], bv, bj)) {
                bv = pv[buf][g];
                bj = pj[buf][g];
                bp = pp[buf][g];
            }
        buf ^= 1;
    };
    auto tail_sumsq = [&](int p, int r0) {
        const double* a = A + p * ld;
        double s = 0.0;
#pragma unroll
        for (int q = 0; q < RPL; ++q) {
            const int i = lane + 32 * q;
            if (i >= r0 && i < m) s = fma(a[i], a[i], s);
        }
        return wsum(s);
    };
    double r11 = 0.0;
    int k = 0;
    int prev_pc = -1, prev_k = -1;
    double prev_alpha = 0.0;
    bool prev_reflect = false, prev_flip = false;
    auto finalise = [&]() {  // warp 0 writes alpha e1 into the previous pivot column
        if (prev_pc >= 0 && wid == 0) {
            double* ap = A + prev_pc * ld;
            if (prev_reflect) {
#pragma unroll
                for (int q = 0; q < RPL; ++q) {
                    const int i = lane + 32 * q;
                    if (i == prev_k) ap[i] = prev_flip ? -prev_alpha : prev_alpha;
                    else if (i > prev_k && i < m) ap[i] = 0.0;
                }
            } else if (prev_flip && lane == 0) {
                ap[prev_k] = -ap[prev_k];
            }
        }
        prev_pc = -1;
    };
    while (k < kmax) {
        double bv;
        int piv, pc;
        argmax(k, bv, piv, pc);  // its barrier also orders the previous step's column updates
        finalise();
        double x0 = A[k + pc * ld];
        double tail = tail_sumsq(pc, k + 1);
        double exact = sqrt(fma(x0, x0, tail));
        bool stop = (k == 0) ? !(exact > 0.0) : (d.eps > 0.0 && exact < d.eps * r11);
        if (stop && k > 0) {  // refresh every trailing norm and retry once
            __syncthreads();  // finalise() visible before the column walks
            for (int p = wid; p < n; p += kNW) {
                if (s_lpos[p] < k) continue;
                const double* a = A + p * ld;
                double s = 0.0;
#pragma unroll
                for (int q = 0; q < RPL; ++q) {
                    const int i = lane + 32 * q;
                    if (i >= k && i < m) s = fma(a[i], a[i], s);
                }
                s = wsum(s);
                if (lane == 0) s_vn1[p] = s_vn2[p] = sqrt(s);
            }
            __syncthreads();
            argmax(k, bv, piv, pc);
            exact = bv;
            stop = d.eps > 0.0 && exact < d.eps * r11;
            if (!stop) {
                x0 = A[k + pc * ld];
                tail = tail_sumsq(pc, k + 1);
            }
        }
        if (stop) break;
        double alpha = sqrt(fma(x0, x0, tail));
        if (x0 > 0.0) alpha = -alpha;
        const double v0 = x0 - alpha;
        const double vns = fma(v0, v0, tail);
        const bool reflect = vns > 0.0;
        const double t = reflect ? 2.0 / vns : 0.0;
        const bool flip = (reflect ? alpha : x0) < 0.0;
        double v[RPL];
        {
            const double* ap = A + pc * ld;
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int i = lane + 32 * q;
                v[q] = (i < k || i >= m) ? 0.0 : (i == k ? v0 : ap[i]);
            }
        }
        if (wid == 0 && d.V) {
            double* vk = d.V + static_cast<long long>(k) * d.ldv;
#pragma unroll
            for (int q = 0; q < RPL; ++q) {
                const int i = lane + 32 * q;
                if (i < m) vk[i] = i < k ? 0.0 : (i == k ? 1.0 : (reflect ? v[q] / v0 : 0.0));
            }
        }
        if (tid == 0) {
            if (d.tau) d.tau[k] = reflect ? t * v0 * v0 : 0.0;
            if (d.sign) d.sign[k] = flip ? -1.0 : 1.0;
            if (d.perm) d.perm[k] = pc;
        }
        if (k == 0) r11 = fabs(reflect ? alpha : x0);
        // trailing columns (logical position > k after the swap k <-> piv), warp per column;
        // the swap itself is written by the column's warp (the pivot's by warp 0)
        if (tid == 0) s_lpos[pc] = k;
        // CPW columns per warp iteration: their loads and reductions overlap
        for (int p0 = wid; p0 < n; p0 += kNW * CPW) {
            bool act[CPW];
            double x[CPW][RPL];
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                const int p = p0 + kNW * c;
                const int lp = p < n ? s_lpos[p] : -1;
                act[c] = p < n && p != pc && lp >= k;
                if (act[c] && lp == k && lane == 0) s_lpos[p] = piv;
                const double* a = A + (act[c] ? p : 0) * ld;
#pragma unroll
                for (int q = 0; q < RPL; ++q) {
                    const int i = lane + 32 * q;
                    x[c][q] = (act[c] && i >= k && i < m) ? a[i] : 0.0;
                }
            }
            if (reflect) {
                double sc[CPW];
#pragma unroll
                for (int c = 0; c < CPW; ++c) {
                    sc[c] = 0.0;
#pragma unroll
                    for (int q = 0; q < RPL; ++q) sc[c] = fma(v[q], x[c][q], sc[c]);
                }
#pragma unroll
                for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                    for (int c = 0; c < CPW; ++c) sc[c] += __shfl_xor_sync(0xffffffffu, sc[c], o);
#pragma unroll
                for (int c = 0; c < CPW; ++c) {
                    const double tw = -t * sc[c];
#pragma unroll
                    for (int q = 0; q < RPL; ++q) x[c][q] = fma(tw, v[q], x[c][q]);
                }
            }
#pragma unroll
            for (int c = 0; c < CPW; ++c) {
                if (act[c]) {  // warp-uniform
                const int p = p0 + kNW * c;
                double* a = A + p * ld;
                // row k (lane k % 32 of slot k / 32), flipped when the pivot's diagonal is negative
                // (through shared memory: selecting x[c][k / 32] in registers turns into a
                // dynamically indexed local array)
#pragma unroll
                for (int q = 0; q < RPL; ++q)
                    if (lane + 32 * q == k) s_akk[wid] = x[c][q];
                __syncwarp();
                double akk = s_akk[wid];
                __syncwarp();
                if (flip) akk = -akk;
#pragma unroll
                for (int q = 0; q < RPL; ++q) {
                    const int i = lane + 32 * q;
                    if (i == k) x[c][q] = akk;
                    if (i >= k && i < m && (reflect || i == k)) a[i] = x[c][q];
                }
                if (k + 1 < kmax) {
                    const double vn1 = s_vn1[p];
                    if (vn1 != 0.0) {
                        double qq = fabs(akk) / vn1;
                        qq = fmax(0.0, (1.0 - qq) * (1.0 + qq));
                        const double ratio = vn1 / s_vn2[p];
                        if (qq * ratio * ratio <= tol3z) {
                            double s2 = 0.0;
#pragma unroll
                            for (int q = 0; q < RPL; ++q) {
                                const int i = lane + 32 * q;
                                if (i > k && i < m) s2 = fma(x[c][q], x[c][q], s2);
                            }
                            s2 = wsum(s2);
                            if (lane == 0) s_vn1[p] = s_vn2[p] = sqrt(s2);
                        } else if (lane == 0) {
                            s_vn1[p] = vn1 * sqrt(qq);
                        }
                    }
                }
                }
            }
        }
        prev_pc = pc;
        prev_k = k;
        prev_alpha = alpha;
        prev_reflect = reflect;
        prev_flip = flip;
        ++k;
        __syncthreads();  // column data and state visible to the next scan
    }
    __syncthreads();
    finalise();
    if (tid == 0) {
        *d.rank = k;
        *d.r11 = r11;
    }
}

template <int RPL, bool GLB, int NC>
void launch_narrow(const CpqrDesc* d, const int* idx, int cnt, size_t smem, cudaStream_t st) {
    static SmemCfg configured;
    if (!GLB) smem_optin(reinterpret_cast<const void*>(k_cpqr_narrow<RPL, GLB, NC>), smem, configured);
    k_cpqr_narrow<RPL, GLB, NC><<<cnt, kThreads, GLB ? 0 : smem, st>>>(d, idx);
}

template <int NC>
void launch_nc(int cls, const CpqrDesc* d, const int* idx, int cnt, size_t smem, cudaStream_t st) {
    switch (cls) {
        case 0: launch_narrow<1, false, NC>(d, idx, cnt, smem, st); break;
        case 1: launch_narrow<2, false, NC>(d, idx, cnt, smem, st); break;
        case 2: launch_narrow<4, false, NC>(d, idx, cnt, smem, st); break;
        case 3: launch_narrow<1, true, NC>(d, idx, cnt, smem, st); break;
        case 4: launch_narrow<2, true, NC>(d, idx, cnt, smem, st); break;
        default: launch_narrow<4, true, NC>(d, idx, cnt, smem, st); break;
    }
}

}  // namespace

size_t cpqr_narrow_smem(int m, int n) { return sizeof(double) * static_cast<size_t>(m | 1) * n; }

// classes 0..5: NC = 4 (n <= 1024); 6..11: NC = 8 (n <= 2048).  Within each
// half: 0..2 staged (m <= 32 / 64 / 128), 3..5 in place in global memory.
int cpqr_narrow_class(int m, int n) {
    if (m < 1 || m > 128 || n > 2048) return -1;
    const int r = m <= 32 ? 0 : (m <= 64 ? 1 : 2);
    return (n > 1024 ? 6 : 0) + (cpqr_narrow_smem(m, n) <= kNarrowSmem ? r : 3 + r);
}

// taller blocks, in place: class 0 (m <= 256), 1 (m <= 512); -1 not eligible
int cpqr_tall_class(int m, int n) {
    if (m <= 128 || m > 512 || n > kTallMaxN) return -1;
    return m <= 256 ? 0 : 1;
}

void launch_cpqr_tall(int cls, const CpqrDesc* d_desc, const int* d_idx, int cnt, cudaStream_t st) {
    if (cnt <= 0) return;
    if (cls == 0)
        k_cpqr_tall<8, 4><<<cnt, kThreads, 0, st>>>(d_desc, d_idx);
    else
        k_cpqr_tall<16, 2><<<cnt, kThreads, 0, st>>>(d_desc, d_idx);
}

void launch_cpqr_narrow(int cls, const CpqrDesc* d_desc, const int* d_idx, int cnt, size_t smem, cudaStream_t st) {
    if (cnt <= 0) return;
    if (cls < 6)
        launch_nc<4>(cls, d_desc, d_idx, cnt, smem, st);
    else
        launch_nc<8>(cls - 6, d_desc, d_idx, cnt, smem, st);
}

}  // namespace spqr
