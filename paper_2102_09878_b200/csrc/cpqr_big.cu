// Grid-cooperative truncated CPQR for large interfaces (3D top levels).
//
// Semantics: truncated_cpqr (proj/src/dense_kernels.cpp:124-232) — greedy
// column-norm pivoting (first maximum by logical position), exact-norm stop
// rule with one refresh and retry, Householder alpha = -sign+(x0)||x||,
// LAPACK-style norm downdate with recompute below sqrt(eps).
//
// One problem per launch; one CTA per SM cooperates on it.  CTA c owns the
// physical columns c, c+G, c+2G, ...; their logical positions and downdated
// norms live in the CTA's shared memory, the matrix stays in place in HBM/L2.
// Per pivot step there is exactly one grid-wide barrier (the argmax partials).
// After it every CTA reduces the same partials, stages the same pivot column
// into shared memory and computes the same Householder scalars, so all
// decisions agree without further synchronisation.  The pivot column itself
// (alpha e1 and the V column) is finalised by its owner one step later, after
// every CTA is past the barrier that proves nobody still reads it.
#include <cooperative_groups.h>

#include <cfloat>
#include <cstdlib>
#include <cmath>

#include "dev.h"

namespace cg = cooperative_groups;

namespace spqr {

namespace {

constexpr int kThreads = 1024;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct BigScratch {
    double* vn1;   // n: refreshed norms (global mirror used by the retry)
    double* pval;  // G argmax partials: value
    int* pidx;     // G: logical position
    int* pphys;    // G: physical column
};

// better candidate: larger norm, then smaller logical position (first max)
__device__ __forceinline__ bool better(double v, int j, double bv, int bj) { return v > bv || (v == bv && j < bj); }

// block-wide sum, result in every thread
__device__ __forceinline__ double block_sum(double s, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    s = wsum(s);
    __syncthreads();
    if (lane == 0) red[wid] = s;
    __syncthreads();
    double t = 0.0;
    for (int q = 0; q < nw; ++q) t += red[q];
    return t;
}

// Trailing update of U owned columns per warp at a time (ILP over columns).
// xs holds the pivot column rows [k, m); column j gets a_j -= t (v^T a_j) v,
// then the row-k flip and the norm downdate.
template <int U>
__device__ void trailing(double* A, long long ld, int m, int k, int kmax, int G, int cta, int nown, const int* lpos,
                         double* lv1, double* lv2, const double* xs, double v0, double t, bool reflect, bool flip,
                         double tol3z) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int t0 = wid * U; t0 < nown; t0 += nw * U) {
        double* a[U];
        bool act[U];
#pragma unroll
        for (int c = 0; c < U; ++c) {
            const int tt = t0 + c;
            act[c] = tt < nown && lpos[tt] > k;
            a[c] = A + static_cast<long long>(cta + G * tt) * ld;
        }
        double akk[U];
        if (reflect) {
            double w[U];
#pragma unroll
            for (int c = 0; c < U; ++c) w[c] = (lane == 0 && act[c]) ? v0 * a[c][k] : 0.0;
            for (int i = k + 1 + lane; i < m; i += 32) {
                const double x = xs[i];
#pragma unroll
                for (int c = 0; c < U; ++c)
                    if (act[c]) w[c] = fma(x, a[c][i], w[c]);
            }
#pragma unroll
            for (int c = 0; c < U; ++c) w[c] = wsum(w[c]) * t;
            for (int i = k + 1 + lane; i < m; i += 32) {
                const double x = xs[i];
#pragma unroll
                for (int c = 0; c < U; ++c)
                    if (act[c]) a[c][i] = fma(-w[c], x, a[c][i]);
            }
#pragma unroll
            for (int c = 0; c < U; ++c) akk[c] = (lane == 0 && act[c]) ? fma(-w[c], v0, a[c][k]) : 0.0;
        } else {
#pragma unroll
            for (int c = 0; c < U; ++c) akk[c] = (lane == 0 && act[c]) ? a[c][k] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < U; ++c) {
            if (!act[c]) continue;
            if (flip) akk[c] = -akk[c];
            if (lane == 0 && (reflect || flip)) a[c][k] = akk[c];
            if (k + 1 >= kmax) continue;
            int recompute = 0;
            if (lane == 0) {
                const double v1 = lv1[t0 + c];
                if (v1 != 0.0) {
                    double q = fabs(akk[c]) / v1;
                    q = fmax(0.0, (1.0 - q) * (1.0 + q));
                    const double ratio = v1 / lv2[t0 + c];
                    if (q * ratio * ratio <= tol3z)
                        recompute = 1;
                    else
                        lv1[t0 + c] = v1 * sqrt(q);
                }
            }
            recompute = __shfl_sync(0xffffffffu, recompute, 0);
            if (recompute) {
                __syncwarp();  // other lanes' stores of this column are visible
                double s = 0.0;
                for (int i = k + 1 + lane; i < m; i += 32) s = fma(a[c][i], a[c][i], s);
                s = sqrt(wsum(s));
                if (lane == 0) lv1[t0 + c] = lv2[t0 + c] = s;
            }
        }
    }
}

// The cooperative algorithm on G CTAs (rank cta); gsync() is the barrier between them (a
// grid barrier for the whole-GPU launch, a cluster barrier for thread-block clusters).
template <class Sync>
__device__ __forceinline__ void cpqr_coop_body(const CpqrDesc& d, const BigScratch& S, const int G, const int cta,
                                               Sync&& gsync) {
    const int m = d.m, n = d.n, kmax = min(m, n);
    const long long ld = d.ld;
    double* A = d.a;
    const int nown = n > cta ? (n - cta + G - 1) / G : 0;
    extern __shared__ double smem[];
    double* xs = smem;      // m: staged pivot column
    double* lv1 = xs + m;   // nown: downdated norms of owned columns
    double* lv2 = lv1 + nown;
    int* lpos = reinterpret_cast<int*>(lv2 + nown);  // nown: logical positions
    __shared__ double red[32];
    __shared__ int redi[32], redp[32];
    __shared__ int s_piv, s_pc;
    const double tol3z = sqrt(DBL_EPSILON);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;

    for (int t = threadIdx.x; t < nown; t += blockDim.x) lpos[t] = cta + G * t;
    for (int t = wid; t < nown; t += nw) {
        const double* c = A + static_cast<long long>(cta + G * t) * ld;
        double s = 0.0;
        for (int i = lane; i < m; i += 32) s = fma(c[i], c[i], s);
        s = sqrt(wsum(s));
        if (lane == 0) lv1[t] = lv2[t] = s;
    }
    if (kmax == 0) {
        if (cta == 0 && threadIdx.x == 0) {
            *d.rank = 0;
            *d.r11 = 0.0;
        }
        return;
    }

    // grid-wide first max over logical positions >= k0; sets s_piv / s_pc
    auto argmax = [&](int k0) {
        double bv = -1.0;
        int bj = n, bp = -1;
        for (int t = threadIdx.x; t < nown; t += blockDim.x) {
            const int j = lpos[t];
            if (j < k0) continue;
            if (better(lv1[t], j, bv, bj)) {
                bv = lv1[t];
                bj = j;
                bp = cta + G * t;
            }
        }
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
        __syncthreads();
        if (lane == 0) {
            red[wid] = bv;
            redi[wid] = bj;
            redp[wid] = bp;
        }
        __syncthreads();
        if (wid == 0) {
            bv = lane < nw ? red[lane] : -1.0;
            bj = lane < nw ? redi[lane] : n;
            bp = lane < nw ? redp[lane] : -1;
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
                S.pval[cta] = bv;
                S.pidx[cta] = bj;
                S.pphys[cta] = bp;
            }
        }
        gsync();
        if (wid == 0) {  // every CTA reduces the same partials to the same answer
            bv = -1.0;
            bj = n;
            bp = -1;
            for (int q = lane; q < G; q += 32) {
                const double v = __ldcg(S.pval + q);
                const int j = __ldcg(S.pidx + q);
                if (better(v, j, bv, bj)) {
                    bv = v;
                    bj = j;
                    bp = __ldcg(S.pphys + q);
                }
            }
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
                s_piv = bj;
                s_pc = bp;
            }
        }
        __syncthreads();
    };
    // stage rows [k, m) of column pc into xs; returns sum_{i>k} x_i^2 (same in every CTA)
    auto stage = [&](int pc, int k) {
        const double* c = A + static_cast<long long>(pc) * ld;
        double s = 0.0;
        for (int i = k + threadIdx.x; i < m; i += blockDim.x) {
            const double x = __ldcg(c + i);
            xs[i] = x;
            if (i > k) s = fma(x, x, s);
        }
        return block_sum(s, red);  // its barriers also publish xs
    };
    // owner writes V(:, kk) and alpha e1 into the (previous) pivot column
    auto finalise = [&](int pc, int kk, double alpha, double v0, bool reflect, bool flip) {
        if (pc % G != cta) return;
        double* ap = A + static_cast<long long>(pc) * ld;
        if (d.V) {
            double* vk = d.V + static_cast<long long>(kk) * d.ldv;
            for (int i = threadIdx.x; i < m; i += blockDim.x)
                vk[i] = i < kk ? 0.0 : (i == kk ? 1.0 : (reflect ? xs[i] / v0 : 0.0));
        }
        if (reflect) {
            for (int i = kk + threadIdx.x; i < m; i += blockDim.x) ap[i] = i == kk ? (flip ? -alpha : alpha) : 0.0;
        } else if (flip && threadIdx.x == 0) {
            ap[kk] = -ap[kk];
        }
    };

    double r11 = 0.0;
    int k = 0;
    int prev_pc = -1;
    double prev_alpha = 0.0, prev_v0 = 0.0;
    bool prev_reflect = false, prev_flip = false;
    while (k < kmax) {
        __syncthreads();
        argmax(k);
        if (prev_pc >= 0) finalise(prev_pc, k - 1, prev_alpha, prev_v0, prev_reflect, prev_flip);
        prev_pc = -1;
        __syncthreads();  // xs is free again
        int piv = s_piv, pc = s_pc;
        double tail = stage(pc, k);
        double x0 = xs[k];
        double exact = sqrt(fma(x0, x0, tail));
        bool stop = (k == 0) ? !(exact > 0.0) : (d.eps > 0.0 && exact < d.eps * r11);
        if (stop && k > 0) {  // refresh every trailing norm and retry once
            for (int t = wid; t < nown; t += nw) {
                if (lpos[t] < k) continue;
                const double* c = A + static_cast<long long>(cta + G * t) * ld;
                double s = 0.0;
                for (int i = k + lane; i < m; i += 32) s = fma(c[i], c[i], s);
                s = sqrt(wsum(s));
                if (lane == 0) {
                    lv1[t] = lv2[t] = s;
                    S.vn1[cta + G * t] = s;
                }
            }
            __syncthreads();
            argmax(k);  // its grid barrier publishes S.vn1
            piv = s_piv;
            pc = s_pc;
            exact = __ldcg(S.vn1 + pc);
            stop = d.eps > 0.0 && exact < d.eps * r11;
            if (!stop) {
                tail = stage(pc, k);
                x0 = xs[k];
            }
        }
        if (stop) break;
        // logical swap k <-> piv on the owned columns
        for (int t = threadIdx.x; t < nown; t += blockDim.x) {
            const int p = cta + G * t;
            lpos[t] = p == pc ? k : (lpos[t] == k ? piv : lpos[t]);
        }
        double alpha = sqrt(fma(x0, x0, tail));
        if (x0 > 0.0) alpha = -alpha;
        const double v0 = x0 - alpha;
        const double vns = fma(v0, v0, tail);
        const bool reflect = vns > 0.0;
        const double tt = reflect ? 2.0 / vns : 0.0;
        const bool flip = (reflect ? alpha : x0) < 0.0;  // sign of A(k,k) after the step
        if (cta == 0 && threadIdx.x == 0) {
            if (d.tau) d.tau[k] = reflect ? tt * v0 * v0 : 0.0;
            if (d.sign) d.sign[k] = flip ? -1.0 : 1.0;
            if (d.perm) d.perm[k] = pc;
        }
        if (k == 0) r11 = reflect ? fabs(alpha) : fabs(x0);
        __syncthreads();  // lpos
        const int per_warp = (nown + nw - 1) / nw;
        if (per_warp >= 4)
            trailing<4>(A, ld, m, k, kmax, G, cta, nown, lpos, lv1, lv2, xs, v0, tt, reflect, flip, tol3z);
        else if (per_warp >= 2)
            trailing<2>(A, ld, m, k, kmax, G, cta, nown, lpos, lv1, lv2, xs, v0, tt, reflect, flip, tol3z);
        else
            trailing<1>(A, ld, m, k, kmax, G, cta, nown, lpos, lv1, lv2, xs, v0, tt, reflect, flip, tol3z);
        prev_pc = pc;
        prev_alpha = alpha;
        prev_v0 = v0;
        prev_reflect = reflect;
        prev_flip = flip;
        ++k;
    }
    if (prev_pc >= 0) {  // loop ran to kmax: the last pivot column is still pending
        gsync();
        finalise(prev_pc, k - 1, prev_alpha, prev_v0, prev_reflect, prev_flip);
    }
    if (cta == 0 && threadIdx.x == 0) {
        *d.rank = k;
        *d.r11 = r11;
    }
}

__global__ void __launch_bounds__(kThreads, 1) k_cpqr_big(CpqrDesc d, BigScratch S) {
    cg::grid_group grid = cg::this_grid();
    cpqr_coop_body(d, S, static_cast<int>(gridDim.x), static_cast<int>(blockIdx.x), [&] { grid.sync(); });
}

// One problem per thread-block cluster of CS CTAs (distinct problems run concurrently, one
// cluster each): the same algorithm with a cluster barrier (~1 us) in place of the grid
// barrier.  The cluster's partials and the pivot column go through global memory (L2,
// __ldcg); a fence before every barrier makes the CTAs' global stores visible at cluster scope.
template <int CS>
__global__ void __launch_bounds__(kThreads, 1) k_cpqr_clus(const CpqrDesc* __restrict__ ds, const int* __restrict__ idx) {
    cg::cluster_group cl = cg::this_cluster();
    const CpqrDesc d = ds[idx[blockIdx.x / CS]];
    BigScratch S;
    S.vn1 = d.work;
    S.pval = d.work + d.n;
    S.pidx = reinterpret_cast<int*>(S.pval + CS);
    S.pphys = S.pidx + CS;
    cpqr_coop_body(d, S, CS, static_cast<int>(cl.block_rank()), [&] {
        __threadfence();
        cl.sync();
    });
}

}  // namespace

template <int CS>
void launch_clus_cs(const CpqrDesc* ds, const int* idx, int np, size_t smem, cudaStream_t st);

// cluster size: 16 CTAs (non-portable; C3 CPQR 4.6 s against 5.1 s with 8) when the device can
// hold such a cluster of 1024-thread CTAs, else the portable 8; SPQR_CPQR_CLUSTER=8|16 forces one
int cpqr_clus_ctas() {
    static const int cs = [] {
        if (const char* e = std::getenv("SPQR_CPQR_CLUSTER")) return std::atoi(e) == 16 ? 16 : 8;
        if (cudaFuncSetAttribute(reinterpret_cast<const void*>(k_cpqr_clus<16>),
                                 cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
            cudaGetLastError();
            return 8;
        }
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(kThreads);
        cfg.dynamicSmemBytes = 64 * 1024;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        cudaFuncSetAttribute(reinterpret_cast<const void*>(k_cpqr_clus<16>),
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
        int nclus = 0;
        if (cudaOccupancyMaxActiveClusters(&nclus, reinterpret_cast<const void*>(k_cpqr_clus<16>), &cfg) != cudaSuccess) {
            cudaGetLastError();
            return 8;
        }
        return nclus >= 4 ? 16 : 8;
    }();
    return cs;
}

size_t cpqr_clus_smem_bytes(int m, int n) {
    const size_t cs = static_cast<size_t>(cpqr_clus_ctas());
    const size_t nown = (static_cast<size_t>(n) + cs - 1) / cs;
    return sizeof(double) * (static_cast<size_t>(m) + 2 * nown) + sizeof(int) * nown;
}

template <int CS>
void launch_clus_cs(const CpqrDesc* ds, const int* idx, int np, size_t smem, cudaStream_t st) {
    static SmemCfg configured;
    smem_optin(reinterpret_cast<const void*>(k_cpqr_clus<CS>), smem, configured);
    if (CS > 8) cudaFuncSetAttribute(reinterpret_cast<const void*>(k_cpqr_clus<CS>),
                                     cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(static_cast<unsigned>(np) * CS);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CS;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_cpqr_clus<CS>, ds, idx);
}

// problems idx[0..np) of ds, one cluster each; every problem's d.work holds >= n + 32 doubles
void launch_cpqr_clus(const CpqrDesc* ds, const int* idx, int np, size_t smem, cudaStream_t st) {
    if (np <= 0) return;
    if (cpqr_clus_ctas() == 16)
        launch_clus_cs<16>(ds, idx, np, smem, st);
    else
        launch_clus_cs<8>(ds, idx, np, smem, st);
}

int cpqr_big_grid() {
    static int g = 0;
    if (!g) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&g, cudaDevAttrMultiProcessorCount, dev);
    }
    return g;
}

size_t cpqr_big_smem_bytes(int m, int n) {
    const size_t G = static_cast<size_t>(cpqr_big_grid());
    const size_t nown = (static_cast<size_t>(n) + G - 1) / G;
    return sizeof(double) * (static_cast<size_t>(m) + 2 * nown) + sizeof(int) * nown;
}

// d.work: cpqr_big_work_doubles(n) doubles; one problem, whole GPU.
void launch_cpqr_big(const CpqrDesc& d, cudaStream_t st) {
    const int G = cpqr_big_grid();
    const size_t smem = cpqr_big_smem_bytes(d.m, d.n);
    static SmemCfg configured;
    smem_optin(reinterpret_cast<const void*>(k_cpqr_big), smem, configured);
    BigScratch S;
    S.vn1 = d.work;
    S.pval = d.work + d.n;
    S.pidx = reinterpret_cast<int*>(S.pval + G);
    S.pphys = S.pidx + G;
    CpqrDesc dd = d;
    void* args[] = {&dd, &S};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_cpqr_big), G, kThreads, args, smem, st);
}

}  // namespace spqr
