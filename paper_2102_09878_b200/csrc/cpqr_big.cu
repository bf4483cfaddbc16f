// Grid-cooperative truncated CPQR for large interfaces (3D top levels).
//
// Semantics: truncated_cpqr (proj/src/dense_kernels.cpp:124-232) — greedy
// column-norm pivoting (first maximum), exact-norm stop rule with one refresh
// and retry, Householder alpha = -sign+(x0)||x||, LAPACK-style norm downdate.
// One problem per launch, all CTAs of the GPU cooperate: CTA c owns physical
// columns c, c+G, ... .  Per pivot step there is one grid-wide barrier (argmax
// partials); every CTA then reduces the same partials and recomputes the same
// pivot norm and Householder scalars, so decisions are identical everywhere
// without further synchronisation.  The pivot column is finalised (alpha e1,
// V column) by its owner one step later, after every CTA has used it.
#include <cooperative_groups.h>

#include <cfloat>
#include <cmath>

#include "dev.h"

namespace cg = cooperative_groups;

namespace spqr {

namespace {

constexpr int kThreads = 256;

__device__ __forceinline__ double wsum2(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

struct BigScratch {
    double* vn1;   // n, indexed by physical column
    double* vn2;   // n
    double* pval;  // G partial argmax values
    int* pidx;     // G partial argmax logical positions
    int* pos;      // n: logical position of physical column (global mirror)
    int* ph;       // n: physical column at logical position
};

// block-wide norm of column `col` rows [r0, m) (all threads; result to all)
__device__ double block_colnorm(const double* A, long long ld, int col, int r0, int m, double* red) {
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
    double s = 0.0;
    const double* c = A + static_cast<long long>(col) * ld;
    for (int i = r0 + threadIdx.x; i < m; i += blockDim.x) s = fma(c[i], c[i], s);
    s = wsum2(s);
    __syncthreads();
    if (lane == 0) red[wid] = s;
    __syncthreads();
    double t = 0.0;
    for (int q = 0; q < static_cast<int>(blockDim.x >> 5); ++q) t += red[q];
    return sqrt(t);
}

__global__ void __launch_bounds__(kThreads) k_cpqr_big(CpqrDesc d, BigScratch S) {
    cg::grid_group grid = cg::this_grid();
    const int G = gridDim.x, cta = blockIdx.x;
    const int m = d.m, n = d.n, kmax = min(m, n);
    const long long ld = d.ld;
    double* A = d.a;
    __shared__ double red[32];
    __shared__ int redi[32];
    __shared__ int spiv;
    extern __shared__ int sh[];  // ph (n) and pos (n), CTA-local copies
    int* ph = sh;
    int* pos = sh + n;
    const double tol3z = sqrt(DBL_EPSILON);
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
    for (int j = threadIdx.x; j < n; j += blockDim.x) {
        ph[j] = j;
        pos[j] = j;
    }
    // initial norms of owned columns (warp per column)
    for (int p = cta + G * wid; p < n; p += G * nw) {
        double s = 0.0;
        const double* c = A + p * ld;
        for (int i = lane; i < m; i += 32) s = fma(c[i], c[i], s);
        s = sqrt(wsum2(s));
        if (lane == 0) S.vn1[p] = S.vn2[p] = s;
    }
    if (kmax == 0) {
        if (cta == 0 && threadIdx.x == 0) {
            *d.rank = 0;
            *d.r11 = 0.0;
        }
        return;
    }
    double r11 = 0.0;
    int k = 0;
    int prev_pc = -1;
    double prev_alpha = 0.0, prev_v0 = 0.0, prev_vns = 0.0;
    bool prev_flip = false;
    auto argmax = [&](int k0) {  // over logical positions >= k0: (vn1[ph[j]], j), first max
        double bv = -1.0;
        int bj = n;
        for (int p = cta + G * static_cast<int>(threadIdx.x); p < n; p += G * blockDim.x) {
            const int j = pos[p];
            if (j < k0) continue;
            const double v = S.vn1[p];
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
            for (int q = 0; q < nw; ++q)
                if (red[q] > b || (red[q] == b && redi[q] < jj)) {
                    b = red[q];
                    jj = redi[q];
                }
            S.pval[cta] = b;
            S.pidx[cta] = jj;
        }
        grid.sync();
        if (threadIdx.x == 0) {  // every CTA reduces the same partials in the same order
            double b = -1.0;
            int jj = n;
            for (int q = 0; q < G; ++q)
                if (S.pval[q] > b || (S.pval[q] == b && S.pidx[q] < jj)) {
                    b = S.pval[q];
                    jj = S.pidx[q];
                }
            spiv = jj;
        }
        __syncthreads();
        return spiv;
    };
    while (k < kmax) {
        __syncthreads();  // norms written by other warps of this CTA
        int piv = argmax(k);
        // the previous pivot column is final now (every CTA has passed the barrier)
        if (prev_pc >= 0 && prev_pc % G == cta) {
            double* ap = A + prev_pc * ld;
            const int kk = k - 1;
            for (int i = threadIdx.x; i < m - kk; i += blockDim.x) {
                if (d.V) {
                    double* vk = d.V + static_cast<long long>(kk) * d.ldv;
                    vk[kk + i] = (i == 0) ? 1.0 : (prev_vns > 0.0 ? ap[kk + i] / prev_v0 : 0.0);
                }
            }
            if (d.V)
                for (int i = threadIdx.x; i < kk; i += blockDim.x) d.V[static_cast<long long>(kk) * d.ldv + i] = 0.0;
            __syncthreads();
            if (prev_vns > 0.0)
                for (int i = threadIdx.x; i < m - kk; i += blockDim.x) ap[kk + i] = (i == 0) ? (prev_flip ? -prev_alpha : prev_alpha) : 0.0;
            else if (prev_flip && threadIdx.x == 0)
                ap[kk] = -ap[kk];
        }
        prev_pc = -1;  // finalised; a stop below must not finalise it again
        double exact = block_colnorm(A, ld, ph[piv], k, m, red);
        bool stop = (k == 0) ? !(exact > 0.0) : (d.eps > 0.0 && exact < d.eps * r11);
        if (stop && k > 0) {  // refresh all trailing norms, retry once
            grid.sync();
            for (int p = cta + G * wid; p < n; p += G * nw) {
                if (pos[p] < k) continue;
                double s = 0.0;
                const double* c = A + p * ld;
                for (int i = k + lane; i < m; i += 32) s = fma(c[i], c[i], s);
                s = sqrt(wsum2(s));
                if (lane == 0) S.vn1[p] = S.vn2[p] = s;
            }
            grid.sync();
            piv = argmax(k);
            exact = S.vn1[ph[piv]];
            stop = d.eps > 0.0 && exact < d.eps * r11;
        }
        if (stop) break;
        // logical swap k <-> piv (every CTA, local copies)
        __syncthreads();
        if (threadIdx.x == 0 && piv != k) {
            const int a = ph[k], b = ph[piv];
            ph[k] = b;
            ph[piv] = a;
            pos[b] = k;
            pos[a] = piv;
        }
        __syncthreads();
        const int pc = ph[k];
        const double* ap = A + pc * ld;
        double alpha = exact;
        const double x0 = ap[k];
        if (x0 > 0.0) alpha = -alpha;
        const double v0 = x0 - alpha;
        // ||v||^2 = v0^2 + sum_{i>k} x_i^2 (block reduction, identical in every CTA)
        double s = 0.0;
        for (int i = k + 1 + threadIdx.x; i < m; i += blockDim.x) s = fma(ap[i], ap[i], s);
        s = wsum2(s);
        __syncthreads();
        if (lane == 0) red[wid] = s;
        __syncthreads();
        double tail = 0.0;
        for (int q = 0; q < nw; ++q) tail += red[q];
        const double vns = fma(v0, v0, tail);
        const double t = vns > 0.0 ? 2.0 / vns : 0.0;
        const bool flip = alpha < 0.0;  // sign of R(k,k) after the update (A(k,k) = alpha)
        if (cta == 0 && threadIdx.x == 0) {
            if (d.tau) d.tau[k] = vns > 0.0 ? t * v0 * v0 : 0.0;
            if (d.sign) d.sign[k] = flip ? -1.0 : 1.0;
            if (d.perm) d.perm[k] = pc;
        }
        if (k == 0) r11 = flip ? -alpha : alpha;
        // trailing update of owned columns (warp per column), row-k flip, downdate
        for (int p = cta + G * wid; p < n; p += G * nw) {
            const int j = pos[p];
            if (j <= k) continue;
            double* aj = A + p * ld;
            if (vns > 0.0) {
                double w = (lane == 0) ? v0 * aj[k] : 0.0;
                for (int i = k + 1 + lane; i < m; i += 32) w = fma(ap[i], aj[i], w);
                w = wsum2(w);
                const double tw = t * w;
                for (int i = k + 1 + lane; i < m; i += 32) aj[i] = fma(-tw, ap[i], aj[i]);
                if (lane == 0) aj[k] = fma(-tw, v0, aj[k]);
            }
            __syncwarp();
            if (lane == 0 && flip) aj[k] = -aj[k];
            __syncwarp();
            if (k + 1 < kmax) {
                const double v1 = S.vn1[p];
                if (v1 != 0.0) {
                    double tt = fabs(aj[k]) / v1;
                    tt = fmax(0.0, (1.0 - tt) * (1.0 + tt));
                    const double ratio = v1 / S.vn2[p];
                    if (tt * ratio * ratio <= tol3z) {
                        double q = 0.0;
                        for (int i = k + 1 + lane; i < m; i += 32) q = fma(aj[i], aj[i], q);
                        q = sqrt(wsum2(q));
                        if (lane == 0) S.vn1[p] = S.vn2[p] = q;
                    } else if (lane == 0) {
                        S.vn1[p] = v1 * sqrt(tt);
                    }
                }
            }
        }
        prev_pc = pc;
        prev_alpha = alpha;
        prev_v0 = v0;
        prev_vns = vns;
        prev_flip = flip;
        ++k;
    }
    // finalise the last pivot column
    grid.sync();
    if (prev_pc >= 0 && prev_pc % G == cta) {
        double* ap = A + prev_pc * ld;
        const int kk = k - 1;
        if (d.V) {
            double* vk = d.V + static_cast<long long>(kk) * d.ldv;
            for (int i = threadIdx.x; i < m; i += blockDim.x)
                vk[i] = (i < kk) ? 0.0 : (i == kk ? 1.0 : (prev_vns > 0.0 ? ap[i] / prev_v0 : 0.0));
        }
        __syncthreads();
        if (prev_vns > 0.0)
            for (int i = threadIdx.x; i < m - kk; i += blockDim.x) ap[kk + i] = (i == 0) ? (prev_flip ? -prev_alpha : prev_alpha) : 0.0;
        else if (prev_flip && threadIdx.x == 0)
            ap[kk] = -ap[kk];
    }
    if (cta == 0 && threadIdx.x == 0) {
        *d.rank = k;
        *d.r11 = r11;
    }
}

}  // namespace

// d.work: cpqr_big_work_doubles(n) doubles; one problem, whole GPU.
void launch_cpqr_big(const CpqrDesc& d, cudaStream_t st) {
    int dev = 0, sms = 0, per = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const size_t smem = sizeof(int) * 2 * static_cast<size_t>(d.n);
    if (smem > 48 * 1024) cudaFuncSetAttribute(k_cpqr_big, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, k_cpqr_big, kThreads, smem);
    const int G = sms * std::max(1, std::min(per, 2));
    BigScratch S;
    S.vn1 = d.work;
    S.vn2 = d.work + d.n;
    S.pval = d.work + 2 * d.n;
    S.pidx = reinterpret_cast<int*>(d.work + 2 * d.n + G);
    S.pos = S.pidx + G;
    S.ph = S.pos + d.n;
    CpqrDesc dd = d;
    void* args[] = {&dd, &S};
    cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_cpqr_big), G, kThreads, args, smem, st);
}


}  // namespace spqr
