// W sweep plan + device CGLS / CSNE drivers.
#include "solve.h"

#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>

namespace spqr {

SolvePlan build_solve_plan(const DeviceFactorization& F, cudaStream_t st) {
    SolvePlan P;
    P.mem = std::make_unique<DeviceArena>(size_t(64) << 20);
    SharedPinned& sp = SharedPinned::get();
    std::lock_guard<std::mutex> pin_lock(sp.mu);
    PinnedArena& pin = sp.arena;
    pin.reset();
    Uploader up{P.mem.get(), &pin, st};
    const int* d_idx = up.put(F.idx);
    // group factors by batch (batch ids increase chronologically; within a
    // batch the factors commute)
    std::vector<size_t> ord(F.W.size());
    for (size_t q = 0; q < ord.size(); ++q) ord[q] = q;
    std::stable_sort(ord.begin(), ord.end(), [&](size_t a, size_t b) { return F.W[a].batch < F.W[b].batch; });
    long long maxcontrib = 1;
    // factors at least this wide run one per CTA (SPQR_BIG_FACTOR overrides, for tests)
    const int big_cols = std::getenv("SPQR_BIG_FACTOR") ? std::atoi(std::getenv("SPQR_BIG_FACTOR")) : kBigFactorCols;
    size_t i = 0;
    while (i < ord.size()) {
        size_t j = i;
        while (j < ord.size() && F.W[ord[j]].batch == F.W[ord[i]].batch) ++j;
        std::vector<WFac> fac, bfac;
        long long contrib = 0;
        std::vector<std::pair<int, int>> lists;  // (coupled column, contribution index), chronological
        int maxc = 1, bmaxc = 1;
        for (size_t q = i; q < j; ++q) {
            const DevWFactor& w = F.W[ord[q]];
            WFac f{};
            f.kind = w.kind;
            f.c = w.c;
            f.k = w.k;
            f.cols = d_idx + w.cols_off;
            f.coupled = d_idx + w.coupled_off;
            f.a = w.a;
            f.tau = w.tau;
            f.sign = w.sign;
            f.contrib_off = contrib;
            if (w.kind == 0 && w.k > 0) {
                for (int t = 0; t < w.k; ++t) lists.emplace_back(F.idx[w.coupled_off + t], static_cast<int>(contrib + t));
                contrib += w.k;
            }
            // triangular factors: the warp path's back substitution is c sequential
            // steps of c/32 work; rotations: the CTA path pays two block barriers per
            // reflector, so only very tall ones move
            if (w.kind == 0 ? w.c >= big_cols : w.c >= 8 * big_cols) {
                bmaxc = std::max(bmaxc, w.c);
                bfac.push_back(f);
            } else {
                maxc = std::max(maxc, w.c);
                fac.push_back(f);
            }
        }
        SolvePlan::Batch b;
        b.fac = up.put(fac);
        b.nf = static_cast<int>(fac.size());
        b.maxc = maxc;
        b.bfac = up.put(bfac);
        b.nbf = static_cast<int>(bfac.size());
        b.bmaxc = bmaxc;
        if (!lists.empty()) {
            // per coupled column (ascending), its contributions in chronological order:
            // the indices increase with time, so sorting the pairs gives exactly that
            std::sort(lists.begin(), lists.end());
            std::vector<int> ptr{0}, idx, col;
            idx.reserve(lists.size());
            for (size_t a = 0; a < lists.size();) {
                size_t e = a;
                while (e < lists.size() && lists[e].first == lists[a].first) idx.push_back(lists[e++].second);
                col.push_back(lists[a].first);
                ptr.push_back(static_cast<int>(idx.size()));
                a = e;
            }
            b.rptr = up.put(ptr);
            b.ridx = up.put(idx);
            b.rcol = up.put(col);
            b.ncol = static_cast<int>(col.size());
        }
        maxcontrib = std::max(maxcontrib, contrib);
        P.batches.push_back(b);
        i = j;
    }
    P.contrib = P.mem->alloc_n<double>(maxcontrib);
    for (const auto& b : P.batches) {
        const int k = (b.nf > 0 ? 1 : 0) + (b.nbf > 0 ? 1 : 0);
        P.launches_per_sweep += k;
        P.launches_per_sweep_t += k + (b.ncol > 0 ? 1 : 0);
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    return P;
}

long long sweep(const SolvePlan& P, SweepMode mode, double* d_z, cudaStream_t st) {
    long long L = 0;
    const int nb = static_cast<int>(P.batches.size());
    const bool forward = (mode == kWtSolve || mode == kWApply);  // chronological order
    for (int q = 0; q < nb; ++q) {
        const auto& b = P.batches[forward ? q : nb - 1 - q];
        if (b.nf > 0) {
            launch_wsweep(b.fac, b.nf, d_z, P.contrib, static_cast<int>(mode), b.maxc, st);
            ++L;
        }
        if (b.nbf > 0) {  // same batch: the factors commute, the order of the two launches is free
            launch_wsweep_big(b.bfac, b.nbf, d_z, P.contrib, static_cast<int>(mode), b.bmaxc, st);
            ++L;
        }
        if ((mode == kWtSolve || mode == kWtApply) && b.ncol > 0) {
            launch_wreduce(b.rptr, b.ridx, b.rcol, b.ncol, P.contrib, d_z, mode == kWtSolve ? -1.0 : 1.0, st);
            ++L;
        }
    }
    return L;
}

DevMatrix upload_matrix(const Csc& A, cudaStream_t st) {
    DevMatrix D;
    D.m = A.m;
    D.n = A.n;
    D.mem = std::make_unique<DeviceArena>(size_t(64) << 20);
    // CSR of A with columns ascending per row (so each row dot runs in the
    // reference's column order)
    std::vector<int> rp(A.m + 1, 0), ri(A.nnz());
    std::vector<double> rv(A.nnz());
    for (Index k = 0; k < A.nnz(); ++k) rp[A.i[k] + 1]++;
    for (Index r = 0; r < A.m; ++r) rp[r + 1] += rp[r];
    std::vector<int> pos(rp.begin(), rp.end() - 1);
    for (Index j = 0; j < A.n; ++j)
        for (Index k = A.p[j]; k < A.p[j + 1]; ++k) {
            ri[pos[A.i[k]]] = j;
            rv[pos[A.i[k]]++] = A.x[k];
        }
    SharedPinned& sp = SharedPinned::get();
    std::lock_guard<std::mutex> pin_lock(sp.mu);
    sp.arena.reset();
    Uploader up{D.mem.get(), &sp.arena, st};
    D.rp = up.put(rp);
    D.ri = up.put(ri);
    D.rv = up.put(rv);
    D.cp = up.put(A.p);
    D.ci = up.put(A.i);
    D.cv = up.put(A.x);
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    return D;
}

CglsWork make_cgls_work(int m, int n) {
    CglsWork w;
    w.mem = std::make_unique<DeviceArena>(size_t(16) << 20);
    const int big = std::max(m, n);
    w.r = w.mem->alloc_n<double>(std::max(m, 1));
    w.q = w.mem->alloc_n<double>(std::max(m, 1));
    w.t = w.mem->alloc_n<double>(std::max(n, 1));
    w.s = w.mem->alloc_n<double>(std::max(n, 1));
    w.p = w.mem->alloc_n<double>(std::max(n, 1));
    w.y = w.mem->alloc_n<double>(std::max(n, 1));
    w.v = w.mem->alloc_n<double>(std::max(n, 1));
    w.nblocks = std::max(1, std::min(4 * sm_count(), (big + 255) / 256));
    w.partial = w.mem->alloc_n<double>(w.nblocks);
    w.scal = w.mem->alloc_n<double>(16);
    w.brk = w.mem->alloc_n<int>(4);
    return w;
}

namespace {

struct Dots {
    const CglsWork& w;
    cudaStream_t st;
    long long& launches;
    void norm2(int n, const double* a, const double* wt, double* out) {  // sum (a*w)^2 or a.a
        launch_dot_partial(n, a, a, wt, w.partial, w.nblocks, st);
        launch_finish_sum(w.partial, w.nblocks, out, st);
        launches += 2;
    }
};

}  // namespace

SolveReport gpu_cgls(const DevMatrix& A, const SolvePlan* W, const double* d_b, double* d_u, double tol, int maxit,
                     const double* d_w, CglsWork& ws, cudaStream_t st) {
    const double t0 = now_s();
    SolveReport rep;
    const int m = A.m, n = A.n;
    long long L = 0;
    Dots dots{ws, st, L};
    // scalars: 0 nres0^2, 1 gamma(a), 2 gamma(b), 3 qq, 4 alpha, 5 tn^2
    double* sc = ws.scal;
    launch_copy(m, d_b, ws.r, st);
    launch_spmv_csr(n, A.cp, A.ci, A.cv, ws.r, ws.t, st);  // t = A^T r
    dots.norm2(n, ws.t, d_w ? d_w : nullptr, sc + 0);
    double h0 = 0.0;
    CK(cudaMemcpyAsync(&h0, sc + 0, sizeof(double), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    const double nres0 = std::sqrt(h0);
    CK(cudaMemsetAsync(d_u, 0, sizeof(double) * n, st));
    if (nres0 == 0.0) {
        rep.converged = true;
        rep.residual_history = {0.0};
        rep.t_solve = now_s() - t0;
        return rep;
    }
    rep.residual_history.push_back(1.0);
    launch_copy(n, ws.t, ws.s, st);
    if (W) L += sweep(*W, kWtSolve, ws.s, st);
    launch_copy(n, ws.s, ws.p, st);
    CK(cudaMemsetAsync(ws.y, 0, sizeof(double) * n, st));
    double* gamma = sc + 1;
    double* gnew = sc + 2;
    dots.norm2(n, ws.s, nullptr, gamma);
    struct {
        double tn2;
        int brk;
    } hres;
    double* hpin = nullptr;
    CK(cudaMallocHost(reinterpret_cast<void**>(&hpin), 2 * sizeof(double)));
    for (int it = 1; it <= maxit; ++it) {
        launch_copy(n, ws.p, ws.v, st);
        if (W) L += sweep(*W, kWSolve, ws.v, st);
        launch_spmv_csr(m, A.rp, A.ri, A.rv, ws.v, ws.q, st);  // q = A v
        dots.norm2(m, ws.q, nullptr, sc + 3);
        launch_cgls_alpha(gamma, sc + 3, sc + 4, ws.brk, st);
        launch_axpy_dev(n, sc + 4, 1.0, ws.p, ws.y, st);
        launch_axpy_dev(m, sc + 4, -1.0, ws.q, ws.r, st);
        launch_spmv_csr(n, A.cp, A.ci, A.cv, ws.r, ws.t, st);
        dots.norm2(n, ws.t, d_w, sc + 5);
        L += 7;
        CK(cudaMemcpyAsync(hpin, sc + 5, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hpin + 1, ws.brk, sizeof(int), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaGetLastError());
        hres.tn2 = hpin[0];
        std::memcpy(&hres.brk, hpin + 1, sizeof(int));
        if (hres.brk) break;
        const double rel = std::sqrt(hres.tn2) / nres0;
        rep.residual_history.push_back(rel);
        rep.iterations = it;
        if (rel <= tol || !std::isfinite(rel)) {
            rep.converged = rel <= tol;
            break;
        }
        launch_copy(n, ws.t, ws.s, st);
        if (W) L += sweep(*W, kWtSolve, ws.s, st);
        dots.norm2(n, ws.s, nullptr, gnew);
        launch_cgls_p_update(n, ws.s, gnew, gamma, ws.p, st);
        L += 3;
        std::swap(gamma, gnew);
    }
    cudaFreeHost(hpin);
    launch_copy(n, ws.y, d_u, st);
    if (W) L += sweep(*W, kWSolve, d_u, st);
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    rep.t_solve = now_s() - t0;
    rep.launches = L;
    return rep;
}

SolveReport gpu_csne(const DevMatrix& A, const SolvePlan& W, const double* d_b, double* d_u, int refine, const double* d_w,
                     double tol, CglsWork& ws, cudaStream_t st) {
    const double t0 = now_s();
    SolveReport rep;
    const int m = A.m, n = A.n;
    long long L = 0;
    Dots dots{ws, st, L};
    double* sc = ws.scal;
    auto hostval = [&](const double* d) {
        double h = 0.0;
        CK(cudaMemcpyAsync(&h, d, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        CK(cudaGetLastError());
        return h;
    };
    launch_spmv_csr(n, A.cp, A.ci, A.cv, d_b, ws.t, st);
    dots.norm2(n, ws.t, d_w, sc + 0);
    const double nres0 = std::sqrt(hostval(sc + 0));
    launch_copy(n, ws.t, d_u, st);
    sweep(W, kWtSolve, d_u, st);
    sweep(W, kWSolve, d_u, st);
    // one = 1.0 on device for axpy with a device scalar
    const double one = 1.0, mone = -1.0;
    CK(cudaMemcpyAsync(sc + 6, &one, sizeof(double), cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(sc + 7, &mone, sizeof(double), cudaMemcpyHostToDevice, st));
    auto residual_normal = [&]() {  // t = A^T (b - A u)
        launch_spmv_csr(m, A.rp, A.ri, A.rv, d_u, ws.q, st);
        launch_copy(m, d_b, ws.r, st);
        launch_axpy_dev(m, sc + 6, -1.0, ws.q, ws.r, st);
        launch_spmv_csr(n, A.cp, A.ci, A.cv, ws.r, ws.t, st);
    };
    auto record = [&]() {
        if (nres0 == 0.0) {
            rep.residual_history.push_back(0.0);
            return;
        }
        residual_normal();
        dots.norm2(n, ws.t, d_w, sc + 5);
        rep.residual_history.push_back(std::sqrt(hostval(sc + 5)) / nres0);
    };
    record();
    for (int step = 0; step < refine; ++step) {
        residual_normal();
        launch_copy(n, ws.t, ws.v, st);
        sweep(W, kWtSolve, ws.v, st);
        sweep(W, kWSolve, ws.v, st);
        launch_axpy_dev(n, sc + 6, 1.0, ws.v, d_u, st);
        record();
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    rep.iterations = refine;
    rep.converged = rep.residual_history.back() <= tol;
    rep.t_solve = now_s() - t0;
    return rep;
}

}  // namespace spqr
