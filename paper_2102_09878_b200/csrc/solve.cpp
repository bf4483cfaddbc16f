// W sweep plan + device CGLS / CSNE drivers.
#include "solve.h"

#include <cstdio>
#include <cstdlib>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <stdexcept>

namespace spqr {

namespace {

// The level schedule of one sweep mode (see solve.h), host side: levels from the walk-order
// conflicts, factors bucketed per level, descriptors (device pointers into W) and the
// accumulation lists.  Pure host work, so the schedules of several modes are built
// concurrently and uploaded afterwards.
struct HostLevel {
    std::vector<WFac> fac, bfac;
    std::vector<int> rptr, ridx, rcol;
    int maxc = 1, bmaxc = 1;
};
struct HostSchedule {
    std::vector<HostLevel> levels;
    long long maxcontrib = 0;
};

HostSchedule host_schedule(const DeviceFactorization& F, int mode, const int* d_idx) {
    const int nfac = static_cast<int>(F.W.size());
    // factors at least this wide run one per CTA (SPQR_BIG_FACTOR overrides, for tests)
    static const int big_cols =
        std::getenv("SPQR_BIG_FACTOR") ? std::atoi(std::getenv("SPQR_BIG_FACTOR")) : kBigFactorCols;
    const bool forward = (mode == kWtSolve || mode == kWApply);
    const bool accumulate = (mode == kWtSolve || mode == kWtApply);
    const size_t n = F.N > 0 ? static_cast<size_t>(F.N) : 1;
    std::vector<int> lastW(n, 0), lastR(n, 0), lastA(n, 0);
    std::vector<int> level(nfac);
    int nlev = 0;
    for (int t = 0; t < nfac; ++t) {
        const int q = forward ? t : nfac - 1 - t;
        const DevWFactor& w = F.W[q];
        const int* cols = F.idx.data() + w.cols_off;
        const int* cp = F.idx.data() + w.coupled_off;
        const int k = (w.kind == 0) ? w.k : 0;
        int L = 0;
        for (int i = 0; i < w.c; ++i) L = std::max({L, lastW[cols[i]], lastR[cols[i]], lastA[cols[i]]});
        if (accumulate) {
            int La = 0;
            for (int j = 0; j < k; ++j) {
                L = std::max({L, lastW[cp[j]], lastR[cp[j]]});
                La = std::max(La, lastA[cp[j]]);
            }
            L = std::max(L + 1, La);
            for (int j = 0; j < k; ++j) lastA[cp[j]] = std::max(lastA[cp[j]], L);
        } else {
            for (int j = 0; j < k; ++j) L = std::max(L, lastW[cp[j]]);
            ++L;
            for (int j = 0; j < k; ++j) lastR[cp[j]] = std::max(lastR[cp[j]], L);
        }
        for (int i = 0; i < w.c; ++i) {
            lastW[cols[i]] = L;
            lastR[cols[i]] = std::max(lastR[cols[i]], L);
        }
        level[q] = L;
        nlev = std::max(nlev, L);
    }
    // bucket the factors by level, in walk order
    std::vector<int> cnt(nlev + 2, 0);
    for (int q = 0; q < nfac; ++q) ++cnt[level[q] + 1];
    for (int l = 0; l <= nlev; ++l) cnt[l + 1] += cnt[l];
    std::vector<int> byl(nfac), pos(cnt.begin(), cnt.end() - 1);
    for (int t = 0; t < nfac; ++t) {
        const int q = forward ? t : nfac - 1 - t;
        byl[pos[level[q]]++] = q;
    }
    HostSchedule H;
    H.levels.resize(nlev);
    std::vector<std::pair<int, int>> lists;  // (coupled column, contribution index) in walk order
    std::vector<int> colcnt(n, 0), touched;
    for (int l = 1; l <= nlev; ++l) {
        HostLevel& hl = H.levels[l - 1];
        lists.clear();
        long long contrib = 0;
        for (int e = cnt[l]; e < cnt[l + 1]; ++e) {
            const DevWFactor& w = F.W[byl[e]];
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
            if (accumulate && w.kind == 0 && w.k > 0) {
                for (int t = 0; t < w.k; ++t) lists.emplace_back(F.idx[w.coupled_off + t], static_cast<int>(contrib + t));
                contrib += w.k;
            }
            // triangular factors: the warp path's back substitution is c sequential steps of
            // c/32 work; rotations: the CTA path pays two block barriers per reflector, so only
            // very tall ones move
            if (w.kind == 0 ? w.c >= big_cols : w.c >= 8 * big_cols) {
                hl.bmaxc = std::max(hl.bmaxc, w.c);
                hl.bfac.push_back(f);
            } else {
                hl.maxc = std::max(hl.maxc, w.c);
                hl.fac.push_back(f);
            }
        }
        if (!lists.empty()) {
            // per coupled column (ascending) its contributions in walk order: a counting sort
            // by column, stable, so each column's indices keep their (ascending) walk order
            touched.clear();
            for (const auto& pr : lists)
                if (colcnt[pr.first]++ == 0) touched.push_back(pr.first);
            std::sort(touched.begin(), touched.end());
            hl.rcol = touched;
            hl.rptr.assign(touched.size() + 1, 0);
            for (size_t c = 0; c < touched.size(); ++c) {
                hl.rptr[c + 1] = hl.rptr[c] + colcnt[touched[c]];
                colcnt[touched[c]] = hl.rptr[c];  // becomes the next write position
            }
            hl.ridx.resize(lists.size());
            for (const auto& pr : lists) hl.ridx[colcnt[pr.first]++] = pr.second;
            for (int c : touched) colcnt[c] = 0;
        }
        H.maxcontrib = std::max(H.maxcontrib, contrib);
    }
    return H;
}

void upload_schedule(SolvePlan& P, int mode, const HostSchedule& H, Uploader& up) {
    SolvePlan::Schedule& S = P.sched[mode];
    S.levels.clear();
    S.launches = 0;
    for (const HostLevel& hl : H.levels) {
        SolvePlan::Level lv;
        lv.fac = up.put(hl.fac);
        lv.nf = static_cast<int>(hl.fac.size());
        lv.maxc = hl.maxc;
        lv.bfac = up.put(hl.bfac);
        lv.nbf = static_cast<int>(hl.bfac.size());
        lv.bmaxc = hl.bmaxc;
        if (!hl.rcol.empty()) {
            lv.rptr = up.put(hl.rptr);
            lv.ridx = up.put(hl.ridx);
            lv.rcol = up.put(hl.rcol);
            lv.ncol = static_cast<int>(hl.rcol.size());
        }
        S.launches += (lv.nf > 0) + (lv.nbf > 0) + (lv.ncol > 0);
        S.levels.push_back(lv);
        P.maxc = std::max(P.maxc, lv.maxc);
        P.bmaxc = std::max(P.bmaxc, lv.bmaxc);
    }
    S.built = true;
}

void build_schedules(SolvePlan& P, const DeviceFactorization& F, cudaStream_t st, std::initializer_list<int> modes) {
    SharedPinned& sp = SharedPinned::get();
    std::lock_guard<std::mutex> pin_lock(sp.mu);
    PinnedArena& pin = sp.arena;
    pin.reset();
    static const bool prof = std::getenv("SPQR_PROF") != nullptr;
    const double t0 = prof ? now_s() : 0.0;
    Uploader up{P.mem.get(), &pin, st};
    if (!P.d_idx) P.d_idx = up.put(F.idx);
    const double t1 = prof ? now_s() : 0.0;
    const std::vector<int> ms(modes);
    std::vector<HostSchedule> hs(ms.size());
#pragma omp parallel for num_threads(static_cast<int>(ms.size())) if (ms.size() > 1)
    for (int i = 0; i < static_cast<int>(ms.size()); ++i) hs[i] = host_schedule(F, ms[i], P.d_idx);
    const double t2 = prof ? now_s() : 0.0;
    long long maxcontrib = P.ncontrib;
    for (size_t i = 0; i < ms.size(); ++i) {
        upload_schedule(P, ms[i], hs[i], up);
        maxcontrib = std::max(maxcontrib, hs[i].maxcontrib);
    }
    if (maxcontrib > P.ncontrib) {
        P.contrib = P.mem->alloc_n<double>(maxcontrib);
        P.ncontrib = maxcontrib;
    }
    prepare_wsweep(P.maxc, P.bmaxc);
    const double t3 = prof ? now_s() : 0.0;
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    if (prof)
        std::fprintf(stderr, "[spqr prof] solve plan: idx upload %.4f schedules %.4f upload %.4f sync %.4f s (%zu idx)\n",
                     t1 - t0, t2 - t1, t3 - t2, now_s() - t3, F.idx.size());
}

}  // namespace

SolvePlan build_solve_plan(const DeviceFactorization& F, cudaStream_t st) {
    const double t0 = now_s();
    SolvePlan P;
    P.mem = std::make_unique<DeviceArena>(size_t(64) << 20);
    build_schedules(P, F, st, {kWSolve, kWtSolve});  // the CGLS / CSNE sweeps; apply modes on demand
    double gathered = 0.0;
    for (const auto& w : F.W) gathered += w.c + (w.kind == 0 ? w.k : 0);
    P.sweep_bytes = 8.0 * static_cast<double>(F.nnz_w()) + 16.0 * gathered;
    P.launches_per_sweep = P.sched[kWSolve].launches;
    P.launches_per_sweep_t = P.sched[kWtSolve].launches;
    P.t_build = now_s() - t0;
    return P;
}

void ensure_schedule(SolvePlan& P, const DeviceFactorization& F, SweepMode mode, cudaStream_t st) {
    if (!P.sched[mode].built) build_schedules(P, F, st, {static_cast<int>(mode)});
}

long long sweep(const SolvePlan& P, SweepMode mode, double* d_z, cudaStream_t st) {
    if (!P.sched[mode].built) throw std::logic_error("W sweep schedule not built (ensure_schedule)");
    long long L = 0;
    for (const auto& lv : P.sched[mode].levels) {
        if (lv.nf > 0) {
            launch_wsweep(lv.fac, lv.nf, d_z, P.contrib, static_cast<int>(mode), lv.maxc, st);
            ++L;
        }
        if (lv.nbf > 0) {  // same level: independent factors, the order of the two launches is free
            launch_wsweep_big(lv.bfac, lv.nbf, d_z, P.contrib, static_cast<int>(mode), lv.bmaxc, st);
            ++L;
        }
        if (lv.ncol > 0) {
            launch_wreduce(lv.rptr, lv.ridx, lv.rcol, lv.ncol, P.contrib, d_z, mode == kWtSolve ? -1.0 : 1.0, st);
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
    CK(cudaMallocHost(reinterpret_cast<void**>(&w.hpin), 2 * sizeof(double)));
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

namespace {

// One captured CUDA graph per half-iteration of CGLS: the kernel sequence of an
// iteration is fixed (the W level schedules, the spmvs, the reductions), so it is
// recorded once per solve and replayed with one launch, instead of ~100 launches.
struct CapturedGraph {
    cudaGraph_t g = nullptr;
    cudaGraphExec_t x = nullptr;
    ~CapturedGraph() {
        if (x) cudaGraphExecDestroy(x);
        if (g) cudaGraphDestroy(g);
    }
    template <class F>
    void capture(cudaStream_t st, F&& body) {
        CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
        body();
        CK(cudaStreamEndCapture(st, &g));
        CK(cudaGraphInstantiate(&x, g, 0));
    }
    void launch(cudaStream_t st) const { CK(cudaGraphLaunch(x, st)); }
};

}  // namespace

SolveReport gpu_cgls(const DevMatrix& A, const SolvePlan* W, const double* d_b, double* d_u, double tol, int maxit,
                     const double* d_w, CglsWork& ws, cudaStream_t st) {
    const double t0 = now_s();
    SolveReport rep;
    const int m = A.m, n = A.n;
    long long L = 0;
    Dots dots{ws, st, L};
    // scalars: 0 nres0^2, 1 gamma, 2 gamma_new, 3 qq, 4 alpha, 5 tn^2
    double* sc = ws.scal;
    launch_copy(m, d_b, ws.r, st);
    launch_spmv_csr(n, A.cp, A.ci, A.cv, ws.r, ws.t, st);  // t = A^T r
    dots.norm2(n, ws.t, d_w ? d_w : nullptr, sc + 0);
    L += 2;
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
        rep.launches = L;
        return rep;
    }
    rep.residual_history.push_back(1.0);
    // sweep timing: e[0..1] eager sweeps, e[2..3] inside g1, e[4..5] inside g2
    cudaEvent_t e[6];
    for (auto& x : e) CK(cudaEventCreate(&x));
    auto acc = [&](int a) {
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e[a], e[a + 1]));
        rep.sweep_ms += ms;
        ++rep.sweeps;
    };
    launch_copy(n, ws.t, ws.s, st);
    if (W) {
        CK(cudaEventRecord(e[0], st));
        L += sweep(*W, kWtSolve, ws.s, st);
        CK(cudaEventRecord(e[1], st));
    }
    launch_copy(n, ws.s, ws.p, st);
    CK(cudaMemsetAsync(ws.y, 0, sizeof(double) * n, st));
    double* gamma = sc + 1;
    double* gnew = sc + 2;
    dots.norm2(n, ws.s, nullptr, gamma);
    L += 2;
    double* hpin = ws.hpin;
    // half-iteration 1 (solve.cpp:50-62): v = W^{-1} p, q = A v, alpha, y, r, t = A^T r, ||w.t||
    long long L1 = 0, L2 = 0;
    CapturedGraph g1, g2;
    g1.capture(st, [&] {
        Dots d1{ws, st, L1};
        launch_copy(n, ws.p, ws.v, st);
        if (W) {
            CK(cudaEventRecordWithFlags(e[2], st, cudaEventRecordExternal));  // a record node in the graph
            L1 += sweep(*W, kWSolve, ws.v, st);
            CK(cudaEventRecordWithFlags(e[3], st, cudaEventRecordExternal));
        }
        launch_spmv_csr(m, A.rp, A.ri, A.rv, ws.v, ws.q, st);  // q = A v
        d1.norm2(m, ws.q, nullptr, sc + 3);
        launch_cgls_alpha(gamma, sc + 3, sc + 4, ws.brk, st);
        launch_axpy_dev(n, sc + 4, 1.0, ws.p, ws.y, st);
        launch_axpy_dev(m, sc + 4, -1.0, ws.q, ws.r, st);
        launch_spmv_csr(n, A.cp, A.ci, A.cv, ws.r, ws.t, st);
        d1.norm2(n, ws.t, d_w, sc + 5);
        L1 += 7;
        CK(cudaMemcpyAsync(hpin, sc + 5, sizeof(double), cudaMemcpyDeviceToHost, st));
        CK(cudaMemcpyAsync(hpin + 1, ws.brk, sizeof(int), cudaMemcpyDeviceToHost, st));
    });
    // half-iteration 2 (:66-71): s = W^{-T} t, gamma_new, p = s + (gamma_new/gamma) p, gamma = gamma_new
    g2.capture(st, [&] {
        Dots d2{ws, st, L2};
        launch_copy(n, ws.t, ws.s, st);
        if (W) {
            CK(cudaEventRecordWithFlags(e[4], st, cudaEventRecordExternal));  // a record node in the graph
            L2 += sweep(*W, kWtSolve, ws.s, st);
            CK(cudaEventRecordWithFlags(e[5], st, cudaEventRecordExternal));
        }
        d2.norm2(n, ws.s, nullptr, gnew);
        launch_cgls_p_update(n, ws.s, gnew, gamma, ws.p, st);
        launch_copy(1, gnew, gamma, st);
        L2 += 3;
    });
    if (W) {
        CK(cudaStreamSynchronize(st));
        acc(0);
    }
    bool g2_pending = false;
    for (int it = 1; it <= maxit; ++it) {
        g1.launch(st);
        L += L1;
        CK(cudaStreamSynchronize(st));
        CK(cudaGetLastError());
        if (W) {
            if (g2_pending) acc(4);
            acc(2);
        }
        g2_pending = false;
        int brk = 0;
        std::memcpy(&brk, hpin + 1, sizeof(int));
        if (brk) break;
        const double rel = std::sqrt(hpin[0]) / nres0;
        rep.residual_history.push_back(rel);
        rep.iterations = it;
        if (rel <= tol || !std::isfinite(rel)) {
            rep.converged = rel <= tol;
            break;
        }
        g2.launch(st);
        L += L2;
        g2_pending = true;
    }
    launch_copy(n, ws.y, d_u, st);
    if (W) {
        CK(cudaEventRecord(e[0], st));
        L += sweep(*W, kWSolve, d_u, st);
        CK(cudaEventRecord(e[1], st));
    }
    CK(cudaStreamSynchronize(st));
    CK(cudaGetLastError());
    if (W) {
        if (g2_pending) acc(4);
        acc(0);
    }
    for (auto& x : e) cudaEventDestroy(x);
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
