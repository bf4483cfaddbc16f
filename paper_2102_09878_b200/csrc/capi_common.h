// Shared pieces of the C ABI implementation (capi.cpp, capi_engine.cpp).
#pragma once

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "../../include/spaqr_b200.h"
#include "engine.h"
#include "solve.h"

namespace spqr {

inline void capi_put_err(char* err, int errlen, const std::string& s) {
    if (!err || errlen <= 0) return;
    std::strncpy(err, s.c_str(), static_cast<size_t>(errlen - 1));
    err[errlen - 1] = 0;
}

// The reference's exceptions as status codes (spaqr_b200.h): SingularFrontError{cluster, reason}
// -> SPQR_E_SINGULAR (+ cluster id and "... | reason: <reason>"), std::invalid_argument ->
// SPQR_E_SHAPE, CUDA failures -> SPQR_E_CUDA, anything else -> SPQR_E_OTHER.
template <class F>
int capi_guarded(char* err, int errlen, int* err_cluster, F&& f) {
    try {
        f();
        return SPQR_OK;
    } catch (const SingularFrontError& e) {
        if (err_cluster) *err_cluster = e.cluster;
        capi_put_err(err, errlen, std::string(e.what()) + " | reason: " + e.reason);
        return SPQR_E_SINGULAR;
    } catch (const std::invalid_argument& e) {
        capi_put_err(err, errlen, e.what());
        return SPQR_E_SHAPE;
    } catch (const CudaError& e) {
        capi_put_err(err, errlen, e.what());
        return SPQR_E_CUDA;
    } catch (const std::exception& e) {
        capi_put_err(err, errlen, e.what());
        return SPQR_E_OTHER;
    }
}

// Host bookkeeping threads: SPQR_HOST_THREADS if set (one process per GPU shares the host's
// cores: torchrun exports OMP_NUM_THREADS=1), else all cores but one (measured best on the
// 16-core B200 hosts) unless the user chose an OpenMP count.
inline void capi_set_threads() {
#ifdef _OPENMP
    if (const char* s = std::getenv("SPQR_HOST_THREADS")) {
        const int n = std::atoi(s);
        if (n > 0) omp_set_num_threads(n);
    } else if (!std::getenv("OMP_NUM_THREADS")) {
        const int np = omp_get_num_procs();
        omp_set_num_threads(np > 1 ? np - 1 : 1);
    }
#endif
}

// The engine's observer as the C ABI's callback: the view's arrays point into the EngineView.
inline FactorizeObserver make_observer(spqr_observer_fn fn, void* user) {
    if (!fn) return FactorizeObserver();
    return [fn, user](const char* phase, int stage, int detail, const EngineView& v) {
        spqr_engine_view cv{};
        cv.nfronts = static_cast<int>(v.front_cluster.size());
        cv.front_cluster = v.front_cluster.data();
        cv.rows_ptr = v.rows_ptr.data();
        cv.rows = v.rows.data();
        cv.keys_ptr = v.keys_ptr.data();
        cv.keys = v.keys.data();
        cv.key_width = v.key_width.data();
        cv.block_off = v.block_off.data();
        cv.values = v.values.data();
        cv.nclusters = static_cast<int>(v.cols_ptr.size()) - 1;
        cv.cols_ptr = v.cols_ptr.data();
        cv.cols = v.cols.data();
        cv.nwave = static_cast<int>(v.wave.size());
        cv.wave = v.wave.data();
        cv.pivots = v.pivots;
        cv.dropped = v.dropped;
        cv.trailing = v.trailing;
        fn(user, phase, stage, detail, &cv);
    };
}

// Factorization::q_apply_t / q_apply (transforms.cpp:113-127) on a host vector of length M:
// the RowReflects (store_q) are rotations on row ids, so they run through the W-sweep level
// schedules (solve.cpp) with z of length M — q_apply_t as the forward walk applying H^T
// (wt_solve's rotation step), q_apply as the backward walk applying H (w_solve's).
struct QSweep {
    DeviceFactorization view;  // W = the Q factors, idx = their row ids, N = M
    SolvePlan plan;
    bool built = false;
    double* d_y = nullptr;
    std::unique_ptr<DeviceArena> mem;
};
inline void q_sweep(const DeviceFactorization& F, QSweep& qs, int mode, double* y, cudaStream_t st) {
    if (!F.has_q) throw std::logic_error("the factorization holds no Q (store_q was not set)");
    if (!qs.built) {
        qs.view.M = qs.view.N = F.M;
        qs.view.W = F.Q;
        qs.view.idx = F.qidx;
        qs.plan = build_solve_plan(qs.view, st);
        qs.mem = std::make_unique<DeviceArena>(sizeof(double) * std::max<size_t>(F.M, 1) + 4096);
        qs.d_y = qs.mem->alloc_n<double>(std::max<size_t>(F.M, 1));
        qs.built = true;
    }
    const SweepMode sm = mode == SPQR_Q_APPLY_T ? kWtSolve : kWSolve;
    CK(cudaMemcpyAsync(qs.d_y, y, sizeof(double) * F.M, cudaMemcpyHostToDevice, st));
    ensure_schedule(qs.plan, qs.view, sm, st);
    sweep(qs.plan, sm, qs.d_y, st);
    CK(cudaMemcpyAsync(y, qs.d_y, sizeof(double) * F.M, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
}

// save_factorization (proj/src/transforms.cpp:206-240): SPQRFW01 file of a device W.
inline void save_device_factorization(const DeviceFactorization& F, const char* path) {
    std::vector<std::pair<const char*, std::vector<char>>> mirror;
    auto grab = [&](const char* base, size_t used) {
        mirror.emplace_back(base, std::vector<char>(used));
        if (used) CK(cudaMemcpy(mirror.back().second.data(), base, used, cudaMemcpyDeviceToHost));
    };
    F.warena->for_each_chunk(grab);
    if (F.has_q && F.qarena) F.qarena->for_each_chunk(grab);
    auto host = [&](const double* d) -> const double* {
        const char* c = reinterpret_cast<const char*>(d);
        for (const auto& m : mirror)
            if (c >= m.first && c < m.first + m.second.size())
                return reinterpret_cast<const double*>(m.second.data() + (c - m.first));
        throw std::logic_error("save_factorization: factor data outside the W / Q arenas");
    };
    std::FILE* f = std::fopen(path, "wb");
    if (!f) throw std::runtime_error(std::string("cannot open ") + path + " for writing");
    std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(f, &std::fclose);
    auto i64 = [&](long long v) {
        const int64_t x = v;
        std::fwrite(&x, 8, 1, f);
    };
    auto f64s = [&](const double* v, size_t n) {
        if (n) std::fwrite(v, 8, n, f);
    };
    auto ivec = [&](const int* v, size_t n) {
        i64(static_cast<long long>(n));
        for (size_t i = 0; i < n; ++i) i64(v[i]);
    };
    std::fwrite("SPQRFW01", 1, 8, f);
    i64(F.M);
    i64(F.N);
    f64s(&F.eps, 1);
    ivec(F.pivot_row.data(), F.pivot_row.size());
    ivec(F.dropped_rows.data(), F.dropped_rows.size());
    ivec(F.trailing_rows.data(), F.trailing_rows.size());
    i64(static_cast<long long>(F.W.size()));
    auto reflectors = [&](const DevWFactor& w) {  // put_reflectors: V c x k (unit diagonal explicit), tau, sign
        i64(w.c);
        i64(w.k);
        f64s((w.c > 0 && w.k > 0) ? host(w.a) : nullptr, static_cast<size_t>(w.c) * w.k);
        i64(w.k);
        f64s(w.k ? host(w.tau) : nullptr, w.k);
        i64(w.k);
        f64s(w.k ? host(w.sign) : nullptr, w.k);
    };
    for (const DevWFactor& w : F.W) {
        const int* cols = F.idx.data() + w.cols_off;
        if (w.kind == 0) {  // a = [R | C], c x (c + k), column-major
            const double* a = w.c ? host(w.a) : nullptr;
            i64(0);
            ivec(cols, w.c);
            i64(w.c);
            i64(w.c);
            f64s(a, static_cast<size_t>(w.c) * w.c);
            ivec(F.idx.data() + w.coupled_off, w.k);
            i64(w.scale_only ? 0 : w.c);  // scale_all's factor keeps the default-constructed C (0 x 0)
            i64(w.k);
            f64s(a ? a + static_cast<size_t>(w.c) * w.c : nullptr, static_cast<size_t>(w.c) * w.k);
        } else {  // V c x k (unit diagonal explicit), tau k, sign k
            i64(1);
            ivec(cols, w.c);
            reflectors(w);
        }
    }
    i64(F.has_q ? 1 : 0);  // transforms.cpp:230-237: Q as (rows, reflectors) per RowReflect
    if (F.has_q) {
        i64(static_cast<long long>(F.Q.size()));
        for (const DevWFactor& q : F.Q) {
            ivec(F.qidx.data() + q.cols_off, q.c);
            reflectors(q);
        }
    }
    if (std::ferror(f)) throw std::runtime_error(std::string("write failed: ") + path);
}

}  // namespace spqr
