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

// Host bookkeeping threads: all cores but one (measured best on the 16-core B200 hosts)
// unless the user chose a count.
inline void capi_set_threads() {
#ifdef _OPENMP
    if (!std::getenv("OMP_NUM_THREADS")) {
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

// save_factorization (proj/src/transforms.cpp:206-240): SPQRFW01 file of a device W.
inline void save_device_factorization(const DeviceFactorization& F, const char* path) {
    std::vector<std::pair<const char*, std::vector<char>>> mirror;
    F.warena->for_each_chunk([&](const char* base, size_t used) {
        mirror.emplace_back(base, std::vector<char>(used));
        if (used) CK(cudaMemcpy(mirror.back().second.data(), base, used, cudaMemcpyDeviceToHost));
    });
    auto host = [&](const double* d) -> const double* {
        const char* c = reinterpret_cast<const char*>(d);
        for (const auto& m : mirror)
            if (c >= m.first && c < m.first + m.second.size())
                return reinterpret_cast<const double*>(m.second.data() + (c - m.first));
        throw std::logic_error("save_factorization: factor data outside the W arena");
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
            i64(w.c);
            i64(w.k);
            f64s((w.c > 0 && w.k > 0) ? host(w.a) : nullptr, static_cast<size_t>(w.c) * w.k);
            i64(w.k);
            f64s(w.k ? host(w.tau) : nullptr, w.k);
            i64(w.k);
            f64s(w.k ? host(w.sign) : nullptr, w.k);
        }
    }
    i64(0);  // has_q: the GPU engine does not store Q (store_q is a test-only option)
    if (std::ferror(f)) throw std::runtime_error(std::string("write failed: ") + path);
}

}  // namespace spqr
