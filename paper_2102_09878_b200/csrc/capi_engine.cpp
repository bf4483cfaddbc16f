// Engine- and solver-level C ABI (include/spaqr_b200.h, second half): the reference's
//   spaqr_factorize(A, h, row_owner, opt)        proj/include/spaqr/factorize.h:51-53
//   cgls(A, W, b, u, opt, weights)               proj/include/spaqr/solve.h:30-31
//   save_factorization / load_factorization      proj/include/spaqr/transforms.h:75-76
//   Factorization::w_apply/w_solve/wt_apply/wt_solve   transforms.h:66-69
// on a caller-supplied hierarchy and row ownership, with W resident on the GPU.
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>

#include "../../include/spaqr_b200.h"
#include "capi_common.h"
#include "dev.h"
#include "engine.h"
#include "solve.h"

using namespace spqr;

struct spqr_factorization {
    int device = 0;
    cudaStream_t st = nullptr;
    DeviceFactorization F;
    SolvePlan plan;
    QSweep qs;  // store_q: q_apply / q_apply_t
    std::unique_ptr<DeviceArena> mem;
    double* d_z = nullptr;
    double ev_factorize_ms = 0.0;
    ~spqr_factorization() {
        if (st) {
            cudaSetDevice(device);
            cudaStreamSynchronize(st);
            cudaStreamDestroy(st);
        }
    }
};

namespace {

spqr_factorization* new_handle(int device) {
    auto* H = new spqr_factorization;
    H->device = device;
    CK(cudaSetDevice(device));
    CK(cudaStreamCreateWithFlags(&H->st, cudaStreamNonBlocking));
    return H;
}

void finish_handle(spqr_factorization* H) {
    H->plan = build_solve_plan(H->F, H->st);
    H->mem = std::make_unique<DeviceArena>(size_t(8) << 20);
    H->d_z = H->mem->alloc_n<double>(std::max<Index>(H->F.N, 1));
}

// ---- SPQRFW01 reader (transforms.cpp:242-289): W straight into the device W arena ----
struct Reader {
    std::FILE* f;
    std::string path;
    int64_t i64() {
        int64_t v = 0;
        if (std::fread(&v, 8, 1, f) != 1) throw std::runtime_error(path + ": truncated file");
        return v;
    }
    int64_t size() {
        const int64_t n = i64();
        if (n < 0) throw std::runtime_error("corrupt size field in factorization file");
        return n;
    }
    void f64s(double* o, size_t n) {
        if (n && std::fread(o, 8, n, f) != n) throw std::runtime_error(path + ": truncated file");
    }
    std::vector<int> ivec() {
        const int64_t n = size();
        std::vector<int> v(static_cast<size_t>(n));
        for (auto& x : v) x = static_cast<int>(i64());
        return v;
    }
    // get_mat: rows, cols, column-major values
    std::vector<double> mat(int64_t& r, int64_t& c) {
        r = size();
        c = size();
        std::vector<double> m(static_cast<size_t>(r * c));
        f64s(m.data(), m.size());
        return m;
    }
};

}  // namespace

// ------------------------------------------------------------- C ABI -------
extern "C" {

int spqr_factorize(int m, int n, const int* colptr, const int* rowind, const double* vals, int num_levels,
                   int nclusters, const int* cluster_info, const int* cluster_colptr, const int* cluster_cols,
                   const int* finest_of_col, int ntree, const int* tree_parent, int tree_root, const int* row_owner,
                   double eps, int skip_levels, int device, spqr_observer_fn obs, void* obs_user,
                   spqr_factorization** out, char* err, int errlen, int* err_cluster) {
    return spqr_factorize_ex(m, n, colptr, rowind, vals, num_levels, nclusters, cluster_info, cluster_colptr,
                             cluster_cols, finest_of_col, ntree, tree_parent, tree_root, row_owner, eps, skip_levels, 0,
                             device, obs, obs_user, out, err, errlen, err_cluster);
}

int spqr_factorize_ex(int m, int n, const int* colptr, const int* rowind, const double* vals, int num_levels,
                      int nclusters, const int* cluster_info, const int* cluster_colptr, const int* cluster_cols,
                      const int* finest_of_col, int ntree, const int* tree_parent, int tree_root, const int* row_owner,
                      double eps, int skip_levels, int store_q, int device, spqr_observer_fn obs, void* obs_user,
                      spqr_factorization** out, char* err, int errlen, int* err_cluster) {
    *out = nullptr;
    spqr_factorization* H = nullptr;
    const int rc = capi_guarded(err, errlen, err_cluster, [&] {
        if (m < n) throw std::invalid_argument("matrix must have at least as many rows as columns");  // :798-799
        if (!row_owner) throw std::invalid_argument("row_owner size mismatch");                      // :800-801
        if (nclusters <= 0 || ntree <= 0 || tree_root < 0 || tree_root >= ntree)
            throw std::invalid_argument("hierarchy: empty cluster or tree arrays");
        capi_set_threads();
        Csc A = csc_canonical(m, n, colptr, rowind, vals);
        auto tree = std::make_shared<SeparatorTree>();
        tree->num_levels = num_levels;
        tree->root = tree_root;
        tree->nodes.resize(ntree);
        for (int t = 0; t < ntree; ++t) {
            if (tree_parent[t] < -1 || tree_parent[t] >= ntree) throw std::invalid_argument("hierarchy: bad tree parent");
            tree->nodes[t].parent = tree_parent[t];
        }
        ClusterHierarchy h;
        h.num_levels = num_levels;
        h.clusters.resize(nclusters);
        for (int c = 0; c < nclusters; ++c) {
            auto& C = h.clusters[c];
            const int* ci = cluster_info + 5 * c;
            C.tree_node = ci[0];
            C.level = ci[1];
            C.parent = ci[2];
            C.stage = ci[3];
            C.interior = ci[4] != 0;
            if (C.tree_node < 0 || C.tree_node >= ntree || C.parent < -1 || C.parent >= nclusters)
                throw std::invalid_argument("hierarchy: bad cluster " + std::to_string(c));
            C.cols.assign(cluster_cols + cluster_colptr[c], cluster_cols + cluster_colptr[c + 1]);
            for (int j : C.cols)
                if (j < 0 || j >= n) throw std::invalid_argument("hierarchy: column out of range");
        }
        h.finest_of_col.assign(finest_of_col, finest_of_col + n);
        for (int q : h.finest_of_col)
            if (q < 0 || q >= nclusters || h.clusters[q].level != num_levels + 1)
                throw std::invalid_argument("hierarchy: finest_of_col must name a stage-(L+1) cluster");
        h.tree = tree.get();
        std::vector<int> owner(row_owner, row_owner + m);
        for (int q : owner)
            if (q < 0 || q >= nclusters || h.clusters[q].level != num_levels + 1)
                throw std::invalid_argument("row_owner must name stage-(L+1) clusters");
        H = new_handle(device);
        FactorizeOptions fo;
        fo.eps = eps;
        fo.skip_levels = skip_levels;
        fo.store_q = store_q != 0;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, H->st));
        const FactorizeObserver ob = make_observer(obs, obs_user);
        H->F = gpu_factorize(A, h, owner, fo, H->st, obs ? &ob : nullptr);
        finish_handle(H);
        CK(cudaEventRecord(e1, H->st));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        H->ev_factorize_ms = ms;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    });
    if (rc != SPQR_OK) {
        delete H;
        return rc;
    }
    *out = H;
    return SPQR_OK;
}

void spqr_factorization_destroy(spqr_factorization* f) { delete f; }

void spqr_factorization_info(const spqr_factorization* f, long long* o) {
    std::fill(o, o + 8, 0LL);
    o[0] = f->F.M;
    o[1] = f->F.N;
    o[2] = static_cast<long long>(f->F.W.size());
    o[3] = f->F.nnz_w();
    o[4] = static_cast<long long>(f->F.dropped_rows.size());
    o[5] = static_cast<long long>(f->F.trailing_rows.size());
    o[6] = static_cast<long long>(f->F.stages.size());
    o[7] = static_cast<long long>(f->plan.sched[kWSolve].levels.size());
}

long long spqr_factorization_nq(const spqr_factorization* f) {
    return f->F.has_q ? static_cast<long long>(f->F.Q.size()) : -1;
}

void spqr_factorization_rows(const spqr_factorization* f, int* pivot_row, int* dropped, int* trailing) {
    std::copy(f->F.pivot_row.begin(), f->F.pivot_row.end(), pivot_row);
    std::copy(f->F.dropped_rows.begin(), f->F.dropped_rows.end(), dropped);
    std::copy(f->F.trailing_rows.begin(), f->F.trailing_rows.end(), trailing);
}

int spqr_factorization_stage(const spqr_factorization* f, int s, long long* out5) {
    if (s < 0 || s >= static_cast<int>(f->F.stages.size())) return SPQR_E_SHAPE;
    const StageStats& st = f->F.stages[s];
    out5[0] = st.stage;
    out5[1] = static_cast<long long>(st.front_cols.size());
    out5[2] = st.top_rows;
    out5[3] = st.top_cols;
    out5[4] = st.nnz_w;
    return SPQR_OK;
}

int spqr_factorization_stage_fronts(const spqr_factorization* f, int s, int* front_cols) {
    if (s < 0 || s >= static_cast<int>(f->F.stages.size())) return SPQR_E_SHAPE;
    std::copy(f->F.stages[s].front_cols.begin(), f->F.stages[s].front_cols.end(), front_cols);
    return SPQR_OK;
}

int spqr_factorization_apply(spqr_factorization* f, int mode, double* z) {
    int cl = -1;
    return capi_guarded(nullptr, 0, &cl, [&] {
        CK(cudaSetDevice(f->device));
        if (mode == SPQR_Q_APPLY_T || mode == SPQR_Q_APPLY) {
            q_sweep(f->F, f->qs, mode, z, f->st);
            return;
        }
        if (mode < 0 || mode > 3) throw std::invalid_argument("mode must be SPQR_W_APPLY..SPQR_Q_APPLY");
        const Index n = f->F.N;
        CK(cudaMemcpyAsync(f->d_z, z, sizeof(double) * n, cudaMemcpyHostToDevice, f->st));
        static const SweepMode map[4] = {kWApply, kWSolve, kWtApply, kWtSolve};
        ensure_schedule(f->plan, f->F, map[mode], f->st);
        sweep(f->plan, map[mode], f->d_z, f->st);
        CK(cudaMemcpyAsync(z, f->d_z, sizeof(double) * n, cudaMemcpyDeviceToHost, f->st));
        CK(cudaStreamSynchronize(f->st));
    });
}

int spqr_factorization_save(const spqr_factorization* f, const char* path, char* err, int errlen) {
    int cl = -1;
    return capi_guarded(err, errlen, &cl, [&] { save_device_factorization(f->F, path); });
}

int spqr_factorization_load(const char* path, int device, spqr_factorization** out, char* err, int errlen) {
    *out = nullptr;
    spqr_factorization* H = nullptr;
    int cl = -1;
    const int rc = capi_guarded(err, errlen, &cl, [&] {
        std::FILE* fp = std::fopen(path, "rb");
        if (!fp) throw std::runtime_error(std::string("cannot open ") + path);
        std::unique_ptr<std::FILE, int (*)(std::FILE*)> guard(fp, &std::fclose);
        Reader r{fp, path};
        char magic[8];
        if (std::fread(magic, 1, 8, fp) != 8 || std::memcmp(magic, "SPQRFW01", 8) != 0)
            throw std::runtime_error(std::string(path) + ": not a factorization file (bad magic)");
        H = new_handle(device);
        DeviceFactorization& F = H->F;
        F.M = static_cast<Index>(r.i64());
        F.N = static_cast<Index>(r.i64());
        r.f64s(&F.eps, 1);
        F.pivot_row = r.ivec();
        F.dropped_rows = r.ivec();
        F.trailing_rows = r.ivec();
        const int64_t nw = r.size();
        F.W.reserve(static_cast<size_t>(nw));
        F.warena = std::make_unique<DeviceArena>(size_t(128) << 20);
        // factors are staged on the host and uploaded in one copy per arena chunk-sized batch
        std::vector<double> stage;
        std::vector<std::pair<double*, size_t>> pending;  // device destination, offset in stage
        auto flush = [&] {
            for (size_t i = 0; i < pending.size(); ++i) {
                const size_t o = pending[i].second;
                const size_t e = (i + 1 < pending.size()) ? pending[i + 1].second : stage.size();
                if (e > o) CK(cudaMemcpyAsync(pending[i].first, stage.data() + o, sizeof(double) * (e - o),
                                              cudaMemcpyHostToDevice, H->st));
            }
            CK(cudaStreamSynchronize(H->st));
            stage.clear();
            pending.clear();
        };
        auto put = [&](size_t n) -> double* {
            double* d = F.warena->alloc_n<double>(std::max<size_t>(n, 1));
            pending.emplace_back(d, stage.size());
            return d;
        };
        for (int64_t q = 0; q < nw; ++q) {
            const int64_t tag = r.i64();
            DevWFactor w;
            w.cluster = -1;
            if (tag == 0) {  // TriangularScale: cols, R, coupled, C
                const std::vector<int> cols = r.ivec();
                int64_t rr, rc2;
                const std::vector<double> R = r.mat(rr, rc2);
                const std::vector<int> cp = r.ivec();
                int64_t cr, cc;
                const std::vector<double> C = r.mat(cr, cc);
                const int c = static_cast<int>(cols.size());
                if (rr != c || rc2 != c || static_cast<int64_t>(cp.size()) != cc || (cc > 0 && cr != c))
                    throw std::runtime_error(std::string(path) + ": inconsistent TriangularScale");
                w.kind = 0;
                w.c = c;
                w.k = static_cast<int>(cp.size());
                w.scale_only = (cr == 0 && cc == 0);
                w.cols_off = static_cast<long long>(F.idx.size());
                F.idx.insert(F.idx.end(), cols.begin(), cols.end());
                w.coupled_off = static_cast<long long>(F.idx.size());
                F.idx.insert(F.idx.end(), cp.begin(), cp.end());
                w.a = put(static_cast<size_t>(c) * (c + w.k));  // [R | C], c x (c + k)
                stage.insert(stage.end(), R.begin(), R.end());
                stage.insert(stage.end(), C.begin(), C.end());
                if (c == 0 && w.k == 0) stage.push_back(0.0);
            } else if (tag == 1) {  // ColumnRotation: cols, V, tau, sign
                const std::vector<int> cols = r.ivec();
                int64_t vr, vc;
                const std::vector<double> V = r.mat(vr, vc);
                const int64_t nt = r.size();
                std::vector<double> tau(static_cast<size_t>(nt));
                r.f64s(tau.data(), tau.size());
                const int64_t ns = r.size();
                std::vector<double> sg(static_cast<size_t>(ns));
                r.f64s(sg.data(), sg.size());
                const int c = static_cast<int>(cols.size());
                if (vr != c || nt != vc || ns != vc) throw std::runtime_error(std::string(path) + ": inconsistent ColumnRotation");
                w.kind = 1;
                w.c = c;
                w.k = static_cast<int>(vc);
                w.cols_off = static_cast<long long>(F.idx.size());
                F.idx.insert(F.idx.end(), cols.begin(), cols.end());
                w.coupled_off = static_cast<long long>(F.idx.size());
                w.a = put(V.size());
                stage.insert(stage.end(), V.begin(), V.end());
                if (V.empty()) stage.push_back(0.0);
                w.tau = put(tau.size());
                stage.insert(stage.end(), tau.begin(), tau.end());
                if (tau.empty()) stage.push_back(0.0);
                w.sign = put(sg.size());
                stage.insert(stage.end(), sg.begin(), sg.end());
                if (sg.empty()) stage.push_back(0.0);
            } else {
                throw std::runtime_error(std::string(path) + ": unknown factor tag");
            }
            for (long long t = w.cols_off; t < static_cast<long long>(F.idx.size()); ++t)
                if (F.idx[t] < 0 || F.idx[t] >= F.N) throw std::runtime_error(std::string(path) + ": column out of range");
            F.W.push_back(w);
            if (stage.size() > (size_t(32) << 20)) flush();
        }
        flush();
        // Q (has_q, transforms.cpp:277-286): RowReflects kept on the device for q_apply(_t)
        F.has_q = r.i64() != 0;
        if (F.has_q) {
            F.qarena = std::make_unique<DeviceArena>(size_t(64) << 20);
            const int64_t nq = r.size();
            auto qput = [&](size_t n) -> double* {
                double* d = F.qarena->alloc_n<double>(std::max<size_t>(n, 1));
                pending.emplace_back(d, stage.size());
                return d;
            };
            for (int64_t q = 0; q < nq; ++q) {
                const std::vector<int> rows = r.ivec();
                int64_t vr, vc;
                const std::vector<double> V = r.mat(vr, vc);
                const int64_t nt = r.size();
                std::vector<double> tau(static_cast<size_t>(nt));
                r.f64s(tau.data(), tau.size());
                const int64_t ns = r.size();
                std::vector<double> sg(static_cast<size_t>(ns));
                r.f64s(sg.data(), sg.size());
                const int c = static_cast<int>(rows.size());
                if (vr != c || nt != vc || ns != vc) throw std::runtime_error(std::string(path) + ": inconsistent RowReflect");
                for (int x : rows)
                    if (x < 0 || x >= F.M) throw std::runtime_error(std::string(path) + ": row out of range");
                DevWFactor w;
                w.kind = 1;
                w.c = c;
                w.k = static_cast<int>(vc);
                w.cols_off = static_cast<long long>(F.qidx.size());
                F.qidx.insert(F.qidx.end(), rows.begin(), rows.end());
                w.coupled_off = static_cast<long long>(F.qidx.size());
                w.a = qput(V.size());
                stage.insert(stage.end(), V.begin(), V.end());
                if (V.empty()) stage.push_back(0.0);
                w.tau = qput(tau.size());
                stage.insert(stage.end(), tau.begin(), tau.end());
                if (tau.empty()) stage.push_back(0.0);
                w.sign = qput(sg.size());
                stage.insert(stage.end(), sg.begin(), sg.end());
                if (sg.empty()) stage.push_back(0.0);
                F.Q.push_back(w);
                if (stage.size() > (size_t(32) << 20)) flush();
            }
            flush();
        }
        finish_handle(H);
    });
    if (rc != SPQR_OK) {
        delete H;
        return rc;
    }
    *out = H;
    return SPQR_OK;
}

int spqr_cgls(int m, int n, const int* colptr, const int* rowind, const double* vals, spqr_factorization* W,
              const double* b, double* u, double tol, int maxit, const double* weights, int device, int* iters,
              int* converged, double* hist, int* nhist, double* t_solve, char* err, int errlen) {
    int cl = -1;
    return capi_guarded(err, errlen, &cl, [&] {
        if (W && (W->F.N != n)) throw std::invalid_argument("factorization column count does not match A");
        if (W) device = W->device;
        CK(cudaSetDevice(device));
        cudaStream_t st = W ? W->st : nullptr;
        cudaStream_t own = nullptr;
        if (!st) {
            CK(cudaStreamCreateWithFlags(&own, cudaStreamNonBlocking));
            st = own;
        }
        std::unique_ptr<CUstream_st, void (*)(cudaStream_t)> sguard(own, [](cudaStream_t s) {
            if (s) cudaStreamDestroy(s);
        });
        const Csc A = csc_canonical(m, n, colptr, rowind, vals);
        DevMatrix dA = upload_matrix(A, st);
        CglsWork ws = make_cgls_work(m, n);
        DeviceArena mem(size_t(8) << 20);
        double* d_b = mem.alloc_n<double>(std::max(m, 1));
        double* d_u = mem.alloc_n<double>(std::max(n, 1));
        double* d_w = weights ? mem.alloc_n<double>(std::max(n, 1)) : nullptr;
        CK(cudaMemcpyAsync(d_b, b, sizeof(double) * m, cudaMemcpyHostToDevice, st));
        if (d_w) CK(cudaMemcpyAsync(d_w, weights, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        const SolveReport rep = gpu_cgls(dA, W ? &W->plan : nullptr, d_b, d_u, tol > 0 ? tol : 1e-12,
                                         maxit > 0 ? maxit : 500, d_w, ws, st);
        CK(cudaMemcpyAsync(u, d_u, sizeof(double) * n, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        *iters = rep.iterations;
        *converged = rep.converged;
        *nhist = static_cast<int>(rep.residual_history.size());
        std::copy(rep.residual_history.begin(), rep.residual_history.end(), hist);
        *t_solve = rep.t_solve;
    });
}

}  // extern "C"
