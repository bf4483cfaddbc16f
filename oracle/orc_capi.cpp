// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_core.h header).
// Flat C ABI over the restatement so pytest / bench.py (cpu_baseline leg) can
// drive it through ctypes.  Errors: functions return 0 on success, 1 for a
// SingularFrontError (cluster id in *err_cluster), 2 for invalid_argument,
// 3 for anything else; the message is copied into err[errlen].
#include <cstring>
#include <memory>

#include "orc_core.h"

using namespace orc;

namespace {

void put_err(char* err, int errlen, const std::string& s) {
    if (!err || errlen <= 0) return;
    std::strncpy(err, s.c_str(), static_cast<size_t>(errlen - 1));
    err[errlen - 1] = 0;
}

template <class F>
int guarded(char* err, int errlen, int* err_cluster, F&& f) {
    try {
        f();
        return 0;
    } catch (const SingularFrontError& e) {
        if (err_cluster) *err_cluster = e.cluster;
        put_err(err, errlen, std::string(e.what()) + " | reason: " + e.reason);
        return 1;
    } catch (const std::invalid_argument& e) {
        put_err(err, errlen, e.what());
        return 2;
    } catch (const std::exception& e) {
        put_err(err, errlen, e.what());
        return 3;
    }
}

Csc make_csc(int m, int n, const int* p, const int* i, const double* x) {
    // Input is taken as triplets in CSC order so from_triplets canonicalises it.
    std::vector<Trip> t;
    for (int j = 0; j < n; ++j)
        for (int k = p[j]; k < p[j + 1]; ++k) t.push_back({i[k], j, x[k]});
    return csc_from_triplets(m, n, t);
}

Mat make_mat(int r, int c, const double* a) {
    Mat M(r, c);
    if (r > 0 && c > 0) std::memcpy(M.a.data(), a, sizeof(double) * static_cast<size_t>(r) * c);
    return M;
}

// Invariant observer: factorize.cpp test invariants (test_factorize.cpp:309-366):
// row conservation, couplings only along root-to-leaf paths, non-participants
// untouched by an elimination, freshly gained keys carry only appended rows.
struct InvObs : FactorizeObserver {
    const ClusterHierarchy* h = nullptr;
    Index M = 0;
    std::map<int, Front> prev;
    bool has_prev = false;
    std::vector<std::string> phases;
    std::vector<int> stages, details;
    int violations = 0;
    void on_phase(const char* phase, int stage, int detail, const EngineView& v) override {
        phases.emplace_back(phase);
        stages.push_back(stage);
        details.push_back(detail);
        Index live = 0;
        for (const auto& kv : *v.fronts) live += static_cast<Index>(kv.second.rows.size());
        if (live + v.pivots + v.dropped + v.trailing != M) ++violations;
        for (const auto& [c, f] : *v.fronts)
            for (const auto& [key, blk] : f.blocks)
                if (key != c && blk.size() > 0 && !h->related(c, key) && !blk.block_is_zero(0, blk.r, 0, blk.c)) ++violations;
        if (std::string(phase) == "eliminate" && has_prev) {
            const int c = detail;
            for (const auto& [id, nf] : *v.fronts) {
                auto it = prev.find(id);
                if (it == prev.end()) continue;
                const Front& of = it->second;
                if (of.blocks.count(c)) continue;
                if (nf.rows.size() < of.rows.size()) { ++violations; continue; }
                for (size_t i = 0; i < of.rows.size(); ++i)
                    if (nf.rows[i] != of.rows[i]) ++violations;
                const Index onr = static_cast<Index>(of.rows.size());
                for (const auto& [key, blk] : of.blocks) {
                    if (blk.c == 0) continue;
                    auto nb = nf.blocks.find(key);
                    if (nb == nf.blocks.end()) { ++violations; continue; }
                    if (nb->second.c != blk.c) { ++violations; continue; }
                    for (Index j = 0; j < blk.c; ++j)
                        for (Index i = 0; i < onr; ++i)
                            if (nb->second(i, j) != blk(i, j)) { ++violations; j = blk.c; break; }
                }
                for (const auto& [key, blk] : nf.blocks)
                    if (!of.blocks.count(key) && blk.c > 0 && onr > 0 && !blk.block_is_zero(0, onr, 0, blk.c)) ++violations;
            }
        }
        prev = *v.fronts;
        has_prev = true;
    }
};

struct PipeH {
    std::unique_ptr<Pipeline> p;
    std::unique_ptr<InvObs> obs;
};

struct TreeH {
    PatternGraph g;
    SeparatorTree t;
    ClusterHierarchy h;
    std::vector<Index> perm;
};

}  // namespace

extern "C" {

int orc_default_num_levels(int n) { return default_num_levels(n); }

// ------------------------------------------------------------- pipeline ---
void* orc_pipeline_new(int m, int n, const int* colptr, const int* rowind, const double* vals, const double* coords,
                       int dim, const int* parts, int levels, double eps, int skip, int store_q, int solver,
                       int check_invariants, char* err, int errlen, int* err_code, int* err_cluster) {
    auto* H = new PipeH;
    *err_code = guarded(err, errlen, err_cluster, [&] {
        Csc A = make_csc(m, n, colptr, rowind, vals);
        PipelineOptions o;
        o.eps = eps;
        o.levels = levels;
        o.skip_levels = skip;
        o.store_q = store_q != 0;
        o.solver = static_cast<SolverKind>(solver);
        Coords X;
        if (coords) {
            X.n = n;
            X.dim = dim;
            X.x.assign(coords, coords + static_cast<size_t>(n) * dim);
        }
        std::vector<int> pv;
        if (parts) pv.assign(parts, parts + n);
        if (check_invariants) {
            H->obs = std::make_unique<InvObs>();
            H->obs->M = m;
        }
        // The observer needs the hierarchy, which the pipeline builds; it is
        // attached through a small shim that fills h on first call.
        struct Shim : FactorizeObserver {
            InvObs* o;
            Pipeline** pp;
            void on_phase(const char* ph, int s, int d, const EngineView& v) override {
                if (!o->h) o->h = &(*pp)->h;
                o->on_phase(ph, s, d, v);
            }
        } shim;
        Pipeline* raw = nullptr;
        shim.o = H->obs.get();
        shim.pp = &raw;
        // Pipeline's constructor runs the factorization; give the shim a stable
        // pointer to the object under construction via placement.
        void* mem = ::operator new(sizeof(Pipeline));
        raw = static_cast<Pipeline*>(mem);
        try {
            new (mem) Pipeline(A, o, coords ? &X : nullptr, parts ? &pv : nullptr, H->obs ? &shim : nullptr);
        } catch (...) {
            ::operator delete(mem);
            throw;
        }
        H->p.reset(raw);
    });
    if (*err_code) {
        delete H;
        return nullptr;
    }
    return H;
}

void orc_pipeline_free(void* h) { delete static_cast<PipeH*>(h); }

// info: M, N, L, nclusters, nW, nQ, n_dropped, n_trailing, n_stages, nnz_w, nnz(Aw), violations, nphases
void orc_pipeline_info(void* hv, long long* o) {
    auto* H = static_cast<PipeH*>(hv);
    const Pipeline& P = *H->p;
    o[0] = P.Aw.m;
    o[1] = P.Aw.n;
    o[2] = P.h.num_levels;
    o[3] = static_cast<long long>(P.h.clusters.size());
    o[4] = P.has_f ? static_cast<long long>(P.F.W.size()) : 0;
    o[5] = P.has_f ? static_cast<long long>(P.F.Q.size()) : 0;
    o[6] = P.has_f ? static_cast<long long>(P.F.dropped_rows.size()) : 0;
    o[7] = P.has_f ? static_cast<long long>(P.F.trailing_rows.size()) : 0;
    o[8] = P.has_f ? static_cast<long long>(P.F.stages.size()) : 0;
    o[9] = P.has_f ? P.F.nnz_w() : 0;
    o[10] = P.Aw.nnz();
    o[11] = H->obs ? H->obs->violations : -1;
    o[12] = H->obs ? static_cast<long long>(H->obs->phases.size()) : 0;
}

void orc_pipeline_times(void* hv, double* o) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    o[0] = P.t_partition;
    o[1] = P.t_factorize;
}

void orc_pipeline_perm(void* hv, int* o) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    std::copy(P.perm.begin(), P.perm.end(), o);
}
void orc_pipeline_owner(void* hv, int* o) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    std::copy(P.owner.begin(), P.owner.end(), o);
}
void orc_pipeline_weights(void* hv, double* o) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    std::copy(P.weights.begin(), P.weights.end(), o);
}
void orc_pipeline_scaled(void* hv, int* p, int* i, double* x) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    std::copy(P.Aw.p.begin(), P.Aw.p.end(), p);
    std::copy(P.Aw.i.begin(), P.Aw.i.end(), i);
    std::copy(P.Aw.x.begin(), P.Aw.x.end(), x);
}
void orc_pipeline_rows(void* hv, int* pivot_row, int* dropped, int* trailing) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    std::copy(P.F.pivot_row.begin(), P.F.pivot_row.end(), pivot_row);
    std::copy(P.F.dropped_rows.begin(), P.F.dropped_rows.end(), dropped);
    std::copy(P.F.trailing_rows.begin(), P.F.trailing_rows.end(), trailing);
}
// cluster info: tree_node, level, parent, stage, interior, ncols
void orc_pipeline_cluster(void* hv, int c, int* info) {
    const auto& C = static_cast<PipeH*>(hv)->p->h.clusters[c];
    info[0] = C.tree_node;
    info[1] = C.level;
    info[2] = C.parent;
    info[3] = C.stage;
    info[4] = C.interior;
    info[5] = static_cast<int>(C.cols.size());
}
void orc_pipeline_cluster_cols(void* hv, int c, int* o) {
    const auto& C = static_cast<PipeH*>(hv)->p->h.clusters[c];
    std::copy(C.cols.begin(), C.cols.end(), o);
}
// stage: stage, nfronts, top_rows, top_cols, nnz_w(lo), times[5] in t
void orc_pipeline_stage(void* hv, int s, long long* o, double* t) {
    const auto& st = static_cast<PipeH*>(hv)->p->F.stages[s];
    o[0] = st.stage;
    o[1] = static_cast<long long>(st.front_cols.size());
    o[2] = st.top_rows;
    o[3] = st.top_cols;
    o[4] = st.nnz_w;
    t[0] = st.t_eliminate;
    t[1] = st.t_reassign;
    t[2] = st.t_scale;
    t[3] = st.t_sparsify;
    t[4] = st.t_merge;
}
void orc_pipeline_stage_fronts(void* hv, int s, int* cols, double* aspect) {
    const auto& st = static_cast<PipeH*>(hv)->p->F.stages[s];
    std::copy(st.front_cols.begin(), st.front_cols.end(), cols);
    std::copy(st.front_aspect.begin(), st.front_aspect.end(), aspect);
}
void orc_pipeline_phase(void* hv, int i, char* name, int namelen, int* stage, int* detail) {
    auto* H = static_cast<PipeH*>(hv);
    put_err(name, namelen, H->obs->phases[i]);
    *stage = H->obs->stages[i];
    *detail = H->obs->details[i];
}
// W factor i: kind (0 triangular, 1 rotation), ncols, second dim (|coupled| or k), rows of V
void orc_pipeline_wfactor(void* hv, int i, int* o) {
    const auto& f = static_cast<PipeH*>(hv)->p->F.W[i];
    if (const auto* t = std::get_if<TriangularScale>(&f)) {
        o[0] = 0;
        o[1] = static_cast<int>(t->cols.size());
        o[2] = static_cast<int>(t->coupled.size());
    } else {
        const auto& r = std::get<ColumnRotation>(f);
        o[0] = 1;
        o[1] = static_cast<int>(r.cols.size());
        o[2] = r.Q.count();
    }
}
// Triangular: cols, R (c x c), coupled, C (c x |coupled|). Rotation: cols, V (m x k), tau, sign.
void orc_pipeline_wfactor_data(void* hv, int i, int* cols, double* a, int* coupled, double* b, double* c) {
    const auto& f = static_cast<PipeH*>(hv)->p->F.W[i];
    if (const auto* t = std::get_if<TriangularScale>(&f)) {
        std::copy(t->cols.begin(), t->cols.end(), cols);
        std::copy(t->R.a.begin(), t->R.a.end(), a);
        std::copy(t->coupled.begin(), t->coupled.end(), coupled);
        std::copy(t->C.a.begin(), t->C.a.end(), b);
    } else {
        const auto& r = std::get<ColumnRotation>(f);
        std::copy(r.cols.begin(), r.cols.end(), cols);
        std::copy(r.Q.V.a.begin(), r.Q.V.a.end(), a);
        std::copy(r.Q.tau.begin(), r.Q.tau.end(), b);
        std::copy(r.Q.sign.begin(), r.Q.sign.end(), c);
    }
}

// mode: 0 w_apply, 1 w_solve, 2 wt_apply, 3 wt_solve, 4 q_apply_t, 5 q_apply
int orc_pipeline_apply(void* hv, int mode, double* z, char* err, int errlen) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    int cl = -1;
    return guarded(err, errlen, &cl, [&] {
        const size_t n = (mode >= 4) ? P.F.M : P.F.N;
        Vec v(z, z + n);
        switch (mode) {
            case 0: P.F.w_apply(v); break;
            case 1: P.F.w_solve(v); break;
            case 2: P.F.wt_apply(v); break;
            case 3: P.F.wt_solve(v); break;
            case 4: P.F.q_apply_t(v); break;
            case 5: P.F.q_apply(v); break;
            default: throw std::invalid_argument("bad mode");
        }
        std::copy(v.begin(), v.end(), z);
    });
}

// SPQRFW01 files (transforms.cpp:129-289): save this pipeline's factorization;
// load a file and apply one W/Q sweep with it (mode as orc_pipeline_apply).
int orc_pipeline_save(void* hv, const char* path, char* err, int errlen) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    int cl = -1;
    return guarded(err, errlen, &cl, [&] { save_factorization(P.F, path); });
}

int orc_factor_file_apply(const char* path, int mode, double* z, long long nz, long long* dims, char* err, int errlen) {
    int cl = -1;
    return guarded(err, errlen, &cl, [&] {
        const Factorization F = load_factorization(path);
        dims[0] = F.M;
        dims[1] = F.N;
        dims[2] = static_cast<long long>(F.W.size());
        if (!z) return;
        const size_t n = (mode >= 4) ? F.M : F.N;
        if (static_cast<long long>(n) != nz) throw std::invalid_argument("vector length does not match the factorization");
        Vec v(z, z + n);
        switch (mode) {
            case 0: F.w_apply(v); break;
            case 1: F.w_solve(v); break;
            case 2: F.wt_apply(v); break;
            case 3: F.wt_solve(v); break;
            case 4: F.q_apply_t(v); break;
            case 5: F.q_apply(v); break;
            default: throw std::invalid_argument("bad mode");
        }
        std::copy(v.begin(), v.end(), z);
    });
}

// Pipeline::solve (direct=0) / solve_direct (direct=1). hist needs maxit+2 slots.
int orc_pipeline_solve(void* hv, int direct, const double* b, double* x, double tol, int maxit, int* iters,
                       int* converged, double* hist, int* nhist, double* t_solve, char* err, int errlen) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    int cl = -1;
    return guarded(err, errlen, &cl, [&] {
        Vec bb(b, b + P.Aw.m);
        SolveReport rep;
        Vec xx = direct ? P.solve_direct(bb, &rep) : P.solve(bb, &rep, tol, maxit);
        std::copy(xx.begin(), xx.end(), x);
        *iters = rep.iterations;
        *converged = rep.converged;
        *nhist = static_cast<int>(rep.residual_history.size());
        std::copy(rep.residual_history.begin(), rep.residual_history.end(), hist);
        *t_solve = rep.t_solve;
    });
}

// Plain / weighted CGLS on a raw matrix without a factorization (solve.h:30-31, W = nullptr).
int orc_cgls_plain(int m, int n, const int* p, const int* i, const double* v, const double* b, const double* weights,
                   double tol, int maxit, double* x, int* iters, int* converged, double* hist, int* nhist) {
    Csc A = make_csc(m, n, p, i, v);
    Vec bb(b, b + m), w;
    if (weights) w.assign(weights, weights + n);
    CglsOptions co;
    co.tol = tol;
    co.maxit = maxit;
    Vec u;
    SolveReport rep = cgls(A, nullptr, bb, u, co, weights ? &w : nullptr);
    std::copy(u.begin(), u.end(), x);
    *iters = rep.iterations;
    *converged = rep.converged;
    *nhist = static_cast<int>(rep.residual_history.size());
    std::copy(rep.residual_history.begin(), rep.residual_history.end(), hist);
    return 0;
}

// -------------------------------------------------------- dense kernels ---
void orc_householder_qr(int m, int n, const double* B, double* V, double* tau, double* sign, double* R) {
    ReflectorSet H;
    Mat Rm;
    block_householder_qr(make_mat(m, n, B), H, Rm);
    std::copy(H.V.a.begin(), H.V.a.end(), V);
    std::copy(H.tau.begin(), H.tau.end(), tau);
    std::copy(H.sign.begin(), H.sign.end(), sign);
    std::copy(Rm.a.begin(), Rm.a.end(), R);
}

// mode 0: X <- H^T X, 1: X <- H X (X is m x xc); 2: X <- X H, 3: X <- X H^T (X is xr x m)
void orc_apply_reflectors(int m, int k, const double* V, const double* tau, const double* sign, int mode, int xr,
                          int xc, double* X) {
    ReflectorSet H;
    H.V = make_mat(m, k, V);
    H.tau.assign(tau, tau + k);
    H.sign.assign(sign, sign + k);
    Mat Xm = make_mat(xr, xc, X);
    if (mode == 0) apply_left_t(H, view(Xm));
    if (mode == 1) apply_left(H, view(Xm));
    if (mode == 2) apply_right(H, Xm);
    if (mode == 3) apply_right_t(H, Xm);
    std::copy(Xm.a.begin(), Xm.a.end(), X);
}

// Outputs sized for kmax = min(m,n): perm[kmax], R[kmax*n] (rank x n, ld = rank),
// V[m*kmax] (m x rank), tau[kmax], sign[kmax].
void orc_cpqr(int m, int n, const double* B, double eps, int* rank, double* r11, int* perm, double* R, double* V,
              double* tau, double* sign) {
    TruncatedQR T = truncated_cpqr(make_mat(m, n, B), eps);
    *rank = T.rank;
    *r11 = T.r11;
    std::copy(T.perm.begin(), T.perm.end(), perm);
    std::copy(T.R.a.begin(), T.R.a.end(), R);
    std::copy(T.H.V.a.begin(), T.H.V.a.end(), V);
    std::copy(T.H.tau.begin(), T.H.tau.end(), tau);
    std::copy(T.H.sign.begin(), T.H.sign.end(), sign);
}

int orc_tri_solve(int n, const double* R, int br, int bc, double* B, int side_right, int transpose, char* err, int errlen) {
    int cl = 0;
    return guarded(err, errlen, &cl, [&] {
        Mat Rm = make_mat(n, n, R);
        Mat Bm = make_mat(br, bc, B);
        tri_solve_upper(Rm, view(Bm), side_right ? Side::Right : Side::Left, transpose != 0);
        std::copy(Bm.a.begin(), Bm.a.end(), B);
    });
}

int orc_check_diag(int n, const double* R, char* err, int errlen) {
    int cl = 0;
    return guarded(err, errlen, &cl, [&] { check_diag_invertible(make_mat(n, n, R)); });
}

// ----------------------------------------------------- partition pieces ---
void* orc_graph_tree_new(int n, const int* adjptr, const int* adj, const double* coords, int dim, const int* parts,
                         int L, char* err, int errlen, int* err_code) {
    auto* T = new TreeH;
    int cl = 0;
    *err_code = guarded(err, errlen, &cl, [&] {
        T->g.n = n;
        T->g.adj.resize(n);
        for (int v = 0; v < n; ++v) T->g.adj[v].assign(adj + adjptr[v], adj + adjptr[v + 1]);
        Coords X;
        if (coords) {
            X.n = n;
            X.dim = dim;
            X.x.assign(coords, coords + static_cast<size_t>(n) * dim);
        }
        if (parts) {
            std::vector<int> pv(parts, parts + n);
            T->t = import_partition(T->g, L, pv);
        } else {
            T->t = nested_dissection(T->g, L, coords ? &X : nullptr);
        }
        T->h = build_interfaces(T->t, T->g);
    });
    if (*err_code) {
        delete T;
        return nullptr;
    }
    return T;
}
void orc_tree_free(void* t) { delete static_cast<TreeH*>(t); }
int orc_tree_nnodes(void* t) { return static_cast<int>(static_cast<TreeH*>(t)->t.nodes.size()); }
int orc_tree_root(void* t) { return static_cast<TreeH*>(t)->t.root; }
// node: level, parent, child0, child1, nverts, nsep
void orc_tree_node(void* t, int i, int* o) {
    const auto& nd = static_cast<TreeH*>(t)->t.nodes[i];
    o[0] = nd.level;
    o[1] = nd.parent;
    o[2] = nd.child[0];
    o[3] = nd.child[1];
    o[4] = static_cast<int>(nd.vertices.size());
    o[5] = static_cast<int>(nd.separator.size());
}
void orc_tree_node_sets(void* t, int i, int* verts, int* sep) {
    const auto& nd = static_cast<TreeH*>(t)->t.nodes[i];
    std::copy(nd.vertices.begin(), nd.vertices.end(), verts);
    std::copy(nd.separator.begin(), nd.separator.end(), sep);
}
int orc_tree_nclusters(void* t) { return static_cast<int>(static_cast<TreeH*>(t)->h.clusters.size()); }
void orc_tree_cluster(void* t, int c, int* info) {
    const auto& C = static_cast<TreeH*>(t)->h.clusters[c];
    info[0] = C.tree_node;
    info[1] = C.level;
    info[2] = C.parent;
    info[3] = C.stage;
    info[4] = C.interior;
    info[5] = static_cast<int>(C.cols.size());
}
void orc_tree_cluster_cols(void* t, int c, int* o) {
    const auto& C = static_cast<TreeH*>(t)->h.clusters[c];
    std::copy(C.cols.begin(), C.cols.end(), o);
}
void orc_tree_finest(void* t, int* o) {
    const auto& h = static_cast<TreeH*>(t)->h;
    std::copy(h.finest_of_col.begin(), h.finest_of_col.end(), o);
}
int orc_tree_related(void* t, int a, int b) { return static_cast<TreeH*>(t)->h.related(a, b); }
void orc_tree_order(void* t, int* perm) {
    auto* T = static_cast<TreeH*>(t);
    T->perm = order_columns(T->h);
    std::copy(T->perm.begin(), T->perm.end(), perm);
}
int orc_tree_assign_rows(void* t, int m, int n, const int* p, const int* i, const double* x, int* owner, int* row_of_col,
                         int* col_of_row) {
    auto* T = static_cast<TreeH*>(t);
    Csc A = make_csc(m, n, p, i, x);
    RowMatching mm = match_rows(A);
    std::vector<int> own = assign_rows(A, T->h, mm);
    std::copy(own.begin(), own.end(), owner);
    std::copy(mm.row_of_col.begin(), mm.row_of_col.end(), row_of_col);
    std::copy(mm.col_of_row.begin(), mm.col_of_row.end(), col_of_row);
    return mm.size;
}
int orc_match_rows(int m, int n, const int* p, const int* i, const double* x, int* row_of_col, int* col_of_row) {
    Csc A = make_csc(m, n, p, i, x);
    RowMatching mm = match_rows(A);
    std::copy(mm.row_of_col.begin(), mm.row_of_col.end(), row_of_col);
    std::copy(mm.col_of_row.begin(), mm.col_of_row.end(), col_of_row);
    return mm.size;
}

// A^T A pattern: call with adj == nullptr to get the total adjacency length.
long long orc_ata_graph(int m, int n, const int* p, const int* i, const double* x, int* adjptr, int* adj) {
    Csc A = make_csc(m, n, p, i, x);
    PatternGraph g = ata_graph(A);
    long long tot = 0;
    for (const auto& l : g.adj) tot += static_cast<long long>(l.size());
    if (!adj) return tot;
    long long o = 0;
    for (int v = 0; v < n; ++v) {
        adjptr[v] = static_cast<int>(o);
        for (Index u : g.adj[v]) adj[o++] = u;
    }
    adjptr[n] = static_cast<int>(o);
    return tot;
}

// Canonicalise triplets (sparse.cpp:13-20): returns nnz; call with outputs null to size.
int orc_from_triplets(int m, int n, int nt, const int* r, const int* c, const double* v, int* p, int* i, double* x) {
    std::vector<Trip> t(nt);
    for (int k = 0; k < nt; ++k) t[k] = {r[k], c[k], v[k]};
    Csc A = csc_from_triplets(m, n, t);
    if (p) {
        std::copy(A.p.begin(), A.p.end(), p);
        std::copy(A.i.begin(), A.i.end(), i);
        std::copy(A.x.begin(), A.x.end(), x);
    }
    return A.nnz();
}

}  // extern "C"
