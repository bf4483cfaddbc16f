// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// The same flat C ABI as oracle/orc_capi.cpp (same orc_* symbol names and argument
// meaning), implemented over the UNMODIFIED reference sources
// /root/reference/proj/src/{dense_kernels,sparse,partition,factorize,transforms,
// solve,pipeline}.cpp compiled against the in-repo Eigen API shim
// (oracle/eigen_shim/).  Built by oracle/Makefile.ref into
// oracle/_ref/libspaqr_ref.so (git-ignored; it travels to the GPU box, where
// /root/reference does not exist).  oracle/ref.py loads it through the same
// ctypes front-end as the restatement, so every test can run against the
// reference's own engine code: that is what pins the restatement (orc_*.cpp).
#include <cstring>
#include <memory>
#include <string>

#include "spaqr/dense_kernels.h"
#include "spaqr/factorize.h"
#include "spaqr/partition.h"
#include "spaqr/pipeline.h"
#include "spaqr/solve.h"
#include "spaqr/sparse.h"
#include "spaqr/transforms.h"

using namespace spaqr;

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

SparseMatrix make_csc(int m, int n, const int* p, const int* i, const double* x) {
    std::vector<Eigen::Triplet<double>> t;
    for (int j = 0; j < n; ++j)
        for (int k = p[j]; k < p[j + 1]; ++k) t.emplace_back(i[k], j, x[k]);
    return SparseMatrix::from_triplets(m, n, t);
}

MatrixXd make_mat(int r, int c, const double* a) {
    MatrixXd M(r, c);
    if (r * c) std::memcpy(M.data(), a, sizeof(double) * static_cast<size_t>(r) * c);
    return M;
}

void copy_mat(const MatrixXd& M, double* o) {
    if (M.size()) std::memcpy(o, M.data(), sizeof(double) * static_cast<size_t>(M.size()));
}

// Phase recorder plus the reference's own engine invariants, as its test's
// InvariantObserver states them (test_factorize.cpp:309-366): row conservation,
// couplings only along root-to-leaf paths, non-participants untouched by an
// elimination, freshly gained keys carry only appended rows.
struct PhaseObs : FactorizeObserver {
    const ClusterHierarchy* h = nullptr;
    Index M = 0;
    std::map<int, Front> prev;
    bool has_prev = false;
    std::vector<std::string> phases;
    std::vector<int> stages, details;
    int violations = 0;
    bool check = false;
    void on_phase(const char* phase, int stage, int detail, const EngineView& v) override {
        phases.emplace_back(phase);
        stages.push_back(stage);
        details.push_back(detail);
        if (!check || !h) return;
        Index live = 0;
        for (const auto& kv : *v.fronts) live += static_cast<Index>(kv.second.rows.size());
        if (live + v.pivots + v.dropped + v.trailing != M) ++violations;
        for (const auto& [c, f] : *v.fronts)
            for (const auto& [key, blk] : f.blocks)
                if (key != c && blk.size() > 0 && !h->related(c, key) && !blk.isZero(0.0)) ++violations;
        if (std::string(phase) == "eliminate" && has_prev) {
            const int c = detail;
            for (const auto& [id, nf] : *v.fronts) {
                auto it = prev.find(id);
                if (it == prev.end()) continue;
                const Front& of = it->second;
                if (of.blocks.count(c)) continue;
                if (nf.rows.size() < of.rows.size()) ++violations;
                for (size_t i = 0; i < of.rows.size() && i < nf.rows.size(); ++i)
                    if (nf.rows[i] != of.rows[i]) ++violations;
                const Index onr = static_cast<Index>(of.rows.size());
                for (const auto& [key, blk] : of.blocks) {
                    auto nb = nf.blocks.find(key);
                    if (blk.cols() == 0) continue;
                    if (nb == nf.blocks.end()) {
                        ++violations;
                        continue;
                    }
                    if (nb->second.cols() != blk.cols() || nb->second.rows() < onr ||
                        !(nb->second.topRows(onr) - blk).isZero(0.0))
                        ++violations;
                }
                for (const auto& [key, blk] : nf.blocks)
                    if (!of.blocks.count(key) && blk.cols() > 0 && onr > 0 && blk.rows() >= onr &&
                        !blk.topRows(onr).isZero(0.0))
                        ++violations;
            }
        }
        prev = *v.fronts;
        has_prev = true;
    }
};

struct PipeH {
    std::unique_ptr<Pipeline> p;
    std::unique_ptr<PhaseObs> obs;
    std::vector<int> owner;
};

struct TreeH {
    PatternGraph g;
    SeparatorTree t;
    ClusterHierarchy h;
    std::vector<Index> perm;
};

const Factorization& F_of(void* hv) { return *static_cast<PipeH*>(hv)->p->factorization(); }

}  // namespace

extern "C" {

int orc_default_num_levels(int n) { return default_num_levels(n); }

void* orc_pipeline_new(int m, int n, const int* colptr, const int* rowind, const double* vals, const double* coords,
                       int dim, const int* parts, int levels, double eps, int skip, int store_q, int solver,
                       int check_invariants, char* err, int errlen, int* err_code, int* err_cluster) {
    auto* H = new PipeH;
    *err_code = guarded(err, errlen, err_cluster, [&] {
        SparseMatrix A = make_csc(m, n, colptr, rowind, vals);
        PipelineOptions o;
        o.eps = eps;
        o.levels = levels;
        o.skip_levels = skip;
        o.store_q = store_q != 0;
        o.solver = static_cast<SolverKind>(solver);
        MatrixXd X;
        if (coords) {
            // row-major (n x dim) input, as the restatement takes it
            X = MatrixXd(n, dim);
            for (int i = 0; i < n; ++i)
                for (int d = 0; d < dim; ++d) X(i, d) = coords[static_cast<size_t>(i) * dim + d];
        }
        std::vector<int> pv;
        if (parts) pv.assign(parts, parts + n);
        H->obs = std::make_unique<PhaseObs>();
        H->obs->M = m;
        H->obs->check = check_invariants != 0;
        // The observer needs the hierarchy, which the pipeline builds before it
        // factorizes; reach it through the object under construction.
        struct Shim : FactorizeObserver {
            PhaseObs* o;
            Pipeline* pp;
            void on_phase(const char* ph, int s, int d, const EngineView& v) override {
                if (!o->h) o->h = &pp->hierarchy();
                o->on_phase(ph, s, d, v);
            }
        } shim;
        void* mem = ::operator new(sizeof(Pipeline));
        shim.o = H->obs.get();
        shim.pp = static_cast<Pipeline*>(mem);
        try {
            new (mem) Pipeline(A, o, coords ? &X : nullptr, parts ? &pv : nullptr, &shim);
        } catch (...) {
            ::operator delete(mem);
            throw;
        }
        H->p.reset(static_cast<Pipeline*>(mem));
        H->obs->h = nullptr;
        const Pipeline& P = *H->p;
        if (P.factorization()) {  // pipeline.cpp:52-53 (owner is not kept by Pipeline)
            const RowMatching mm = match_rows(P.scaled());
            H->owner = assign_rows(P.scaled(), P.hierarchy(), mm);
        } else {
            H->owner.assign(m, -1);
        }
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
    const Factorization* F = P.factorization();
    o[0] = P.rows();
    o[1] = P.cols();
    o[2] = P.hierarchy().num_levels;
    o[3] = static_cast<long long>(P.hierarchy().clusters.size());
    o[4] = F ? static_cast<long long>(F->W.size()) : 0;
    o[5] = F ? static_cast<long long>(F->Q.size()) : 0;
    o[6] = F ? static_cast<long long>(F->dropped_rows.size()) : 0;
    o[7] = F ? static_cast<long long>(F->trailing_rows.size()) : 0;
    o[8] = F ? static_cast<long long>(F->stages.size()) : 0;
    o[9] = F ? F->nnz_w() : 0;
    o[10] = P.scaled().nnz();
    o[11] = H->obs->check ? H->obs->violations : -1;
    o[12] = static_cast<long long>(H->obs->phases.size());
}

void orc_pipeline_times(void* hv, double* o) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    o[0] = P.timings().t_partition;
    o[1] = P.timings().t_factorize;
}

void orc_pipeline_perm(void* hv, int* o) {
    const auto& p = static_cast<PipeH*>(hv)->p->permutation();
    std::copy(p.begin(), p.end(), o);
}
void orc_pipeline_owner(void* hv, int* o) {
    const auto& w = static_cast<PipeH*>(hv)->owner;
    std::copy(w.begin(), w.end(), o);
}
void orc_pipeline_weights(void* hv, double* o) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    for (Index i = 0; i < P.cols(); ++i) o[i] = P.column_norms()[P.permutation()[i]];
}
void orc_pipeline_scaled(void* hv, int* p, int* i, double* x) {
    const SparseMatrix& A = static_cast<PipeH*>(hv)->p->scaled();
    std::copy(A.outer(), A.outer() + A.cols() + 1, p);
    std::copy(A.inner(), A.inner() + A.nnz(), i);
    std::copy(A.values(), A.values() + A.nnz(), x);
}
void orc_pipeline_rows(void* hv, int* pivot_row, int* dropped, int* trailing) {
    const Factorization& F = F_of(hv);
    std::copy(F.pivot_row.begin(), F.pivot_row.end(), pivot_row);
    std::copy(F.dropped_rows.begin(), F.dropped_rows.end(), dropped);
    std::copy(F.trailing_rows.begin(), F.trailing_rows.end(), trailing);
}
void orc_pipeline_cluster(void* hv, int c, int* info) {
    const auto& C = static_cast<PipeH*>(hv)->p->hierarchy().clusters[c];
    info[0] = C.tree_node;
    info[1] = C.level;
    info[2] = C.parent;
    info[3] = C.stage;
    info[4] = C.interior;
    info[5] = static_cast<int>(C.cols.size());
}
void orc_pipeline_cluster_cols(void* hv, int c, int* o) {
    const auto& C = static_cast<PipeH*>(hv)->p->hierarchy().clusters[c];
    std::copy(C.cols.begin(), C.cols.end(), o);
}
void orc_pipeline_stage(void* hv, int s, long long* o, double* t) {
    const auto& st = F_of(hv).stages[s];
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
    const auto& st = F_of(hv).stages[s];
    std::copy(st.front_cols.begin(), st.front_cols.end(), cols);
    std::copy(st.front_aspect.begin(), st.front_aspect.end(), aspect);
}
void orc_pipeline_phase(void* hv, int i, char* name, int namelen, int* stage, int* detail) {
    auto* H = static_cast<PipeH*>(hv);
    put_err(name, namelen, H->obs->phases[i]);
    *stage = H->obs->stages[i];
    *detail = H->obs->details[i];
}
void orc_pipeline_wfactor(void* hv, int i, int* o) {
    const auto& f = F_of(hv).W[i];
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
void orc_pipeline_wfactor_data(void* hv, int i, int* cols, double* a, int* coupled, double* b, double* c) {
    const auto& f = F_of(hv).W[i];
    if (const auto* t = std::get_if<TriangularScale>(&f)) {
        std::copy(t->cols.begin(), t->cols.end(), cols);
        copy_mat(t->R, a);
        std::copy(t->coupled.begin(), t->coupled.end(), coupled);
        copy_mat(t->C, b);
    } else {
        const auto& r = std::get<ColumnRotation>(f);
        std::copy(r.cols.begin(), r.cols.end(), cols);
        copy_mat(r.Q.V, a);
        copy_mat(r.Q.tau, b);
        copy_mat(r.Q.sign, c);
    }
}

namespace {
void apply_mode(const Factorization& F, int mode, VectorXd& v) {
    switch (mode) {
        case 0: F.w_apply(v); break;
        case 1: F.w_solve(v); break;
        case 2: F.wt_apply(v); break;
        case 3: F.wt_solve(v); break;
        case 4: F.q_apply_t(v); break;
        case 5: F.q_apply(v); break;
        default: throw std::invalid_argument("bad mode");
    }
}
}  // namespace

int orc_pipeline_apply(void* hv, int mode, double* z, char* err, int errlen) {
    int cl = -1;
    return guarded(err, errlen, &cl, [&] {
        const Factorization& F = F_of(hv);
        const Index n = (mode >= 4) ? F.M : F.N;
        VectorXd v = Eigen::Map<VectorXd>(z, n);
        apply_mode(F, mode, v);
        std::copy(v.data(), v.data() + n, z);
    });
}

int orc_pipeline_save(void* hv, const char* path, char* err, int errlen) {
    int cl = -1;
    return guarded(err, errlen, &cl, [&] { save_factorization(F_of(hv), path); });
}

int orc_factor_file_apply(const char* path, int mode, double* z, long long nz, long long* dims, char* err, int errlen) {
    int cl = -1;
    return guarded(err, errlen, &cl, [&] {
        const Factorization F = load_factorization(path);
        dims[0] = F.M;
        dims[1] = F.N;
        dims[2] = static_cast<long long>(F.W.size());
        if (!z) return;
        const Index n = (mode >= 4) ? F.M : F.N;
        if (static_cast<long long>(n) != nz) throw std::invalid_argument("vector length does not match the factorization");
        VectorXd v = Eigen::Map<VectorXd>(z, n);
        apply_mode(F, mode, v);
        std::copy(v.data(), v.data() + n, z);
    });
}

int orc_pipeline_solve(void* hv, int direct, const double* b, double* x, double tol, int maxit, int* iters,
                       int* converged, double* hist, int* nhist, double* t_solve, char* err, int errlen) {
    const Pipeline& P = *static_cast<PipeH*>(hv)->p;
    int cl = -1;
    return guarded(err, errlen, &cl, [&] {
        VectorXd bb = Eigen::Map<VectorXd>(const_cast<double*>(b), P.rows());
        SolveReport rep;
        VectorXd xx = direct ? P.solve_direct(bb, &rep) : P.solve(bb, &rep, tol, maxit);
        std::copy(xx.data(), xx.data() + xx.size(), x);
        *iters = rep.iterations;
        *converged = rep.converged;
        *nhist = static_cast<int>(rep.residual_history.size());
        std::copy(rep.residual_history.begin(), rep.residual_history.end(), hist);
        *t_solve = rep.t_solve;
    });
}

int orc_cgls_plain(int m, int n, const int* p, const int* i, const double* v, const double* b, const double* weights,
                   double tol, int maxit, double* x, int* iters, int* converged, double* hist, int* nhist) {
    SparseMatrix A = make_csc(m, n, p, i, v);
    VectorXd bb = Eigen::Map<VectorXd>(const_cast<double*>(b), m), w;
    if (weights) w = Eigen::Map<VectorXd>(const_cast<double*>(weights), n);
    CglsOptions co;
    co.tol = tol;
    co.maxit = maxit;
    VectorXd u;
    SolveReport rep = cgls(A, nullptr, bb, u, co, weights ? &w : nullptr);
    std::copy(u.data(), u.data() + u.size(), x);
    *iters = rep.iterations;
    *converged = rep.converged;
    *nhist = static_cast<int>(rep.residual_history.size());
    std::copy(rep.residual_history.begin(), rep.residual_history.end(), hist);
    return 0;
}

// -------------------------------------------------------- dense kernels ---
void orc_householder_qr(int m, int n, const double* B, double* V, double* tau, double* sign, double* R) {
    ReflectorSet H;
    MatrixXd Rm;
    block_householder_qr(make_mat(m, n, B), H, Rm);
    copy_mat(H.V, V);
    copy_mat(H.tau, tau);
    copy_mat(H.sign, sign);
    copy_mat(Rm, R);
}

void orc_apply_reflectors(int m, int k, const double* V, const double* tau, const double* sign, int mode, int xr,
                          int xc, double* X) {
    ReflectorSet H;
    H.V = make_mat(m, k, V);
    H.tau = make_mat(k, 1, tau);
    H.sign = make_mat(k, 1, sign);
    MatrixXd Xm = make_mat(xr, xc, X);
    if (mode == 0) apply_reflectors_left_t(H, Xm);
    if (mode == 1) apply_reflectors_left(H, Xm);
    if (mode == 2) apply_reflectors_right(H, Xm);
    if (mode == 3) apply_reflectors_right_t(H, Xm);
    copy_mat(Xm, X);
}

void orc_cpqr(int m, int n, const double* B, double eps, int* rank, double* r11, int* perm, double* R, double* V,
              double* tau, double* sign) {
    TruncatedQR T = truncated_cpqr(make_mat(m, n, B), eps);
    *rank = T.rank;
    *r11 = T.r11;
    std::copy(T.perm.begin(), T.perm.end(), perm);
    copy_mat(T.R, R);
    copy_mat(T.H.V, V);
    copy_mat(T.H.tau, tau);
    copy_mat(T.H.sign, sign);
}

int orc_tri_solve(int n, const double* R, int br, int bc, double* B, int side_right, int transpose, char* err, int errlen) {
    int cl = 0;
    return guarded(err, errlen, &cl, [&] {
        MatrixXd Rm = make_mat(n, n, R);
        MatrixXd Bm = make_mat(br, bc, B);
        tri_solve_upper(Rm, Bm, side_right ? Side::Right : Side::Left, transpose != 0);
        copy_mat(Bm, B);
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
        MatrixXd X;
        if (coords) {
            X = MatrixXd(n, dim);
            for (int i = 0; i < n; ++i)
                for (int d = 0; d < dim; ++d) X(i, d) = coords[static_cast<size_t>(i) * dim + d];
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
    SparseMatrix A = make_csc(m, n, p, i, x);
    RowMatching mm = match_rows(A);
    std::vector<int> own = assign_rows(A, T->h, mm);
    std::copy(own.begin(), own.end(), owner);
    std::copy(mm.row_of_col.begin(), mm.row_of_col.end(), row_of_col);
    std::copy(mm.col_of_row.begin(), mm.col_of_row.end(), col_of_row);
    return mm.size;
}
int orc_match_rows(int m, int n, const int* p, const int* i, const double* x, int* row_of_col, int* col_of_row) {
    SparseMatrix A = make_csc(m, n, p, i, x);
    RowMatching mm = match_rows(A);
    std::copy(mm.row_of_col.begin(), mm.row_of_col.end(), row_of_col);
    std::copy(mm.col_of_row.begin(), mm.col_of_row.end(), col_of_row);
    return mm.size;
}

long long orc_ata_graph(int m, int n, const int* p, const int* i, const double* x, int* adjptr, int* adj) {
    SparseMatrix A = make_csc(m, n, p, i, x);
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

int orc_from_triplets(int m, int n, int nt, const int* r, const int* c, const double* v, int* p, int* i, double* x) {
    std::vector<Eigen::Triplet<double>> t;
    t.reserve(nt);
    for (int k = 0; k < nt; ++k) t.emplace_back(r[k], c[k], v[k]);
    SparseMatrix A = SparseMatrix::from_triplets(m, n, t);
    if (p) {
        std::copy(A.outer(), A.outer() + n + 1, p);
        std::copy(A.inner(), A.inner() + A.nnz(), i);
        std::copy(A.values(), A.values() + A.nnz(), x);
    }
    return A.nnz();
}

}  // extern "C"
