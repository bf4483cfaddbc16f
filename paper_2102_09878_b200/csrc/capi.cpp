// C ABI (include/spaqr_b200.h) over the B200 spaQR implementation: the
// Pipeline mirror (proj/src/pipeline.cpp) with host partitioning and the GPU
// engine / solver, plus batched dense-kernel entry points.
#include "../../include/spaqr_b200.h"

#include <algorithm>
#include <climits>
#include <cmath>
#include <cstring>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <numeric>
#include <string>
#ifdef _OPENMP
#include <omp.h>
#endif

#include "capi_common.h"
#include "dev.h"
#include "engine.h"
#include "solve.h"

using namespace spqr;

struct spqr_pipeline {
    int device = 0;
    cudaStream_t st = nullptr;
    double eps = 1e-2;
    int levels = 0, skip = 3, solver = SPQR_SOLVER_SPAQR, refine = 1, maxit = 500;
    double tol = 1e-12;
    Csc Aw;
    std::vector<double> d, weights;
    std::vector<Index> perm;
    std::vector<int> owner;
    SeparatorTree tree;
    ClusterHierarchy h;
    bool has_f = false;
    DeviceFactorization F;
    SolvePlan plan;
    QSweep qs;  // store_q: q_apply / q_apply_t
    DevMatrix dA;
    CglsWork ws;
    double* d_w = nullptr;
    double *d_b = nullptr, *d_u = nullptr;
    std::unique_ptr<DeviceArena> mem;
    double t_partition = 0, t_factorize = 0, t_upload = 0;
    double ev_factorize_ms = 0, ev_solve_ms = 0;  // CUDA events on the pipeline stream
    long long solve_launches = 0;
    double sweep_ms = 0;  // W sweeps of the last solve (CUDA events)
    int sweeps = 0;
    ~spqr_pipeline() {
        if (st) cudaStreamDestroy(st);
    }
};

namespace {

template <class F>
int guarded(char* err, int errlen, int* err_cluster, F&& f) {
    return capi_guarded(err, errlen, err_cluster, std::forward<F>(f));
}

int create_impl(int m, int n, const int* colptr, const int* rowind, const double* vals, const double* coords, int dim,
                const int* parts, int levels, double eps, int skip_levels, int solver, int store_q, int ranks, int device,
                spqr_observer_fn obs, void* obs_user, const DistTransport* dist, spqr_pipeline** out, char* err,
                int errlen, int* err_cluster);

}  // namespace

extern "C" {

const char* spqr_version(void) { return "spaqr_b200 0.1 (sm_100a)"; }

int spqr_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) return 0;
    return n;
}

int spqr_pipeline_create(int m, int n, const int* colptr, const int* rowind, const double* vals, const double* coords,
                         int dim, const int* parts, int levels, double eps, int skip_levels, int solver, int device,
                         spqr_pipeline** out, char* err, int errlen, int* err_cluster) {
    return spqr_pipeline_create_observed(m, n, colptr, rowind, vals, coords, dim, parts, levels, eps, skip_levels, solver,
                                         device, nullptr, nullptr, out, err, errlen, err_cluster);
}

int spqr_pipeline_create_observed(int m, int n, const int* colptr, const int* rowind, const double* vals,
                                  const double* coords, int dim, const int* parts, int levels, double eps,
                                  int skip_levels, int solver, int device, spqr_observer_fn obs, void* obs_user,
                                  spqr_pipeline** out, char* err, int errlen, int* err_cluster) {
    return spqr_pipeline_create_ex(m, n, colptr, rowind, vals, coords, dim, parts, levels, eps, skip_levels, solver, 0,
                                   1, device, obs, obs_user, out, err, errlen, err_cluster);
}

int spqr_pipeline_create_ex(int m, int n, const int* colptr, const int* rowind, const double* vals,
                            const double* coords, int dim, const int* parts, int levels, double eps, int skip_levels,
                            int solver, int store_q, int ranks, int device, spqr_observer_fn obs, void* obs_user,
                            spqr_pipeline** out, char* err, int errlen, int* err_cluster) {
    return create_impl(m, n, colptr, rowind, vals, coords, dim, parts, levels, eps, skip_levels, solver, store_q, ranks,
                       device, obs, obs_user, nullptr, out, err, errlen, err_cluster);
}

int spqr_pipeline_create_dist(int m, int n, const int* colptr, const int* rowind, const double* vals,
                              const double* coords, int dim, const int* parts, int levels, double eps, int skip_levels,
                              int device, int rank, int nranks, spqr_send_fn send, spqr_recv_fn recv, void* user,
                              spqr_pipeline** out, char* err, int errlen, int* err_cluster) {
    DistTransport t;
    t.user = user;
    t.rank = rank;
    t.size = nranks;
    t.send = send;
    t.recv = recv;
    if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && (!send || !recv))) {
        *out = nullptr;
        if (err && errlen > 0) std::snprintf(err, errlen, "bad rank / transport");
        return SPQR_E_SHAPE;
    }
    return create_impl(m, n, colptr, rowind, vals, coords, dim, parts, levels, eps, skip_levels, SPQR_SOLVER_SPAQR, 0, 1,
                       device, nullptr, nullptr, nranks > 1 ? &t : nullptr, out, err, errlen, err_cluster);
}

void spqr_pipeline_dist_info(const spqr_pipeline* p, double* out3) {
    out3[0] = p->F.dist_partial ? 1.0 : 0.0;
    out3[1] = p->F.dist_exchange_s;
    out3[2] = static_cast<double>(p->F.dist_bytes);
}

}  // extern "C"

namespace {
int create_impl(int m, int n, const int* colptr, const int* rowind, const double* vals, const double* coords, int dim,
                const int* parts, int levels, double eps, int skip_levels, int solver, int store_q, int ranks, int device,
                spqr_observer_fn obs, void* obs_user, const DistTransport* dist, spqr_pipeline** out, char* err,
                int errlen, int* err_cluster) {
    *out = nullptr;
    auto* P = new spqr_pipeline;
    const int rc = guarded(err, errlen, err_cluster, [&] {
        capi_set_threads();  // 15 host threads on the 16-core hosts: 3.4 s vs 3.7 s at 12 (C2)
        P->device = device;
        CK(cudaSetDevice(device));
        CK(cudaStreamCreateWithFlags(&P->st, cudaStreamNonBlocking));
        P->eps = (solver == SPQR_SOLVER_DIRECT) ? 0.0 : eps;  // pipeline.cpp:24
        P->levels = levels;
        P->skip = skip_levels;
        P->solver = solver;
        P->Aw = csc_canonical(m, n, colptr, rowind, vals);
        if (P->Aw.m < P->Aw.n) throw std::invalid_argument("matrix must have at least as many rows as columns");
        P->d = scale_columns(P->Aw);
        P->mem = std::make_unique<DeviceArena>(size_t(32) << 20);
        if (solver == SPQR_SOLVER_DIAG) {
            P->perm.resize(n);
            std::iota(P->perm.begin(), P->perm.end(), 0);
            P->weights = P->d;
        } else {
            double t0 = now_s();
            double tp[8];
            int np_ = 0;
            tp[np_++] = now_s();
            const Graph g = ata_graph(P->Aw);
            tp[np_++] = now_s();
            const int L = levels > 0 ? levels : default_num_levels(n);
            if (parts) {
                P->tree = import_partition(g, L, parts);
            } else {
                if (coords && dim <= 0) throw std::invalid_argument("coordinate dimension must be positive");
                P->tree = nested_dissection(g, L, coords, dim);
            }
            tp[np_++] = now_s();
            P->h = build_interfaces(P->tree, g);
            tp[np_++] = now_s();
            P->perm = order_columns(P->h);
            P->Aw = permute_columns(P->Aw, P->perm);
            tp[np_++] = now_s();
            const RowMatching mm = match_rows(P->Aw);
            tp[np_++] = now_s();
            P->owner = assign_rows(P->Aw, P->h, mm);
            tp[np_++] = now_s();
            P->t_partition = now_s() - t0;
            if (std::getenv("SPQR_PROF"))
                std::fprintf(stderr,
                             "[spqr prof] partition: ata_graph %.3f nested_dissection %.3f build_interfaces %.3f "
                             "order+permute %.3f match_rows %.3f assign_rows %.3f s\n",
                             tp[1] - tp[0], tp[2] - tp[1], tp[3] - tp[2], tp[4] - tp[3], tp[5] - tp[4], tp[6] - tp[5]);
            P->weights.resize(n);
            for (int i = 0; i < n; ++i) P->weights[i] = P->d[P->perm[i]];
            t0 = now_s();
            FactorizeOptions fo;
            fo.eps = P->eps;
            fo.skip_levels = skip_levels;
            fo.store_q = store_q != 0;
            fo.ranks = std::max(1, ranks);
            fo.dist = dist;
            cudaEvent_t e0, e1;
            CK(cudaEventCreate(&e0));
            CK(cudaEventCreate(&e1));
            CK(cudaEventRecord(e0, P->st));
            const FactorizeObserver ob = make_observer(obs, obs_user);
            P->F = gpu_factorize(P->Aw, P->h, P->owner, fo, P->st, obs ? &ob : nullptr);
            if (!P->F.dist_partial) P->plan = build_solve_plan(P->F, P->st);
            CK(cudaEventRecord(e1, P->st));
            CK(cudaEventSynchronize(e1));
            float ms = 0.f;
            CK(cudaEventElapsedTime(&ms, e0, e1));
            P->ev_factorize_ms = ms;
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            P->has_f = !P->F.dist_partial;  // ranks > 0 of a distributed factorization hold none
            P->t_factorize = now_s() - t0;
        }
        const double t0 = now_s();
        P->dA = upload_matrix(P->Aw, P->st);
        P->ws = make_cgls_work(P->Aw.m, P->Aw.n);
        P->d_w = P->mem->alloc_n<double>(std::max(n, 1));
        P->d_b = P->mem->alloc_n<double>(std::max(m, 1));
        P->d_u = P->mem->alloc_n<double>(std::max(n, 1));
        CK(cudaMemcpyAsync(P->d_w, P->weights.data(), sizeof(double) * n, cudaMemcpyHostToDevice, P->st));
        CK(cudaStreamSynchronize(P->st));
        P->t_upload = now_s() - t0;
    });
    if (rc != SPQR_OK) {
        delete P;
        return rc;
    }
    *out = P;
    return SPQR_OK;
}

}  // namespace

extern "C" {

void spqr_pipeline_destroy(spqr_pipeline* p) { delete p; }

void spqr_pipeline_info(const spqr_pipeline* p, long long* o) {
    std::fill(o, o + 16, 0LL);
    o[0] = p->Aw.m;
    o[1] = p->Aw.n;
    o[2] = p->h.num_levels;
    o[3] = static_cast<long long>(p->h.clusters.size());
    o[4] = static_cast<long long>(p->F.W.size());
    o[5] = static_cast<long long>(p->F.dropped_rows.size());
    o[6] = static_cast<long long>(p->F.trailing_rows.size());
    o[7] = static_cast<long long>(p->F.stages.size());
    o[8] = p->F.nnz_w();
    o[9] = p->Aw.nnz();
    o[10] = static_cast<long long>(p->plan.sched[kWSolve].levels.size());
    o[11] = p->F.ctr.launches;
    o[12] = p->F.ctr.syncs;
    o[13] = p->F.ctr.h2d_bytes;
    o[14] = p->F.ctr.d2h_bytes;
    o[15] = p->plan.launches_per_sweep + p->plan.launches_per_sweep_t;
}

long long spqr_pipeline_nq(const spqr_pipeline* p) { return p->F.has_q ? static_cast<long long>(p->F.Q.size()) : -1; }

int spqr_pipeline_rank_stats(const spqr_pipeline* p, int* nstages, double* flops, double* cross, int* owner) {
    const RankStats& r = p->F.rank;
    if (r.ranks <= 1) return 0;
    const int ns = static_cast<int>(std::max(r.flops.size(), r.cross.size()));
    if (nstages) *nstages = ns;
    for (int s = 0; s < ns; ++s) {
        for (int q = 0; q < r.ranks; ++q)
            if (flops) flops[s * r.ranks + q] = s < static_cast<int>(r.flops.size()) ? r.flops[s][q] : 0.0;
        for (int q = 0; q < 4; ++q)
            if (cross) cross[s * 4 + q] = s < static_cast<int>(r.cross.size()) ? r.cross[s][q] : 0.0;
    }
    if (owner) std::copy(r.owner.begin(), r.owner.end(), owner);
    return r.ranks;
}

int spqr_rank_plan(int m, int n, const int* colptr, const int* rowind, const double* vals, const double* coords, int dim,
                   const int* parts, int levels, int nranks, int* nclusters, int* ntree, int* owner, int* cluster_node,
                   int* cluster_level, int* tree_parent, int* tree_level, char* err, int errlen) {
    int cl = -1;
    return guarded(err, errlen, &cl, [&] {
        Csc A = csc_canonical(m, n, colptr, rowind, vals);
        if (A.m < A.n) throw std::invalid_argument("matrix must have at least as many rows as columns");
        scale_columns(A);
        const Graph g = ata_graph(A);
        const int L = levels > 0 ? levels : default_num_levels(n);
        if (coords && dim <= 0) throw std::invalid_argument("coordinate dimension must be positive");
        const SeparatorTree t = parts ? import_partition(g, L, parts) : nested_dissection(g, L, coords, dim);
        ClusterHierarchy h = build_interfaces(t, g);
        const std::vector<int> own = rank_owners(h, g, nranks);
        if (nclusters) *nclusters = static_cast<int>(h.clusters.size());
        if (ntree) *ntree = static_cast<int>(t.nodes.size());
        for (size_t c = 0; c < h.clusters.size(); ++c) {
            if (owner) owner[c] = own[c];
            if (cluster_node) cluster_node[c] = h.clusters[c].tree_node;
            if (cluster_level) cluster_level[c] = h.clusters[c].level;
        }
        for (size_t v = 0; v < t.nodes.size(); ++v) {
            if (tree_parent) tree_parent[v] = t.nodes[v].parent;
            if (tree_level) tree_level[v] = t.nodes[v].level;
        }
    });
}

void spqr_pipeline_times(const spqr_pipeline* p, double* t) {
    std::fill(t, t + 24, 0.0);
    t[0] = p->t_partition;
    t[1] = p->t_factorize;
    t[2] = p->t_upload;
    t[3] = p->F.ctr.t_qr_ms;
    t[4] = p->F.ctr.qr_flops;
    t[5] = p->F.ctr.qr_bytes;
    t[6] = p->F.ctr.cpqr_flops;
    t[7] = p->F.ctr.cpqr_bytes;
    t[8] = static_cast<double>(p->F.ctr.qr_launches);
    t[9] = p->ev_factorize_ms;
    t[10] = p->ev_solve_ms;
    t[11] = static_cast<double>(p->solve_launches);
    t[12] = static_cast<double>(p->F.ctr.elim_waves);
    t[13] = p->F.ctr.cpqr_redundant_bytes;
    t[14] = p->F.ctr.cpqr_redundant_flops;
    t[15] = p->sweep_ms;
    t[16] = static_cast<double>(p->sweeps);
    t[17] = p->plan.sweep_bytes;
    t[18] = p->plan.t_build;
    t[19] = static_cast<double>(p->plan.sched[kWSolve].levels.size());
    t[20] = static_cast<double>(p->plan.sched[kWtSolve].levels.size());
}

void spqr_pipeline_kernel_stats(const spqr_pipeline* p, double* ms, double* bytes, long long* launches) {
    for (int t = 0; t < K_NTAGS; ++t) {
        ms[t] = p->F.ctr.k_ms[t];
        bytes[t] = p->F.ctr.k_bytes[t];
        launches[t] = p->F.ctr.k_launches[t];
    }
}

int spqr_pipeline_solve(spqr_pipeline* p, int direct, const double* b, double* x, double tol, int maxit, int* iters,
                        int* converged, double* hist, int* nhist, double* t_solve, char* err, int errlen) {
    int cl = -1;
    return guarded(err, errlen, &cl, [&] {
        if (p->F.dist_partial) throw std::logic_error("this rank's part of the factorization was sent to rank 0");
        if (direct && !p->has_f) throw std::logic_error("direct solve requires a factorization");
        CK(cudaSetDevice(p->device));
        const int m = p->Aw.m, n = p->Aw.n;
        const double t0 = now_s();
        CK(cudaMemcpyAsync(p->d_b, b, sizeof(double) * m, cudaMemcpyHostToDevice, p->st));
        SolveReport rep;
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, p->st));
        if (direct)
            rep = gpu_csne(p->dA, p->plan, p->d_b, p->d_u, p->refine, p->d_w, p->tol, p->ws, p->st);
        else
            rep = gpu_cgls(p->dA, p->has_f ? &p->plan : nullptr, p->d_b, p->d_u, tol > 0 ? tol : p->tol,
                           maxit > 0 ? maxit : p->maxit, p->d_w, p->ws, p->st);
        CK(cudaEventRecord(e1, p->st));
        CK(cudaEventSynchronize(e1));
        float ms = 0.f;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        p->ev_solve_ms = ms;
        p->solve_launches = rep.launches;
        p->sweep_ms = rep.sweep_ms;
        p->sweeps = rep.sweeps;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        std::vector<double> u(n);
        CK(cudaMemcpyAsync(u.data(), p->d_u, sizeof(double) * n, cudaMemcpyDeviceToHost, p->st));
        CK(cudaStreamSynchronize(p->st));
        for (int i = 0; i < n; ++i) x[p->perm[i]] = u[i] / p->d[p->perm[i]];  // pipeline.cpp:65-68
        *iters = rep.iterations;
        *converged = rep.converged;
        *nhist = static_cast<int>(rep.residual_history.size());
        std::copy(rep.residual_history.begin(), rep.residual_history.end(), hist);
        *t_solve = now_s() - t0;
    });
}

int spqr_pipeline_apply(spqr_pipeline* p, int mode, double* z) {
    int cl = -1;
    return guarded(nullptr, 0, &cl, [&] {
        CK(cudaSetDevice(p->device));
        if (mode == SPQR_Q_APPLY_T || mode == SPQR_Q_APPLY) {
            if (!p->has_f) throw std::logic_error("no factorization");
            q_sweep(p->F, p->qs, mode, z, p->st);
            return;
        }
        if (mode < 0 || mode > 3) throw std::invalid_argument("unknown apply mode");
        const int n = p->Aw.n;
        CK(cudaMemcpyAsync(p->d_u, z, sizeof(double) * n, cudaMemcpyHostToDevice, p->st));
        static const SweepMode map[4] = {kWApply, kWSolve, kWtApply, kWtSolve};
        if (p->has_f) {
            ensure_schedule(p->plan, p->F, map[mode & 3], p->st);
            sweep(p->plan, map[mode & 3], p->d_u, p->st);
        }
        CK(cudaMemcpyAsync(z, p->d_u, sizeof(double) * n, cudaMemcpyDeviceToHost, p->st));
        CK(cudaStreamSynchronize(p->st));
    });
}

int spqr_pipeline_tree(const spqr_pipeline* p, int* parent, int* root) {
    const int nt = static_cast<int>(p->tree.nodes.size());
    if (parent)
        for (int t = 0; t < nt; ++t) parent[t] = p->tree.nodes[t].parent;
    if (root) *root = p->tree.root;
    return nt;
}

void spqr_pipeline_finest(const spqr_pipeline* p, int* finest_of_col) {
    std::copy(p->h.finest_of_col.begin(), p->h.finest_of_col.end(), finest_of_col);
}

void spqr_pipeline_scaled(const spqr_pipeline* p, int* colptr, int* rowind, double* vals) {
    std::copy(p->Aw.p.begin(), p->Aw.p.end(), colptr);
    std::copy(p->Aw.i.begin(), p->Aw.i.end(), rowind);
    std::copy(p->Aw.x.begin(), p->Aw.x.end(), vals);
}

void spqr_pipeline_perm(const spqr_pipeline* p, int* o) { std::copy(p->perm.begin(), p->perm.end(), o); }
void spqr_pipeline_owner(const spqr_pipeline* p, int* o) { std::copy(p->owner.begin(), p->owner.end(), o); }
void spqr_pipeline_weights(const spqr_pipeline* p, double* o) { std::copy(p->weights.begin(), p->weights.end(), o); }
void spqr_pipeline_rows(const spqr_pipeline* p, int* pr, int* dr, int* tr) {
    std::copy(p->F.pivot_row.begin(), p->F.pivot_row.end(), pr);
    std::copy(p->F.dropped_rows.begin(), p->F.dropped_rows.end(), dr);
    std::copy(p->F.trailing_rows.begin(), p->F.trailing_rows.end(), tr);
}
void spqr_pipeline_cluster(const spqr_pipeline* p, int c, int* info) {
    const auto& C = p->h.clusters[c];
    info[0] = C.tree_node;
    info[1] = C.level;
    info[2] = C.parent;
    info[3] = C.stage;
    info[4] = C.interior;
    info[5] = static_cast<int>(C.cols.size());
}
void spqr_pipeline_cluster_cols(const spqr_pipeline* p, int c, int* o) {
    std::copy(p->h.clusters[c].cols.begin(), p->h.clusters[c].cols.end(), o);
}
void spqr_pipeline_stage(const spqr_pipeline* p, int s, long long* o, double* t) {
    const StageStats& st = p->F.stages[s];
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
void spqr_pipeline_stage_fronts(const spqr_pipeline* p, int s, int* cols, double* aspect) {
    const StageStats& st = p->F.stages[s];
    std::copy(st.front_cols.begin(), st.front_cols.end(), cols);
    std::copy(st.front_aspect.begin(), st.front_aspect.end(), aspect);
}
void spqr_pipeline_wfactor(const spqr_pipeline* p, int i, int* o) {
    const DevWFactor& w = p->F.W[i];
    o[0] = w.kind;
    o[1] = w.c;
    o[2] = w.k;
    o[3] = w.batch;
}
int spqr_pipeline_wfactor_data(const spqr_pipeline* p, int i, int* cols, double* a, int* coupled, double* b, double* c) {
    int cl = -1;
    return guarded(nullptr, 0, &cl, [&] {
        const DevWFactor& w = p->F.W[i];
        std::copy(p->F.idx.begin() + w.cols_off, p->F.idx.begin() + w.cols_off + w.c, cols);
        if (w.kind == 0) {
            std::copy(p->F.idx.begin() + w.coupled_off, p->F.idx.begin() + w.coupled_off + w.k, coupled);
            std::vector<double> buf(static_cast<size_t>(w.c) * (w.c + w.k));
            if (!buf.empty()) CK(cudaMemcpy(buf.data(), w.a, sizeof(double) * buf.size(), cudaMemcpyDeviceToHost));
            std::copy(buf.begin(), buf.begin() + static_cast<long long>(w.c) * w.c, a);
            std::copy(buf.begin() + static_cast<long long>(w.c) * w.c, buf.end(), b);
        } else {
            if (w.c * w.k > 0) CK(cudaMemcpy(a, w.a, sizeof(double) * w.c * w.k, cudaMemcpyDeviceToHost));
            if (w.k > 0) {
                CK(cudaMemcpy(b, w.tau, sizeof(double) * w.k, cudaMemcpyDeviceToHost));
                CK(cudaMemcpy(c, w.sign, sizeof(double) * w.k, cudaMemcpyDeviceToHost));
            }
        }
    });
}

// save_factorization (transforms.cpp:206-240): the device-resident W written in
// the reference's SPQRFW01 layout (little-endian int64 sizes and indices, IEEE
// doubles; TriangularScale = tag 0: cols, R, coupled, C; ColumnRotation = tag
// 1: cols, V, tau, sign; no Q part).  The W arena is mirrored to the host with
// one copy per arena chunk.
int spqr_pipeline_save(const spqr_pipeline* p, const char* path, char* err, int errlen) {
    int cl = -1;
    return guarded(err, errlen, &cl, [&] {
        if (!p->has_f) throw std::logic_error("spqr_pipeline_save: no factorization (solver=direct)");
        save_device_factorization(p->F, path);
    });
}

// ------------------------------------------------------------ dense kernels
int spqr_qr_apply_batched_dev(int nb, int m, int n, int ntot, double* d_a, double* d_tau, double* d_sign, int* d_info,
                              float* ms) {
    int cl = -1;
    return guarded(nullptr, 0, &cl, [&] {
        if (n > m || ntot < n) throw std::invalid_argument("qr: need n <= m and n <= ntot");
        std::vector<int> init(nb, INT_MAX);
        CK(cudaMemcpy(d_info, init.data(), sizeof(int) * nb, cudaMemcpyHostToDevice));
        // path: column-tiled (default when the panel fits), smem-staged, or blocked DMMA;
        // SPQR_QR_PATH=tile|smem|blocked forces one (comparisons, tests)
        const char* force = std::getenv("SPQR_QR_PATH");
        const std::string fp = force ? force : "";
        const int tcls = qr_tile_class(m, n);
        const bool tile = (fp.empty() || fp == "tile") && tcls >= 0;
        const bool staged = !tile && fp != "blocked" && qr_smem_bytes(m, n, ntot) <= kSmemBudget && n <= 1024;
        QrDesc* dq = nullptr;
        int4* dwork = nullptr;
        int nwork = 0;
        int* didx = nullptr;
        double* dT = nullptr;
        if (tile) {
            std::vector<QrDesc> qd(nb);
            for (int b = 0; b < nb; ++b)
                qd[b] = QrDesc{d_a + static_cast<long long>(b) * m * ntot, m, m, n, ntot, d_tau + static_cast<long long>(b) * n,
                               d_sign + static_cast<long long>(b) * n, nullptr, d_info + b, 0, 0};
            std::vector<int> all(nb);
            for (int b = 0; b < nb; ++b) all[b] = b;
            const std::vector<int4> wk = qr_tile_plan(qd.data(), all.data(), nb, sm_count());
            nwork = static_cast<int>(wk.size());
            CK(cudaMalloc(&dq, sizeof(QrDesc) * std::max(nb, 1)));
            CK(cudaMalloc(&dwork, sizeof(int4) * std::max(nwork, 1) + sizeof(int) * std::max(nb, 1)));
            CK(cudaMemset(dwork, 0, sizeof(int4) * std::max(nwork, 1) + sizeof(int) * std::max(nb, 1)));
            CK(cudaMemcpy(dq, qd.data(), sizeof(QrDesc) * nb, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(dwork, wk.data(), sizeof(int4) * nwork, cudaMemcpyHostToDevice));
        } else if (staged) {
            std::vector<QrDesc> qd(nb);
            for (int b = 0; b < nb; ++b)
                qd[b] = QrDesc{d_a + static_cast<long long>(b) * m * ntot, m, m, n, ntot, d_tau + static_cast<long long>(b) * n,
                               d_sign + static_cast<long long>(b) * n, nullptr, d_info + b, 0, 0};
            std::vector<int> all(nb);
            for (int b = 0; b < nb; ++b) all[b] = b;
            CK(cudaMalloc(&dq, sizeof(QrDesc) * std::max(nb, 1)));
            CK(cudaMalloc(&didx, sizeof(int) * std::max(nb, 1)));
            CK(cudaMemcpy(dq, qd.data(), sizeof(QrDesc) * nb, cudaMemcpyHostToDevice));
            CK(cudaMemcpy(didx, all.data(), sizeof(int) * nb, cudaMemcpyHostToDevice));
        } else {
            CK(cudaMalloc(&dT, sizeof(double) * 32 * 32 * std::max(nb, 1)));
        }
        cudaEvent_t e0, e1;
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaEventRecord(e0, 0));
        if (tile && qr_wy_enabled() && qr_wy_ok(m, n, ntot))
            launch_qr_wy(dq, dwork, nwork, reinterpret_cast<int*>(dwork + std::max(nwork, 1)), 0);
        else if (tile)
            launch_qr_tile(tcls, dq, dwork, nwork, qr_tile_smem(tcls, n), reinterpret_cast<int*>(dwork + std::max(nwork, 1)), 0);
        else if (staged)
            launch_qr_split(dq, didx, nb, qr_smem_bytes(m, n, ntot), nullptr, 0, 0);
        else
            blocked_qr_apply(nb, m, n, ntot, d_a, d_tau, d_sign, d_info, dT, 0);
        CK(cudaEventRecord(e1, 0));
        CK(cudaEventSynchronize(e1));
        CK(cudaGetLastError());
        float t = 0.f;
        CK(cudaEventElapsedTime(&t, e0, e1));
        if (ms) *ms = t;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
        launch_info_fixup(d_info, nb, 0);
        CK(cudaStreamSynchronize(0));
        if (dq) cudaFree(dq);
        if (dwork) cudaFree(dwork);
        if (didx) cudaFree(didx);
        if (dT) cudaFree(dT);
    });
}

int spqr_qr_apply_batched(int nb, int m, int n, int ntot, double* a, double* tau, double* sign, int* info) {
    int cl = -1;
    return guarded(nullptr, 0, &cl, [&] {
        const size_t na = static_cast<size_t>(nb) * m * ntot;
        double *da = nullptr, *dt = nullptr, *ds = nullptr;
        int* di = nullptr;
        CK(cudaMalloc(&da, sizeof(double) * std::max<size_t>(na, 1)));
        CK(cudaMalloc(&dt, sizeof(double) * std::max(nb * n, 1)));
        CK(cudaMalloc(&ds, sizeof(double) * std::max(nb * n, 1)));
        CK(cudaMalloc(&di, sizeof(int) * std::max(nb, 1)));
        CK(cudaMemcpy(da, a, sizeof(double) * na, cudaMemcpyHostToDevice));
        float ms = 0;
        const int rc = spqr_qr_apply_batched_dev(nb, m, n, ntot, da, dt, ds, di, &ms);
        if (rc != SPQR_OK) throw std::runtime_error("qr launch failed");
        CK(cudaMemcpy(a, da, sizeof(double) * na, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(tau, dt, sizeof(double) * nb * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(sign, ds, sizeof(double) * nb * n, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(info, di, sizeof(int) * nb, cudaMemcpyDeviceToHost));
        for (int b = 0; b < nb; ++b)
            if (info[b] == INT_MAX) info[b] = -1;
        cudaFree(da);
        cudaFree(dt);
        cudaFree(ds);
        cudaFree(di);
    });
}

namespace {
// truncated CPQR of nb packed m x n problems already on the device (in place);
// per-problem outputs into the caller's device buffers; device time of the
// launches (events on the default stream) into *ms when given
void cpqr_dev_run(DeviceArena& mem, int nb, int m, int n, double* da, double eps, int* dr, double* d11, int* dp,
                  double* dV, double* dt, double* ds, float* ms) {
    const int kmax = std::min(m, n);
    const bool big = 8ull * m * n > kBigCpqrBytes && m >= 32 && cpqr_big_smem_bytes(m, n) <= 200 * 1024 &&
                     !(std::getenv("SPQR_CPQR_PATH") && std::string(std::getenv("SPQR_CPQR_PATH")) == "cluster");
    const size_t wstride = big ? cpqr_big_work_doubles(n) : 3 * static_cast<size_t>(n);
    double* work = mem.alloc_n<double>(std::max<size_t>(static_cast<size_t>(nb) * wstride, 1));
    CK(cudaMemset(dV, 0, sizeof(double) * static_cast<size_t>(nb) * m * kmax));
    std::vector<CpqrDesc> cd(nb);
    for (int b = 0; b < nb; ++b)
        cd[b] = CpqrDesc{da + static_cast<long long>(b) * m * n, m, m, n, eps, dr + b, d11 + b,
                         dV + static_cast<long long>(b) * m * kmax, m, dt + b * kmax, ds + b * kmax, dp + b * kmax,
                         work + static_cast<long long>(b) * wstride};
    CpqrDesc* dc = mem.alloc_n<CpqrDesc>(std::max(nb, 1));
    CK(cudaMemcpy(dc, cd.data(), sizeof(CpqrDesc) * nb, cudaMemcpyHostToDevice));
    std::vector<int> all(nb);
    for (int b = 0; b < nb; ++b) all[b] = b;
    int* didx = mem.alloc_n<int>(std::max(nb, 1));
    CK(cudaMemcpy(didx, all.data(), sizeof(int) * nb, cudaMemcpyHostToDevice));
    const size_t sm = cpqr_smem_bytes(m, n);
    const char* force = std::getenv("SPQR_CPQR_PATH");  // narrow|tall|smem|big|cluster (comparisons, tests)
    const std::string fp = force ? force : "";
    const bool clus = fp == "cluster" && n >= 16 && cpqr_clus_smem_bytes(m, n) <= 200 * 1024;
    const int ncls = (fp.empty() || fp == "narrow") ? cpqr_narrow_class(m, n) : -1;
    const int tcls = (fp.empty() || fp == "tall") ? cpqr_tall_class(m, n) : -1;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ms) {
        CK(cudaEventCreate(&e0));
        CK(cudaEventCreate(&e1));
        CK(cudaDeviceSynchronize());
        CK(cudaEventRecord(e0, 0));
    }
    if (clus)
        launch_cpqr_clus(dc, didx, nb, cpqr_clus_smem_bytes(m, n), 0);
    else if (ncls >= 0)
        launch_cpqr_narrow(ncls, dc, didx, nb, cpqr_narrow_smem(m, n), 0);
    else if (tcls >= 0)
        launch_cpqr_tall(tcls, dc, didx, nb, 0);
    else if (big)
        for (int b = 0; b < nb; ++b) launch_cpqr_big(cd[b], 0);
    else if (sm <= kSmemBudget)
        launch_cpqr_split(dc, didx, nb, sm, nullptr, 0, m, 0);
    else
        launch_cpqr_split(dc, nullptr, 0, 0, didx, nb, m, 0);
    if (ms) {
        CK(cudaEventRecord(e1, 0));
        CK(cudaEventSynchronize(e1));
        CK(cudaEventElapsedTime(ms, e0, e1));
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    CK(cudaDeviceSynchronize());
    CK(cudaGetLastError());
}
}  // namespace

int spqr_cpqr_batched(int nb, int m, int n, const double* a, double eps, int* rank, double* r11, int* perm, double* R,
                      double* V, double* tau, double* sign) {
    int cl = -1;
    return guarded(nullptr, 0, &cl, [&] {
        const int kmax = std::min(m, n);
        const size_t na = static_cast<size_t>(nb) * m * n;
        DeviceArena mem;
        double* da = mem.alloc_n<double>(std::max<size_t>(na, 1));
        double* dV = mem.alloc_n<double>(std::max<size_t>(static_cast<size_t>(nb) * m * kmax, 1));
        double* dt = mem.alloc_n<double>(std::max(nb * kmax, 1));
        double* ds = mem.alloc_n<double>(std::max(nb * kmax, 1));
        int* dp = mem.alloc_n<int>(std::max(nb * kmax, 1));
        int* dr = mem.alloc_n<int>(std::max(nb, 1));
        double* d11 = mem.alloc_n<double>(std::max(nb, 1));
        CK(cudaMemcpy(da, a, sizeof(double) * na, cudaMemcpyHostToDevice));
        cpqr_dev_run(mem, nb, m, n, da, eps, dr, d11, dp, dV, dt, ds, nullptr);
        std::vector<double> A(na);
        CK(cudaMemcpy(A.data(), da, sizeof(double) * na, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(rank, dr, sizeof(int) * nb, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(r11, d11, sizeof(double) * nb, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(perm, dp, sizeof(int) * nb * kmax, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(V, dV, sizeof(double) * static_cast<size_t>(nb) * m * kmax, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(tau, dt, sizeof(double) * nb * kmax, cudaMemcpyDeviceToHost));
        CK(cudaMemcpy(sign, ds, sizeof(double) * nb * kmax, cudaMemcpyDeviceToHost));
        for (int b = 0; b < nb; ++b) {
            double* Rb = R + static_cast<long long>(b) * kmax * n;
            const double* Ab = A.data() + static_cast<long long>(b) * m * n;
            for (int j = 0; j < n; ++j)
                for (int i = 0; i < kmax; ++i) Rb[i + static_cast<long long>(j) * kmax] = i < rank[b] ? Ab[i + static_cast<long long>(j) * m] : 0.0;
        }
    });
}

int spqr_cpqr_batched_dev(int nb, int m, int n, double* d_a, double eps, int* d_rank, float* ms) {
    int cl = -1;
    return guarded(nullptr, 0, &cl, [&] {
        const int kmax = std::min(m, n);
        DeviceArena mem;
        double* dV = mem.alloc_n<double>(std::max<size_t>(static_cast<size_t>(nb) * m * kmax, 1));
        double* dt = mem.alloc_n<double>(std::max(nb * kmax, 1));
        double* ds = mem.alloc_n<double>(std::max(nb * kmax, 1));
        int* dp = mem.alloc_n<int>(std::max(nb * kmax, 1));
        double* d11 = mem.alloc_n<double>(std::max(nb, 1));
        float t = 0.f;
        cpqr_dev_run(mem, nb, m, n, d_a, eps, d_rank, d11, dp, dV, dt, ds, &t);
        if (ms) *ms = t;
    });
}

int spqr_trsm_right_batched(int nb, int nrows, int n, double* b, const double* r) {
    int cl = -1;
    return guarded(nullptr, 0, &cl, [&] {
        DeviceArena mem;
        const size_t nbb = static_cast<size_t>(nb) * nrows * n, nr = static_cast<size_t>(nb) * n * n;
        double* db = mem.alloc_n<double>(std::max<size_t>(nbb, 1));
        double* dr = mem.alloc_n<double>(std::max<size_t>(nr, 1));
        CK(cudaMemcpy(db, b, sizeof(double) * nbb, cudaMemcpyHostToDevice));
        CK(cudaMemcpy(dr, r, sizeof(double) * nr, cudaMemcpyHostToDevice));
        std::vector<TrsmDesc> td(nb);
        for (int q = 0; q < nb; ++q)
            td[q] = TrsmDesc{db + static_cast<long long>(q) * nrows * n, nrows, nrows, n, dr + static_cast<long long>(q) * n * n, n,
                             static_cast<long long>(q) * nrows};
        TrsmDesc* dt = mem.alloc_n<TrsmDesc>(std::max(nb, 1));
        CK(cudaMemcpy(dt, td.data(), sizeof(TrsmDesc) * nb, cudaMemcpyHostToDevice));
        launch_trsm(dt, nb, static_cast<long long>(nb) * nrows, 0);
        CK(cudaDeviceSynchronize());
        CK(cudaGetLastError());
        CK(cudaMemcpy(b, db, sizeof(double) * nbb, cudaMemcpyDeviceToHost));
    });
}

}  // extern "C"
