// The C++ shim a maintainer would add to the reference (proj/src/pipeline_b200.hpp) to run
// its Pipeline / spaqr_factorize / cgls on the B200 library through the C ABI
// (include/spaqr_b200.h).  Same signatures and error types as the reference:
//   Pipeline            proj/include/spaqr/pipeline.h:39-52
//   spaqr_factorize     proj/include/spaqr/factorize.h:51-53
//   cgls                proj/include/spaqr/solve.h:30-31
//   SingularFrontError  proj/include/spaqr/types.h:24-31
// Compiled and run against the reference's own headers by integration/Makefile
// (tests/test_integration.py).
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "spaqr/factorize.h"
#include "spaqr/pipeline.h"
#include "spaqr/solve.h"
#include "spaqr_b200.h"

namespace spaqr {

inline void b200_check(int rc, const char* err, int cluster) {
    if (rc == SPQR_OK) return;
    const std::string what(err);
    if (rc == SPQR_E_SINGULAR) {
        const size_t at = what.find("| reason: ");
        throw SingularFrontError(cluster, at == std::string::npos ? what : what.substr(at + 10));
    }
    if (rc == SPQR_E_SHAPE) throw std::invalid_argument(what);
    throw std::runtime_error(what);
}

class PipelineB200 {
public:
    PipelineB200(const SparseMatrix& A, const PipelineOptions& opt, const MatrixXd* coords = nullptr,
                 const std::vector<int>* parts = nullptr, int device = 0) {
        std::vector<double> xy;  // coords row-major (N x dim)
        if (coords) {
            xy.resize(coords->rows() * coords->cols());
            for (Index v = 0; v < coords->rows(); ++v)
                for (Index d = 0; d < coords->cols(); ++d) xy[v * coords->cols() + d] = (*coords)(v, d);
        }
        char err[512] = {0};
        int cluster = -1;
        const int rc = spqr_pipeline_create_ex(A.rows(), A.cols(), A.outer(), A.inner(), A.values(),
                                               coords ? xy.data() : nullptr, coords ? int(coords->cols()) : 0,
                                               parts ? parts->data() : nullptr, opt.levels, opt.eps, opt.skip_levels,
                                               int(opt.solver), int(opt.store_q), /*ranks=*/1, device,
                                               /*obs=*/nullptr, nullptr, &h_, err, sizeof err, &cluster);
        b200_check(rc, err, cluster);
    }
    PipelineB200(const PipelineB200&) = delete;
    PipelineB200& operator=(const PipelineB200&) = delete;
    ~PipelineB200() { spqr_pipeline_destroy(h_); }

    VectorXd solve(const VectorXd& b, SolveReport* rep = nullptr, double tol = -1, int maxit = -1) const {
        return run(0, b, rep, tol, maxit);
    }
    VectorXd solve_direct(const VectorXd& b, SolveReport* rep = nullptr) const { return run(1, b, rep, -1, -1); }
    Index rows() const { return Index(info(0)); }
    Index cols() const { return Index(info(1)); }

private:
    spqr_pipeline* h_ = nullptr;
    long long info(int i) const {
        long long v[16];
        spqr_pipeline_info(h_, v);
        return v[i];
    }
    VectorXd run(int direct, const VectorXd& b, SolveReport* rep, double tol, int maxit) const {
        if (b.size() != rows()) throw std::invalid_argument("right-hand side length mismatch");
        VectorXd x(cols());
        std::vector<double> hist((maxit > 0 ? maxit : 500) + 4);
        int it = 0, conv = 0, nh = 0;
        double ts = 0;
        char err[512] = {0};
        b200_check(spqr_pipeline_solve(h_, direct, b.data(), x.data(), tol, maxit, &it, &conv, hist.data(), &nh,
                                       &ts, err, sizeof err),
                   err, -1);
        if (rep) {
            rep->iterations = it;
            rep->converged = conv != 0;
            rep->residual_history.assign(hist.begin(), hist.begin() + nh);
            rep->t_solve = ts;
        }
        return x;
    }
};

// spaqr_factorize on the GPU: W stays on the device; w_solve / wt_solve through sweeps.
class FactorizationB200 {
public:
    explicit FactorizationB200(spqr_factorization* h) : h_(h) {}
    FactorizationB200(const FactorizationB200&) = delete;
    FactorizationB200(FactorizationB200&& o) noexcept : h_(o.h_) { o.h_ = nullptr; }
    ~FactorizationB200() {
        if (h_) spqr_factorization_destroy(h_);
    }
    spqr_factorization* handle() const { return h_; }
    long long info(int i) const {
        long long v[8];
        spqr_factorization_info(h_, v);
        return v[i];
    }
    void w_solve(VectorXd& z) const { apply(SPQR_W_SOLVE, z); }
    void wt_solve(VectorXd& z) const { apply(SPQR_WT_SOLVE, z); }
    void w_apply(VectorXd& z) const { apply(SPQR_W_APPLY, z); }
    void wt_apply(VectorXd& z) const { apply(SPQR_WT_APPLY, z); }
    // transforms.h:70-71 (factorizations made with FactorizeOptions::store_q); y has length M
    void q_apply_t(VectorXd& y) const { apply(SPQR_Q_APPLY_T, y); }
    void q_apply(VectorXd& y) const { apply(SPQR_Q_APPLY, y); }
    bool has_q() const { return spqr_factorization_nq(h_) >= 0; }
    void save(const std::string& path) const {
        char err[512] = {0};
        b200_check(spqr_factorization_save(h_, path.c_str(), err, sizeof err), err, -1);
    }
    static FactorizationB200 load(const std::string& path, int device = 0) {
        spqr_factorization* h = nullptr;
        char err[512] = {0};
        b200_check(spqr_factorization_load(path.c_str(), device, &h, err, sizeof err), err, -1);
        return FactorizationB200(h);
    }

private:
    spqr_factorization* h_ = nullptr;
    void apply(int mode, VectorXd& z) const {
        if (spqr_factorization_apply(h_, mode, z.data()) != SPQR_OK) throw std::runtime_error("W sweep failed");
    }
};

inline FactorizationB200 spaqr_factorize_b200(const SparseMatrix& A, const ClusterHierarchy& h,
                                              const std::vector<int>& row_owner, const FactorizeOptions& opt,
                                              int device = 0) {
    if (static_cast<Index>(row_owner.size()) != A.rows()) throw std::invalid_argument("row_owner size mismatch");
    std::vector<int> info, cptr{0}, ccols, tpar;
    for (const auto& c : h.clusters) {
        info.insert(info.end(), {c.tree_node, c.level, c.parent, c.stage, int(c.interior)});
        ccols.insert(ccols.end(), c.cols.begin(), c.cols.end());
        cptr.push_back(int(ccols.size()));
    }
    for (const auto& n : h.tree->nodes) tpar.push_back(n.parent);
    spqr_factorization* f = nullptr;
    char err[512] = {0};
    int cluster = -1;
    const int rc = spqr_factorize_ex(A.rows(), A.cols(), A.outer(), A.inner(), A.values(), h.num_levels,
                                     int(h.clusters.size()), info.data(), cptr.data(), ccols.data(),
                                     h.finest_of_col.data(), int(tpar.size()), tpar.data(), h.tree->root,
                                     row_owner.data(), opt.eps, opt.skip_levels, int(opt.store_q), device,
                                     /*obs=*/nullptr, nullptr, &f, err, sizeof err, &cluster);
    b200_check(rc, err, cluster);
    return FactorizationB200(f);
}

inline SolveReport cgls_b200(const SparseMatrix& A, const FactorizationB200* W, const VectorXd& b, VectorXd& u,
                             const CglsOptions& opt, const VectorXd* weights = nullptr, int device = 0) {
    u = VectorXd::Zero(A.cols());
    std::vector<double> hist(opt.maxit + 4);
    int it = 0, conv = 0, nh = 0;
    double ts = 0;
    char err[512] = {0};
    b200_check(spqr_cgls(A.rows(), A.cols(), A.outer(), A.inner(), A.values(), W ? W->handle() : nullptr, b.data(),
                         u.data(), opt.tol, opt.maxit, weights ? weights->data() : nullptr, device, &it, &conv,
                         hist.data(), &nh, &ts, err, sizeof err),
               err, -1);
    SolveReport rep;
    rep.iterations = it;
    rep.converged = conv != 0;
    rep.residual_history.assign(hist.begin(), hist.begin() + nh);
    rep.t_solve = ts;
    return rep;
}

}  // namespace spaqr
