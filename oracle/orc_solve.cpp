// ORACLE — TEST INFRASTRUCTURE ONLY (see orc_core.h header).
// Restates proj/src/transforms.cpp:1-127 (W / W^-1 / W^T / W^-T sweeps, Q
// sweeps, nnz(W)), proj/src/solve.cpp (preconditioned CGLS, CSNE) and
// proj/src/pipeline.cpp (scale -> dissect -> order -> match -> assign ->
// factorize, solve, unscale).
#include <numeric>

#include "orc_core.h"

namespace orc {

namespace {
Vec gather(const Vec& z, const std::vector<Index>& idx) {
    Vec o(idx.size());
    for (size_t i = 0; i < idx.size(); ++i) o[i] = z[idx[i]];
    return o;
}
void scatter(Vec& z, const std::vector<Index>& idx, const Vec& v) {
    for (size_t i = 0; i < idx.size(); ++i) z[idx[i]] = v[i];
}
View colview(Vec& v) { return View{v.data(), static_cast<Index>(v.size()), 1, static_cast<Index>(v.size())}; }
}  // namespace

// transforms.cpp:25-38
long long Factorization::nnz_w() const {
    long long s = 0;
    for (const auto& f : W) {
        if (const auto* t = std::get_if<TriangularScale>(&f)) {
            const long long c = static_cast<long long>(t->cols.size());
            s += c * (c + 1) / 2 + c * static_cast<long long>(t->coupled.size());
        } else {
            const auto& r = std::get<ColumnRotation>(f);
            const long long m = r.Q.rows(), k = r.Q.count();
            s += k * m - k * (k - 1) / 2 + k;
        }
    }
    return s;
}

// transforms.cpp:40-54
void Factorization::w_apply(Vec& z) const {
    for (const auto& f : W) {
        if (const auto* t = std::get_if<TriangularScale>(&f)) {
            const Vec zs = gather(z, t->cols);
            const Index c = static_cast<Index>(zs.size());
            Vec o(c, 0.0);
            for (Index i = 0; i < c; ++i) {
                double s = 0.0;
                for (Index j = i; j < c; ++j) s += t->R(i, j) * zs[j];
                o[i] = s;
            }
            if (!t->coupled.empty()) {
                const Vec zn = gather(z, t->coupled);
                for (Index i = 0; i < c; ++i) {
                    double s = 0.0;
                    for (size_t j = 0; j < zn.size(); ++j) s += t->C(i, static_cast<Index>(j)) * zn[j];
                    o[i] += s;
                }
            }
            scatter(z, t->cols, o);
        } else {
            const auto& r = std::get<ColumnRotation>(f);
            Vec zc = gather(z, r.cols);
            apply_left_t(r.Q, colview(zc));
            scatter(z, r.cols, zc);
        }
    }
}

// transforms.cpp:56-71
void Factorization::w_solve(Vec& z) const {
    for (auto it = W.rbegin(); it != W.rend(); ++it) {
        if (const auto* t = std::get_if<TriangularScale>(&*it)) {
            Vec zs = gather(z, t->cols);
            const Index c = static_cast<Index>(zs.size());
            if (!t->coupled.empty()) {
                const Vec zn = gather(z, t->coupled);
                for (Index i = 0; i < c; ++i) {
                    double s = 0.0;
                    for (size_t j = 0; j < zn.size(); ++j) s += t->C(i, static_cast<Index>(j)) * zn[j];
                    zs[i] -= s;
                }
            }
            tri_solve_upper(t->R, colview(zs), Side::Left, false);
            scatter(z, t->cols, zs);
        } else {
            const auto& r = std::get<ColumnRotation>(*it);
            Vec zc = gather(z, r.cols);
            apply_left(r.Q, colview(zc));
            scatter(z, r.cols, zc);
        }
    }
}

// transforms.cpp:73-91
void Factorization::wt_apply(Vec& z) const {
    for (auto it = W.rbegin(); it != W.rend(); ++it) {
        if (const auto* t = std::get_if<TriangularScale>(&*it)) {
            const Vec zs = gather(z, t->cols);
            const Index c = static_cast<Index>(zs.size());
            if (!t->coupled.empty()) {
                Vec zn = gather(z, t->coupled);
                for (size_t j = 0; j < zn.size(); ++j) {
                    double s = 0.0;
                    for (Index i = 0; i < c; ++i) s += t->C(i, static_cast<Index>(j)) * zs[i];
                    zn[j] += s;
                }
                scatter(z, t->coupled, zn);
            }
            Vec o(c, 0.0);
            for (Index i = 0; i < c; ++i) {
                double s = 0.0;
                for (Index j = 0; j <= i; ++j) s += t->R(j, i) * zs[j];
                o[i] = s;
            }
            scatter(z, t->cols, o);
        } else {
            const auto& r = std::get<ColumnRotation>(*it);
            Vec zc = gather(z, r.cols);
            apply_left(r.Q, colview(zc));
            scatter(z, r.cols, zc);
        }
    }
}

// transforms.cpp:93-111
void Factorization::wt_solve(Vec& z) const {
    for (const auto& f : W) {
        if (const auto* t = std::get_if<TriangularScale>(&f)) {
            Vec zs = gather(z, t->cols);
            tri_solve_upper(t->R, colview(zs), Side::Left, true);
            scatter(z, t->cols, zs);
            if (!t->coupled.empty()) {
                Vec zn = gather(z, t->coupled);
                const Index c = static_cast<Index>(zs.size());
                for (size_t j = 0; j < zn.size(); ++j) {
                    double s = 0.0;
                    for (Index i = 0; i < c; ++i) s += t->C(i, static_cast<Index>(j)) * zs[i];
                    zn[j] -= s;
                }
                scatter(z, t->coupled, zn);
            }
        } else {
            const auto& r = std::get<ColumnRotation>(f);
            Vec zc = gather(z, r.cols);
            apply_left_t(r.Q, colview(zc));
            scatter(z, r.cols, zc);
        }
    }
}

// transforms.cpp:113-127
void Factorization::q_apply_t(Vec& y) const {
    for (const auto& f : Q) {
        Vec ys = gather(y, f.rows);
        apply_left_t(f.H, colview(ys));
        scatter(y, f.rows, ys);
    }
}
void Factorization::q_apply(Vec& y) const {
    for (auto it = Q.rbegin(); it != Q.rend(); ++it) {
        Vec ys = gather(y, it->rows);
        apply_left(it->H, colview(ys));
        scatter(y, it->rows, ys);
    }
}

namespace {
double wnorm(const Vec& t, const Vec* w) {
    double s = 0.0;
    if (!w)
        for (double v : t) s += v * v;
    else
        for (size_t i = 0; i < t.size(); ++i) s += (t[i] * (*w)[i]) * (t[i] * (*w)[i]);
    return std::sqrt(s);
}
double sqn(const Vec& v) {
    double s = 0.0;
    for (double x : v) s += x * x;
    return s;
}
}  // namespace

// solve.cpp:24-76
SolveReport cgls(const Csc& A, const Factorization* W, const Vec& b, Vec& u, const CglsOptions& opt, const Vec* weights) {
    const double t0 = now_s();
    SolveReport rep;
    if (W) rep.dropped_rows = static_cast<Index>(W->dropped_rows.size());
    const Index n = A.n;
    u.assign(n, 0.0);
    Vec r = b;
    Vec t = spmv_t(A, r);
    const double nres0 = wnorm(t, weights);
    if (nres0 == 0.0) {
        rep.converged = true;
        rep.residual_history = {0.0};
        rep.t_solve = now_s() - t0;
        return rep;
    }
    rep.residual_history.push_back(1.0);
    Vec s = t;
    if (W) W->wt_solve(s);
    Vec p = s, y(n, 0.0);
    double gamma = sqn(s);
    for (int it = 1; it <= opt.maxit; ++it) {
        Vec v = p;
        if (W) W->w_solve(v);
        const Vec q = spmv(A, v);
        const double qq = sqn(q);
        if (qq == 0.0 || gamma == 0.0) break;
        const double alpha = gamma / qq;
        for (Index i = 0; i < n; ++i) y[i] += alpha * p[i];
        for (size_t i = 0; i < r.size(); ++i) r[i] -= alpha * q[i];
        t = spmv_t(A, r);
        const double rel = wnorm(t, weights) / nres0;
        rep.residual_history.push_back(rel);
        rep.iterations = it;
        if (rel <= opt.tol || !std::isfinite(rel)) {
            rep.converged = rel <= opt.tol;
            break;
        }
        s = t;
        if (W) W->wt_solve(s);
        const double gn = sqn(s);
        const double beta = gn / gamma;
        for (Index i = 0; i < n; ++i) p[i] = s[i] + beta * p[i];
        gamma = gn;
    }
    u = y;
    if (W) W->w_solve(u);
    rep.t_solve = now_s() - t0;
    return rep;
}

// solve.cpp:78-108
Vec csne_solve(const Csc& A, const Factorization& W, const Vec& b, int refine, SolveReport* rep, const Vec* weights, double tol) {
    const double t0 = now_s();
    const double nres0 = wnorm(spmv_t(A, b), weights);
    Vec u = spmv_t(A, b);
    W.wt_solve(u);
    W.w_solve(u);
    auto residual_vec = [&]() {
        const Vec Au = spmv(A, u);
        Vec rr(b.size());
        for (size_t i = 0; i < b.size(); ++i) rr[i] = b[i] - Au[i];
        return rr;
    };
    auto record = [&]() {
        if (!rep) return;
        if (nres0 == 0.0) {
            rep->residual_history.push_back(0.0);
            return;
        }
        rep->residual_history.push_back(wnorm(spmv_t(A, residual_vec()), weights) / nres0);
    };
    record();
    for (int step = 0; step < refine; ++step) {
        Vec du = spmv_t(A, residual_vec());
        W.wt_solve(du);
        W.w_solve(du);
        for (size_t i = 0; i < u.size(); ++i) u[i] += du[i];
        record();
    }
    if (rep) {
        rep->iterations = refine;
        rep->converged = rep->residual_history.back() <= tol;
        rep->t_solve = now_s() - t0;
    }
    return u;
}

// pipeline.cpp:19-62
Pipeline::Pipeline(const Csc& A, const PipelineOptions& o, const Coords* coords, const std::vector<int>* parts, FactorizeObserver* obs)
    : opt(o), Aw(A) {
    if (Aw.m < Aw.n) throw std::invalid_argument("matrix must have at least as many rows as columns");
    if (opt.solver == SolverKind::Direct) opt.eps = 0.0;
    d = scale_columns(Aw);
    const Index n = Aw.n;
    if (opt.solver == SolverKind::Diag) {
        perm.resize(n);
        std::iota(perm.begin(), perm.end(), 0);
        weights = d;
        return;
    }
    double t0 = now_s();
    const PatternGraph g = ata_graph(Aw);
    const int L = opt.levels > 0 ? opt.levels : default_num_levels(n);
    if (parts) {
        tree = import_partition(g, L, *parts);
    } else {
        if (coords && coords->n != n) throw std::invalid_argument("coordinate row count does not match column count");
        tree = nested_dissection(g, L, coords);
    }
    h = build_interfaces(tree, g);
    perm = order_columns(h);
    Aw = permute_columns(Aw, perm);
    const RowMatching m = match_rows(Aw);
    owner = assign_rows(Aw, h, m);
    t_partition = now_s() - t0;
    weights.resize(n);
    for (Index i = 0; i < n; ++i) weights[i] = d[perm[i]];
    t0 = now_s();
    FactorizeOptions fo;
    fo.eps = opt.eps;
    fo.skip_levels = opt.skip_levels;
    fo.store_q = opt.store_q;
    F = spaqr_factorize(Aw, h, owner, fo, obs);
    has_f = true;
    t_factorize = now_s() - t0;
}

Vec Pipeline::unscale(const Vec& u) const {  // pipeline.cpp:65-68
    Vec x(Aw.n);
    for (Index i = 0; i < Aw.n; ++i) x[perm[i]] = u[i] / d[perm[i]];
    return x;
}

Vec Pipeline::solve(const Vec& b, SolveReport* rep, double tol, int maxit) const {  // :70-80
    if (static_cast<Index>(b.size()) != Aw.m) throw std::invalid_argument("right-hand side length mismatch");
    CglsOptions co;
    co.tol = tol > 0 ? tol : opt.tol;
    co.maxit = maxit > 0 ? maxit : opt.maxit;
    Vec u;
    SolveReport r = cgls(Aw, has_f ? &F : nullptr, b, u, co, &weights);
    if (has_f) r.dropped_rows = static_cast<Index>(F.dropped_rows.size());
    if (rep) *rep = std::move(r);
    return unscale(u);
}

Vec Pipeline::solve_direct(const Vec& b, SolveReport* rep) const {  // :82-92
    if (!has_f) throw std::logic_error("direct solve requires a factorization");
    if (static_cast<Index>(b.size()) != Aw.m) throw std::invalid_argument("right-hand side length mismatch");
    SolveReport r;
    Vec u = csne_solve(Aw, F, b, opt.refine, rep ? &r : nullptr, &weights, opt.tol);
    if (rep) {
        r.dropped_rows = static_cast<Index>(F.dropped_rows.size());
        *rep = std::move(r);
    }
    return unscale(u);
}

}  // namespace orc
