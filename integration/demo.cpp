// Integration check: the reference's own code (proj/src, compiled unmodified against the
// in-repo Eigen API shim) and the B200 library bound through integration/pipeline_b200.hpp,
// side by side in one process on the same problem.  Prints one "CHECK <name> ok|FAIL ..."
// line per comparison and exits non-zero on any failure.  Without a GPU it only checks that
// the B200 path refuses to run (no CPU fallback).
#include <cmath>
#include <cstdio>
#include <random>
#include <set>

#include "pipeline_b200.hpp"
#include "spaqr/transforms.h"

using namespace spaqr;

namespace {

int failures = 0;
void check(const char* name, bool ok, const std::string& detail = "") {
    std::printf("CHECK %s %s %s\n", name, ok ? "ok" : "FAIL", detail.c_str());
    if (!ok) ++failures;
}

// 2D tall problem (BASELINE config 1 construction, own seeded generator): N stencil rows with
// centre 4+U(0,1) and neighbours -1+0.1 N(0,1), then N rows of 3 N(0,1) entries (a cell and 2
// distinct in-grid neighbours).
struct Problem {
    SparseMatrix A;
    MatrixXd xy;
    VectorXd b;
};
Problem tall_grid(int n, unsigned seed) {
    std::mt19937_64 rng(seed);
    std::uniform_real_distribution<double> U(0.0, 1.0);
    std::normal_distribution<double> G(0.0, 1.0);
    const int N = n * n;
    std::vector<Eigen::Triplet<double>> t;
    auto nbrs = [&](int c) {
        std::vector<int> v;
        const int i = c / n, j = c % n;
        if (i > 0) v.push_back(c - n);
        if (i + 1 < n) v.push_back(c + n);
        if (j > 0) v.push_back(c - 1);
        if (j + 1 < n) v.push_back(c + 1);
        return v;
    };
    for (int c = 0; c < N; ++c) {
        t.emplace_back(c, c, 4.0 + U(rng));
        for (int q : nbrs(c)) t.emplace_back(c, q, -1.0 + 0.1 * G(rng));
    }
    for (int r = 0; r < N; ++r) {
        const int c = static_cast<int>(U(rng) * N) % N;
        std::vector<int> v = nbrs(c);
        std::shuffle(v.begin(), v.end(), rng);
        t.emplace_back(N + r, c, G(rng));
        for (int k = 0; k < 2 && k < static_cast<int>(v.size()); ++k) t.emplace_back(N + r, v[k], G(rng));
    }
    Problem p;
    p.A = SparseMatrix::from_triplets(2 * N, N, t);
    p.xy = MatrixXd(N, 2);
    for (int c = 0; c < N; ++c) {
        p.xy(c, 0) = c / n;
        p.xy(c, 1) = c % n;
    }
    p.b = VectorXd(2 * N);
    for (int r = 0; r < 2 * N; ++r) p.b(r) = G(rng);
    return p;
}

double rel_normal_residual(const SparseMatrix& A, const VectorXd& b, const VectorXd& x) {
    const VectorXd r = b - spmv(A, x);
    return spmv_t(A, r).norm() / spmv_t(A, b).norm();
}

double max_rel(const VectorXd& a, const VectorXd& b) {
    double m = 0.0, s = 0.0;
    for (Index i = 0; i < a.size(); ++i) {
        m = std::max(m, std::abs(a(i) - b(i)));
        s = std::max(s, std::abs(b(i)));
    }
    return m / std::max(s, 1.0);
}

}  // namespace

int main(int argc, char** argv) {
    const std::string tmp = argc > 1 ? argv[1] : "/tmp";
    Problem p = tall_grid(48, 7);
    PipelineOptions opt;
    opt.eps = 1e-2;
    opt.levels = 7;
    if (spqr_device_count() <= 0) {  // CPU-only host: the B200 path must refuse, not fall back
        bool threw = false;
        try {
            PipelineB200 g(p.A, opt, &p.xy);
        } catch (const std::runtime_error&) {
            threw = true;
        }
        check("no_gpu_refuses", threw);
        return failures ? 1 : 0;
    }
    // 1. Pipeline: reference (CPU) vs B200
    Pipeline ref(p.A, opt, &p.xy);
    PipelineB200 gpu(p.A, opt, &p.xy);
    SolveReport rr, rg;
    const VectorXd xr = ref.solve(p.b, &rr);
    const VectorXd xg = gpu.solve(p.b, &rg);
    check("pipeline_iterations", std::abs(rr.iterations - rg.iterations) <= 1,
          std::to_string(rr.iterations) + " vs " + std::to_string(rg.iterations));
    const double er = rel_normal_residual(p.A, p.b, xr), eg = rel_normal_residual(p.A, p.b, xg);
    check("pipeline_residual", std::abs(er - eg) <= 1e-10, std::to_string(er) + " vs " + std::to_string(eg));
    // 2. spaqr_factorize on the reference's hierarchy and row ownership
    const SparseMatrix& Aw = ref.scaled();
    const std::vector<int> owner = assign_rows(Aw, ref.hierarchy(), match_rows(Aw));
    FactorizeOptions fo;
    fo.eps = opt.eps;
    fo.skip_levels = opt.skip_levels;
    FactorizationB200 W = spaqr_factorize_b200(Aw, ref.hierarchy(), owner, fo);
    const Factorization& F = *ref.factorization();
    check("factorize_nW", W.info(2) == static_cast<long long>(F.W.size()),
          std::to_string(W.info(2)) + " vs " + std::to_string(F.W.size()));
    check("factorize_nnz_w", W.info(3) == F.nnz_w());
    VectorXd z(Aw.cols());
    std::mt19937_64 rng(3);
    std::uniform_real_distribution<double> U(-1.0, 1.0);
    for (Index i = 0; i < z.size(); ++i) z(i) = U(rng);
    VectorXd zr = z, zg = z;
    F.w_solve(zr);
    W.w_solve(zg);
    check("w_solve", max_rel(zg, zr) <= 1e-10, std::to_string(max_rel(zg, zr)));
    zr = z;
    zg = z;
    F.wt_solve(zr);
    W.wt_solve(zg);
    check("wt_solve", max_rel(zg, zr) <= 1e-10, std::to_string(max_rel(zg, zr)));
    // 3. cgls(A, W, b, u, opt, weights) with the GPU factor vs the reference's cgls with its own
    CglsOptions co;
    VectorXd ur, ug;
    const SolveReport cr = cgls(Aw, &F, p.b, ur, co);
    const SolveReport cg = cgls_b200(Aw, &W, p.b, ug, co);
    check("cgls_iterations", std::abs(cr.iterations - cg.iterations) <= 1,
          std::to_string(cr.iterations) + " vs " + std::to_string(cg.iterations));
    check("cgls_residual", std::abs(cr.residual_history.back() - cg.residual_history.back()) <= 1e-10);
    // 4. factor files: GPU-written file read by the reference's load_factorization, and the
    //    reference-written file loaded onto the GPU
    W.save(tmp + "/w_gpu.spqr");
    save_factorization(F, tmp + "/w_ref.spqr");
    const Factorization Fg = load_factorization(tmp + "/w_gpu.spqr");
    FactorizationB200 Wr = FactorizationB200::load(tmp + "/w_ref.spqr");
    zr = z;
    zg = z;
    Fg.w_solve(zr);
    Wr.w_solve(zg);
    check("factor_files", max_rel(zg, zr) <= 1e-10 && Fg.W.size() == F.W.size(), std::to_string(max_rel(zg, zr)));
    // 4b. store_q (factorize.h:16): the reference's Q against the GPU's, both ways through files
    {
        FactorizeOptions fq = fo;
        fq.store_q = true;
        const Factorization Fq = spaqr_factorize(Aw, ref.hierarchy(), owner, fq);
        FactorizationB200 Wq = spaqr_factorize_b200(Aw, ref.hierarchy(), owner, fq);
        VectorXd y(Aw.rows());
        for (Index i = 0; i < y.size(); ++i) y(i) = U(rng);
        VectorXd yr = y, yg = y;
        Fq.q_apply_t(yr);
        Wq.q_apply_t(yg);
        check("q_apply_t", Wq.has_q() && max_rel(yg, yr) <= 1e-10, std::to_string(max_rel(yg, yr)));
        yr = y;
        yg = y;
        Fq.q_apply(yr);
        Wq.q_apply(yg);
        check("q_apply", max_rel(yg, yr) <= 1e-10, std::to_string(max_rel(yg, yr)));
        Wq.save(tmp + "/q_gpu.spqr");
        const Factorization Fqg = load_factorization(tmp + "/q_gpu.spqr");
        yr = y;
        yg = y;
        Fqg.q_apply_t(yr);
        Wq.q_apply_t(yg);
        check("q_factor_file", Fqg.has_q && Fqg.Q.size() == Fq.Q.size() && max_rel(yg, yr) <= 1e-10,
              std::to_string(Fqg.Q.size()) + " vs " + std::to_string(Fq.Q.size()));
    }
    // 5. error mapping: a front with fewer coupled rows than columns
    {
        std::vector<Eigen::Triplet<double>> t{{0, 0, 1.0}, {0, 1, 2.0}};
        for (int j = 2; j < 6; ++j) {
            t.emplace_back(2 * j - 3, j, 3.0);
            t.emplace_back(2 * j - 2, j, 0.5);
        }
        const SparseMatrix D = SparseMatrix::from_triplets(9, 6, t);
        const std::vector<int> parts{0, 0, 1, 1, 1, 1};
        PipelineOptions o0;
        o0.eps = 0.0;
        o0.levels = 1;
        int cref = -2, cgpu = -3;
        std::string why_ref, why_gpu;
        try {
            Pipeline bad(D, o0, nullptr, &parts);
        } catch (const SingularFrontError& e) {
            cref = e.cluster;
            why_ref = e.reason;
        }
        try {
            PipelineB200 bad(D, o0, nullptr, &parts);
        } catch (const SingularFrontError& e) {
            cgpu = e.cluster;
            why_gpu = e.reason;
        }
        check("singular_front_error", cref == cgpu && why_ref == why_gpu, why_ref + " | " + why_gpu);
    }
    std::printf("%s\n", failures ? "FAILED" : "ALL OK");
    return failures ? 1 : 0;
}
