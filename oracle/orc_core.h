// ============================================================================
// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// A single-threaded, Eigen-free CPU restatement of the spaQR reference
// (/root/reference/proj, C++20 + Eigen3, which cannot be compiled in this image:
// Eigen, doctest and CLI11 are absent).  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load it, and only as
// the checker or the CPU baseline — never as the product path.
//
// Parity pinning: the reference ships no golden vectors for this path.  The
// restatement is pinned by (a) the reference's own known-answer tests
// (identity factorization exact, CGLS on I bitwise, default_num_levels table,
// 8x8 grid root separator, row-assignment rules) and (b) its property tests
// (QR reconstruction, CPQR truncation rule and SVD rank, W round trips, exact
// factorization = dense LS), all ported to tests/test_oracle_*.py.
// Bitwise agreement with Eigen's blocked HouseholderQR is NOT pinned (Eigen's
// vectorised reduction order cannot be reproduced); Householder reflectors use
// Eigen's published makeHouseholder convention (unit v0, beta = -sign(c0)||x||,
// tau = (beta - c0)/beta), unblocked.
//
// Third-party dependency on the path: Eigen3 (>= 3.3, unpinned:
// proj/CMakeLists.txt:15-20).  Restated algorithms: HouseholderQR
// (makeHouseholder + applyHouseholderOnTheLeft), triangular solves, GEMM/GEMV.
// ============================================================================
#pragma once

#include <cmath>
#include <cstdint>
#include <map>
#include <set>
#include <stdexcept>
#include <string>
#include <variant>
#include <vector>

namespace orc {

// move_extras roundoff rule (factorize.cpp:141-164): candidate squared row norms at
// or below kMoveNoise2 x (largest squared row norm of the eliminated cluster's blocks) count as 0.
constexpr double kMoveNoise2 = (1e3 * 2.220446049250313e-16) * (1e3 * 2.220446049250313e-16);


using Index = int;  // proj/include/spaqr/types.h:11

// Column-major dense FP64 matrix (stands in for Eigen::MatrixXd, types.h:12).
struct Mat {
    Index r = 0, c = 0;
    std::vector<double> a;
    Mat() = default;
    Mat(Index rows, Index cols) : r(rows), c(cols), a(static_cast<size_t>(rows) * cols, 0.0) {}
    static Mat zeros(Index rows, Index cols) { return Mat(rows, cols); }
    static Mat identity(Index n) {
        Mat m(n, n);
        for (Index i = 0; i < n; ++i) m(i, i) = 1.0;
        return m;
    }
    double& operator()(Index i, Index j) { return a[static_cast<size_t>(j) * r + i]; }
    double operator()(Index i, Index j) const { return a[static_cast<size_t>(j) * r + i]; }
    double* col(Index j) { return a.data() + static_cast<size_t>(j) * r; }
    const double* col(Index j) const { return a.data() + static_cast<size_t>(j) * r; }
    size_t size() const { return a.size(); }
    // Eigen conservativeResize(rows, NoChange): keeps the top-left block.
    void resize_rows(Index nr) {
        if (nr == r) return;
        std::vector<double> b(static_cast<size_t>(nr) * c, 0.0);
        const Index keep = std::min(nr, r);
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < keep; ++i) b[static_cast<size_t>(j) * nr + i] = (*this)(i, j);
        a.swap(b);
        r = nr;
    }
    double row_sqnorm(Index i, Index c0 = 0, Index nc = -1) const {
        if (nc < 0) nc = c - c0;
        double s = 0.0;
        for (Index j = c0; j < c0 + nc; ++j) s += (*this)(i, j) * (*this)(i, j);
        return s;
    }
    bool row_is_zero(Index i) const {
        for (Index j = 0; j < c; ++j)
            if ((*this)(i, j) != 0.0) return false;
        return true;
    }
    // max |a_ij| over rows [r0, r0+nr) x cols [c0, c0+nc)
    double max_abs(Index r0, Index nr, Index c0, Index nc) const {
        double m = 0.0;
        for (Index j = c0; j < c0 + nc; ++j)
            for (Index i = r0; i < r0 + nr; ++i) m = std::max(m, std::abs((*this)(i, j)));
        return m;
    }
    bool block_is_zero(Index r0, Index nr, Index c0, Index nc) const {
        for (Index j = c0; j < c0 + nc; ++j)
            for (Index i = r0; i < r0 + nr; ++i)
                if ((*this)(i, j) != 0.0) return false;
        return true;
    }
    Mat block(Index r0, Index c0, Index nr, Index nc) const {
        Mat b(nr, nc);
        for (Index j = 0; j < nc; ++j)
            for (Index i = 0; i < nr; ++i) b(i, j) = (*this)(r0 + i, c0 + j);
        return b;
    }
    void set_block(Index r0, Index c0, const Mat& b) {
        for (Index j = 0; j < b.c; ++j)
            for (Index i = 0; i < b.r; ++i) (*this)(r0 + i, c0 + j) = b(i, j);
    }
    Mat transpose() const {
        Mat t(c, r);
        for (Index j = 0; j < c; ++j)
            for (Index i = 0; i < r; ++i) t(j, i) = (*this)(i, j);
        return t;
    }
    double fro() const {
        double s = 0.0;
        for (double v : a) s += v * v;
        return std::sqrt(s);
    }
};

using Vec = std::vector<double>;

struct SingularFrontError : std::runtime_error {  // types.h:24-31
    SingularFrontError(int cl, const std::string& why)
        : std::runtime_error("singular front (cluster " + std::to_string(cl) + "): " + why),
          cluster(cl), reason(why) {}
    int cluster;
    std::string reason;
};

// ---------------------------------------------------------------- sparse ---
// Canonical CSC (sparse.h:15-38): rows strictly increasing per column,
// duplicates summed, exact zeros pruned.
struct Csc {
    Index m = 0, n = 0;
    std::vector<Index> p, i;
    std::vector<double> x;
    Index nnz() const { return static_cast<Index>(x.size()); }
};
struct Trip { Index r, c; double v; };
Csc csc_from_triplets(Index m, Index n, const std::vector<Trip>& t);  // sparse.cpp:13-20
Vec scale_columns(Csc& A);                                             // sparse.cpp:136-150
Vec spmv(const Csc& A, const Vec& x);                                  // sparse.cpp:164
Vec spmv_t(const Csc& A, const Vec& y);                                // sparse.cpp:166-168
struct PatternGraph { Index n = 0; std::vector<std::vector<Index>> adj; };
PatternGraph ata_graph(const Csc& A);                                  // sparse.cpp:170-195
Csc permute_columns(const Csc& A, const std::vector<Index>& perm);     // sparse.cpp:197-205

// ------------------------------------------------------------- partition ---
struct SeparatorTree {  // partition.h:14-27
    struct Node {
        int id = -1, level = 0, parent = -1;
        int child[2] = {-1, -1};
        std::vector<Index> vertices, separator;
        bool leaf() const { return child[0] < 0; }
    };
    int num_levels = 0, root = 0;
    std::vector<Node> nodes;
};
struct Coords { Index n = 0; int dim = 0; std::vector<double> x; double at(Index v, int d) const { return x[static_cast<size_t>(v) * dim + d]; } };
int default_num_levels(Index n);                                              // partition.cpp:15-19
SeparatorTree nested_dissection(const PatternGraph& g, int L, const Coords* c);  // :186-194
SeparatorTree import_partition(const PatternGraph& g, int L, const std::vector<int>& parts);  // :196-214

struct ClusterHierarchy {  // partition.h:54-75
    struct Cluster {
        int id = -1, tree_node = -1, level = 0, parent = -1, stage = 0;
        bool interior = false;
        std::vector<Index> cols;
    };
    int num_levels = 0;
    std::vector<Cluster> clusters;
    std::vector<int> finest_of_col;
    const SeparatorTree* tree = nullptr;
    int leaf_stage() const { return num_levels + 1; }
    bool related(int a, int b) const;  // partition.cpp:223-229
};
ClusterHierarchy build_interfaces(const SeparatorTree& t, const PatternGraph& g);  // :231-346
std::vector<Index> order_columns(ClusterHierarchy& h);                              // :348-399
struct RowMatching { std::vector<Index> row_of_col, col_of_row; Index size = 0; };
RowMatching match_rows(const Csc& A);                                               // :401-463
std::vector<int> assign_rows(const Csc& A, const ClusterHierarchy& h, const RowMatching& m);  // :465-514

// ---------------------------------------------------------- dense kernels ---
struct ReflectorSet {  // dense_kernels.h:12-21
    Mat V;
    Vec tau, sign;
    mutable Mat T;  // lazily built compact-WY factor
    Index rows() const { return V.r; }
    Index count() const { return V.c; }
};
void block_householder_qr(const Mat& B, ReflectorSet& H, Mat& R);  // dense_kernels.cpp:11-35
// X is an (m x nc) column-major view with leading dimension ld.
struct View { double* p; Index r, c, ld; double& operator()(Index i, Index j) { return p[static_cast<size_t>(j) * ld + i]; } };
inline View view(Mat& m) { return View{m.a.data(), m.r, m.c, m.r}; }
inline View view(Mat& m, Index c0, Index nc) { return View{m.a.data() + static_cast<size_t>(c0) * m.r, m.r, nc, m.r}; }
void apply_left_t(const ReflectorSet& H, View X);   // :96-99   X <- H^T X
void apply_left(const ReflectorSet& H, View X);     // :101-104 X <- H X
void apply_right(const ReflectorSet& H, Mat& X);    // :106-110 X <- X H
void apply_right_t(const ReflectorSet& H, Mat& X);  // :112-116 X <- X H^T
Mat reflectors_to_dense(const ReflectorSet& H);     // :118-122
struct TruncatedQR { ReflectorSet H; Mat R; std::vector<Index> perm; Index rank = 0; double r11 = 0.0; };
TruncatedQR truncated_cpqr(const Mat& B, double eps);  // :124-232
void check_diag_invertible(const Mat& R);              // :234-240
enum class Side { Left, Right };
void tri_solve_upper(const Mat& R, View B, Side side, bool transpose);  // :242-257

// ------------------------------------------------------------ transforms ---
struct TriangularScale { std::vector<Index> cols; Mat R; std::vector<Index> coupled; Mat C; };  // transforms.h:16-21
struct ColumnRotation { std::vector<Index> cols; ReflectorSet Q; };                              // :26-29
using WFactor = std::variant<TriangularScale, ColumnRotation>;
struct RowReflect { std::vector<Index> rows; ReflectorSet H; };
struct StageStats {  // transforms.h:40-47
    int stage = 0;
    double t_eliminate = 0, t_reassign = 0, t_scale = 0, t_sparsify = 0, t_merge = 0;
    std::vector<int> front_cols;
    std::vector<double> front_aspect;
    int top_rows = 0, top_cols = 0;
    long long nnz_w = 0;
};
struct Factorization {  // transforms.h:53-72
    Index M = 0, N = 0;
    double eps = 0.0;
    std::vector<WFactor> W;
    std::vector<RowReflect> Q;
    std::vector<Index> pivot_row, dropped_rows, trailing_rows;
    std::vector<StageStats> stages;
    bool has_q = false;
    long long nnz_w() const;
    void w_apply(Vec& z) const;
    void w_solve(Vec& z) const;
    void wt_apply(Vec& z) const;
    void wt_solve(Vec& z) const;
    void q_apply_t(Vec& y) const;
    void q_apply(Vec& y) const;
};
// SPQRFW01 factor file (transforms.cpp:129-289), orc_serialize.cpp
void save_factorization(const Factorization& f, const std::string& path);
Factorization load_factorization(const std::string& path);


// ------------------------------------------------------------- factorize ---
struct FactorizeOptions { double eps = 1e-2; int skip_levels = 3; bool store_q = false; };  // factorize.h:13-17
struct Front {  // factorize.h:24-29
    int cluster = -1;
    std::vector<Index> rows;
    std::map<int, Mat> blocks;
    bool scaled_ok = false;
};
struct EngineView { const std::map<int, Front>* fronts = nullptr; const std::vector<std::vector<Index>>* cols = nullptr; Index pivots = 0, dropped = 0, trailing = 0; };
struct FactorizeObserver { virtual ~FactorizeObserver() = default; virtual void on_phase(const char* phase, int stage, int detail, const EngineView& v) = 0; };
Factorization spaqr_factorize(const Csc& A, const ClusterHierarchy& h, const std::vector<int>& owner,
                              const FactorizeOptions& opt, FactorizeObserver* obs = nullptr);  // factorize.cpp:795-804

// ----------------------------------------------------------------- solve ---
struct SolveReport { int iterations = 0; bool converged = false; std::vector<double> residual_history; double t_solve = 0.0; Index dropped_rows = 0; };
struct CglsOptions { double tol = 1e-12; int maxit = 500; };
SolveReport cgls(const Csc& A, const Factorization* W, const Vec& b, Vec& u, const CglsOptions& opt, const Vec* weights = nullptr);  // solve.cpp:24-76
Vec csne_solve(const Csc& A, const Factorization& W, const Vec& b, int refine, SolveReport* rep, const Vec* weights, double tol);     // :78-108

// -------------------------------------------------------------- pipeline ---
enum class SolverKind { Spaqr = 0, Direct = 1, Diag = 2 };
struct PipelineOptions { double eps = 1e-2; int levels = 0; int skip_levels = 3; bool store_q = false; SolverKind solver = SolverKind::Spaqr; double tol = 1e-12; int maxit = 500; int refine = 1; };
struct Pipeline {  // pipeline.h:39-82
    PipelineOptions opt;
    Csc Aw;
    Vec d, weights;
    std::vector<Index> perm;
    std::vector<int> owner;
    SeparatorTree tree;
    ClusterHierarchy h;
    bool has_f = false;
    Factorization F;
    double t_partition = 0, t_factorize = 0;
    Pipeline(const Csc& A, const PipelineOptions& o, const Coords* coords, const std::vector<int>* parts, FactorizeObserver* obs = nullptr);
    Vec solve(const Vec& b, SolveReport* rep, double tol = -1.0, int maxit = -1) const;
    Vec solve_direct(const Vec& b, SolveReport* rep) const;
    Vec unscale(const Vec& u) const;
};

double now_s();

}  // namespace orc
