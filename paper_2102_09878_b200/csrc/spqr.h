// spaqr_b200 — host-side types of the B200 implementation of the spaQR hot path.
//
// These mirror the reference's public C++ API (proj/include/spaqr/*.h) with
// Eigen replaced by plain FP64 column-major storage.  The hot path (the
// per-level dense front work of factorize.cpp and the W sweeps of
// transforms.cpp inside CGLS) runs on the GPU: see engine.cpp / kernels.cu /
// solve.cpp.  Partitioning (partition.cpp) is host integer work that must be
// bit-exact with the reference and stays on the host.
#pragma once

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

namespace spqr {

// move_extras roundoff rule (factorize.cpp:141-164): candidate squared row norms at
// or below kMoveNoise2 x (largest squared row norm of the eliminated cluster's blocks) count as 0.
constexpr double kMoveNoise2 = (1e3 * 2.220446049250313e-16) * (1e3 * 2.220446049250313e-16);


using Index = int;  // proj/include/spaqr/types.h:11

struct SingularFrontError : std::runtime_error {  // types.h:24-31
    SingularFrontError(int cl, const std::string& why)
        : std::runtime_error("singular front (cluster " + std::to_string(cl) + "): " + why), cluster(cl), reason(why) {}
    int cluster;
    std::string reason;
};

struct CudaError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// Canonical CSC (sparse.h:15-38).
struct Csc {
    Index m = 0, n = 0;
    std::vector<Index> p, i;
    std::vector<double> x;
    Index nnz() const { return static_cast<Index>(x.size()); }
};
Csc csc_canonical(Index m, Index n, const Index* p, const Index* i, const double* x);  // sparse.cpp:13-20
std::vector<double> scale_columns(Csc& A);                                           // sparse.cpp:136-150
Csc permute_columns(const Csc& A, const std::vector<Index>& perm);                   // sparse.cpp:197-205

struct Graph {  // PatternGraph (sparse.h:65-68), CSR adjacency
    Index n = 0;
    std::vector<Index> ptr, adj;
    const Index* begin(Index v) const { return adj.data() + ptr[v]; }
    const Index* end(Index v) const { return adj.data() + ptr[v + 1]; }
};
Graph ata_graph(const Csc& A);  // sparse.cpp:170-195

struct SeparatorTree {  // partition.h:14-27
    struct Node {
        int level = 0, parent = -1;
        int child[2] = {-1, -1};
        std::vector<Index> vertices, separator;
        bool leaf() const { return child[0] < 0; }
    };
    int num_levels = 0, root = 0;
    std::vector<Node> nodes;
};
int default_num_levels(Index n);  // partition.cpp:15-19
SeparatorTree nested_dissection(const Graph& g, int L, const double* coords, int dim);  // :186-194
SeparatorTree import_partition(const Graph& g, int L, const int* parts);               // :196-214

struct ClusterHierarchy {  // partition.h:54-75
    struct Cluster {
        int tree_node = -1, level = 0, parent = -1, stage = 0;
        bool interior = false;
        std::vector<Index> cols;
    };
    int num_levels = 0;
    std::vector<Cluster> clusters;
    std::vector<int> finest_of_col;
    const SeparatorTree* tree = nullptr;
    bool related(int a, int b) const;
};
ClusterHierarchy build_interfaces(const SeparatorTree& t, const Graph& g);  // :231-346
std::vector<Index> order_columns(ClusterHierarchy& h);                        // :348-399
struct RowMatching { std::vector<Index> row_of_col, col_of_row; Index size = 0; };
RowMatching match_rows(const Csc& A);
// owner rank of every cluster for a G = 2^g GPU subtree split (ranks.cpp)
std::vector<int> rank_owners(const ClusterHierarchy& h, const Graph& g, int G);                                                // :401-463
std::vector<int> assign_rows(const Csc& A, const ClusterHierarchy& h, const RowMatching& m);  // :465-514

// Byte transport between the ranks of a distributed factorization (one process per GPU; the
// Python layer binds it to torch.distributed).  Blocking; returns 0 on success.
struct DistTransport {
    void* user = nullptr;
    int rank = 0, size = 1;
    int (*send)(void* user, int dst, const void* buf, long long n) = nullptr;
    int (*recv)(void* user, int src, void* buf, long long n) = nullptr;
};

struct FactorizeOptions {  // factorize.h:13-17
    double eps = 1e-2;
    int skip_levels = 3;
    bool store_q = false;  // keep the orthogonal row factors Q (tests, diagnostics)
    int ranks = 1;         // > 1: account work and cross-rank traffic of a ranks-GPU subtree split (ranks.cpp)
    const DistTransport* dist = nullptr;  // size > 1: the stages before the first scale_all run subtree-parallel
};

struct StageStats {  // transforms.h:40-47 (+ per-phase device-side timings)
    int stage = 0;
    double t_eliminate = 0, t_reassign = 0, t_scale = 0, t_sparsify = 0, t_merge = 0;
    std::vector<int> front_cols;
    std::vector<double> front_aspect;
    int top_rows = 0, top_cols = 0;
    long long nnz_w = 0;
};

double now_s();

}  // namespace spqr
