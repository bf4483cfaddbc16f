// Subtree ownership for G = 2^g GPUs.
//
// The top g levels of the separator tree (partition.h:14-27; root at level 1, leaves at
// L+1, preorder ids) cut the domain into G subtrees; rank r owns the subtree whose root is
// the r-th level-(g+1) node from the left.  Every cluster (partition.cpp:231-346) whose tree
// node lies in subtree r belongs to rank r, at every granularity.  A piece of a top-g
// separator at granularity k > g sits where subtrees meet (its columns border level-k regions
// of one or more subtrees, the signature build_interfaces groups by): it belongs to the
// lowest-numbered subtree it borders (rank 0 when it borders none).  Pieces at granularity
// k <= g — the top levels — belong to rank 0, onto which the last merges gather every front.
#include <algorithm>
#include <stdexcept>

#include "spqr.h"

namespace spqr {

std::vector<int> rank_owners(const ClusterHierarchy& h, const Graph& g, int G) {
    const SeparatorTree& t = *h.tree;
    int lg = 0;
    while ((1 << lg) < G) ++lg;
    if (G < 1 || (1 << lg) != G) throw std::invalid_argument("rank count must be a power of two");
    if (lg > t.num_levels) throw std::invalid_argument("more ranks than level-(g+1) subtrees");
    // rank of every tree node below the top lg levels (-1 for the top separators)
    std::vector<int> node_rank(t.nodes.size(), -1);
    std::vector<int> path(t.nodes.size(), 0);  // child-choice bits from the root
    std::vector<int> stack{t.root};
    while (!stack.empty()) {
        const int v = stack.back();
        stack.pop_back();
        const auto& nd = t.nodes[v];
        if (nd.level > lg) node_rank[v] = path[v] >> (nd.level - lg - 1);
        for (int b = 0; b < 2; ++b)
            if (nd.child[b] >= 0) {
                path[nd.child[b]] = 2 * path[v] + b;
                stack.push_back(nd.child[b]);
            }
    }
    std::vector<int> owner(h.clusters.size(), 0);
    for (size_t c = 0; c < h.clusters.size(); ++c) {
        const auto& cl = h.clusters[c];
        const int r = node_rank[cl.tree_node];
        if (r >= 0) {
            owner[c] = r;
            continue;
        }
        if (cl.level <= lg) continue;  // top levels: rank 0
        int best = G;
        for (Index v : cl.cols)
            for (const Index* u = g.begin(v); u != g.end(v); ++u) {
                const int f = h.finest_of_col[*u];
                const int ru = f >= 0 ? node_rank[h.clusters[f].tree_node] : -1;
                if (ru >= 0) best = std::min(best, ru);
            }
        owner[c] = best < G ? best : 0;
    }
    return owner;
}

}  // namespace spqr
