// Host-side structure for the spaQR hot path: canonical CSC, the A^T A pattern
// graph, nested dissection, the interface hierarchy, column ordering, row
// matching and row assignment.  This is integer work the GPU engine consumes;
// north_star requires it to be bit-exact with the reference, so every
// tie-break below follows proj/src/partition.cpp / sparse.cpp exactly (cited
// per function).  Data structures are flat (CSR adjacency, sorted vectors)
// rather than the reference's maps.
#include <algorithm>
#include <chrono>
#include <cmath>
#include <deque>
#include <limits>
#include <numeric>

#include "spqr.h"

namespace spqr {

double now_s() {
    return std::chrono::duration<double>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

// sparse.cpp:13-20 semantics: per column rows ascending, duplicates summed in
// input order, exact zeros dropped.
Csc csc_canonical(Index m, Index n, const Index* p, const Index* i, const double* x) {
    Csc A;
    A.m = m;
    A.n = n;
    A.p.assign(n + 1, 0);
    std::vector<std::pair<Index, double>> col;
    for (Index j = 0; j < n; ++j) {
        col.clear();
        for (Index k = p[j]; k < p[j + 1]; ++k) col.emplace_back(i[k], x[k]);
        std::stable_sort(col.begin(), col.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        for (size_t k = 0; k < col.size();) {
            const Index r = col[k].first;
            double s = 0.0;
            for (; k < col.size() && col[k].first == r; ++k) s += col[k].second;
            if (s != 0.0) {
                A.i.push_back(r);
                A.x.push_back(s);
            }
        }
        A.p[j + 1] = static_cast<Index>(A.x.size());
    }
    return A;
}

std::vector<double> scale_columns(Csc& A) {  // sparse.cpp:136-150
    std::vector<double> d(A.n);
    for (Index j = 0; j < A.n; ++j) {
        double s = 0.0;
        for (Index k = A.p[j]; k < A.p[j + 1]; ++k) s += A.x[k] * A.x[k];
        if (s == 0.0) throw std::invalid_argument("column " + std::to_string(j) + " is exactly zero");
        d[j] = std::sqrt(s);
        for (Index k = A.p[j]; k < A.p[j + 1]; ++k) A.x[k] /= d[j];
    }
    return d;
}

Csc permute_columns(const Csc& A, const std::vector<Index>& perm) {  // sparse.cpp:197-205
    Csc B;
    B.m = A.m;
    B.n = static_cast<Index>(perm.size());
    B.p.assign(B.n + 1, 0);
    B.i.reserve(A.nnz());
    B.x.reserve(A.nnz());
    for (Index j = 0; j < B.n; ++j) {  // source columns are canonical already
        for (Index k = A.p[perm[j]]; k < A.p[perm[j] + 1]; ++k) {
            B.i.push_back(A.i[k]);
            B.x.push_back(A.x[k]);
        }
        B.p[j + 1] = static_cast<Index>(B.x.size());
    }
    return B;
}

Graph ata_graph(const Csc& A) {  // sparse.cpp:170-195: row cliques, sorted, unique, no loops
    std::vector<Index> rptr(A.m + 1, 0), rcol(A.nnz());
    for (Index k = 0; k < A.nnz(); ++k) rptr[A.i[k] + 1]++;
    for (Index r = 0; r < A.m; ++r) rptr[r + 1] += rptr[r];
    {
        std::vector<Index> pos(rptr.begin(), rptr.end() - 1);
        for (Index j = 0; j < A.n; ++j)
            for (Index k = A.p[j]; k < A.p[j + 1]; ++k) rcol[pos[A.i[k]]++] = j;
    }
    // adjacency of v = sorted unique columns sharing a row with v, minus v; built
    // per column in parallel (count pass, then fill pass at the prefix offsets)
    Graph g;
    g.n = A.n;
    g.ptr.assign(A.n + 1, 0);
    auto neighbours = [&](Index v, std::vector<Index>& nb) {
        nb.clear();
        for (Index k = A.p[v]; k < A.p[v + 1]; ++k) {
            const Index r = A.i[k];
            for (Index a = rptr[r]; a < rptr[r + 1]; ++a)
                if (rcol[a] != v) nb.push_back(rcol[a]);
        }
        std::sort(nb.begin(), nb.end());
        nb.erase(std::unique(nb.begin(), nb.end()), nb.end());
    };
#pragma omp parallel
    {
        std::vector<Index> nb;
#pragma omp for schedule(dynamic, 1024)
        for (Index v = 0; v < A.n; ++v) {
            neighbours(v, nb);
            g.ptr[v + 1] = static_cast<Index>(nb.size());
        }
    }
    for (Index v = 0; v < A.n; ++v) g.ptr[v + 1] += g.ptr[v];
    g.adj.resize(static_cast<size_t>(g.ptr[A.n]));
#pragma omp parallel
    {
        std::vector<Index> nb;
#pragma omp for schedule(dynamic, 1024)
        for (Index v = 0; v < A.n; ++v) {
            neighbours(v, nb);
            std::copy(nb.begin(), nb.end(), g.adj.begin() + g.ptr[v]);
        }
    }
    return g;
}

int default_num_levels(Index n) {  // partition.cpp:15-19
    if (n <= 64) return 1;
    return std::max(1, static_cast<int>(std::ceil(std::log2(static_cast<double>(n) / 64.0))));
}

namespace {

struct Builder {
    const Graph& g;
    const double* X;
    int dim;
    const int* parts;
    int L;
    SeparatorTree t;
    // mark[v] = id of the tree node whose vertex set is being split (the serial
    // algorithm's "in current set" flag; sibling subtrees run concurrently on
    // disjoint vertex sets, so every per-vertex array is race-free)
    std::vector<int> mark;
    std::vector<signed char> side;
    std::vector<int> dist;

    Builder(const Graph& g_, const double* x, int d, const int* p, int L_)
        : g(g_), X(x), dim(d), parts(p), L(L_), mark(g_.n, -1), side(g_.n, -1), dist(g_.n, -1) {}

    double coord(Index v, int a) const { return X[static_cast<size_t>(v) * dim + a]; }

    // partition.cpp:26-49
    void split_geo(const std::vector<Index>& s, std::vector<Index>& s1, std::vector<Index>& s2) {
        int axis = 0;
        double best = -1.0;
        for (int a = 0; a < dim; ++a) {
            double lo = std::numeric_limits<double>::infinity(), hi = -lo;
            for (Index v : s) {
                lo = std::min(lo, coord(v, a));
                hi = std::max(hi, coord(v, a));
            }
            if (hi - lo > best) {
                best = hi - lo;
                axis = a;
            }
        }
        std::vector<std::pair<double, Index>> key(s.size());
        for (size_t k = 0; k < s.size(); ++k) key[k] = {coord(s[k], axis), s[k]};
        std::sort(key.begin(), key.end());
        const size_t h = s.size() / 2;
        s1.resize(h);
        s2.resize(s.size() - h);
        for (size_t k = 0; k < h; ++k) s1[k] = key[k].second;
        for (size_t k = h; k < s.size(); ++k) s2[k - h] = key[k].second;
    }

    // partition.cpp:51-87
    void split_bfs(const std::vector<Index>& s, std::vector<Index>& s1, std::vector<Index>& s2, int id) {
        auto sweep = [&](Index src) {
            for (Index v : s) dist[v] = -1;
            std::deque<Index> q{src};
            dist[src] = 0;
            Index far = src;
            while (!q.empty()) {
                const Index v = q.front();
                q.pop_front();
                if (dist[v] > dist[far] || (dist[v] == dist[far] && v < far)) far = v;
                for (const Index* u = g.begin(v); u != g.end(v); ++u)
                    if (mark[*u] == id && dist[*u] < 0) {
                        dist[*u] = dist[v] + 1;
                        q.push_back(*u);
                    }
            }
            return far;
        };
        const Index far = sweep(*std::min_element(s.begin(), s.end()));
        sweep(far);
        std::vector<std::pair<int, Index>> key(s.size());
        for (size_t k = 0; k < s.size(); ++k)
            key[k] = {dist[s[k]] < 0 ? std::numeric_limits<int>::max() : dist[s[k]], s[k]};
        std::sort(key.begin(), key.end());
        const size_t h = s.size() / 2;
        s1.resize(h);
        s2.resize(s.size() - h);
        for (size_t k = 0; k < h; ++k) s1[k] = key[k].second;
        for (size_t k = h; k < s.size(); ++k) s2[k - h] = key[k].second;
        for (Index v : s) dist[v] = -1;
    }

    // partition.cpp:103-147 (candidate order = side-2 order; in-pass updates)
    void carve(std::vector<Index>& s1, std::vector<Index>& s2, std::vector<Index>& sep, int id) {
        for (Index v : s1) side[v] = 0;
        for (Index v : s2) side[v] = 1;
        std::vector<Index> cand;
        for (Index v : s2)
            for (const Index* u = g.begin(v); u != g.end(v); ++u)
                if (mark[*u] == id && side[*u] == 0) {
                    cand.push_back(v);
                    break;
                }
        for (Index v : cand) side[v] = 2;
        for (bool moved = true; moved;) {
            moved = false;
            for (Index v : cand) {
                if (side[v] != 2) continue;
                bool t1 = false, t2 = false;
                for (const Index* u = g.begin(v); u != g.end(v); ++u) {
                    if (mark[*u] != id) continue;
                    t1 |= side[*u] == 0;
                    t2 |= side[*u] == 1;
                }
                if (!(t1 && t2)) {
                    side[v] = t2 ? 1 : 0;
                    moved = true;
                }
            }
        }
        std::vector<Index> n1(s1), n2;
        sep.clear();
        for (Index v : cand)
            if (side[v] == 0) n1.push_back(v);
        for (Index v : s2)
            if (side[v] == 1) n2.push_back(v);
        for (Index v : cand)
            if (side[v] == 2) sep.push_back(v);
        std::sort(n1.begin(), n1.end());
        std::sort(n2.begin(), n2.end());
        std::sort(sep.begin(), sep.end());
        for (Index v : s1) side[v] = -1;
        for (Index v : s2) side[v] = -1;
        s1.swap(n1);
        s2.swap(n2);
    }

    // nodes of a subtree rooted at `level` (every inner node has two children)
    int subtree_size(int level) const { return (1 << (L + 2 - level)) - 1; }

    // preorder ids: node id, then the left subtree, then the right one
    void grow(std::vector<Index> s, int level, int parent, int id) {
        std::sort(s.begin(), s.end());
        SeparatorTree::Node& nd = t.nodes[id];
        nd.level = level;
        nd.parent = parent;
        nd.vertices = s;
        if (level == L + 1) return;
        std::vector<Index> s1, s2, sep;
        if (parts) {
            const int bit = L - level;
            for (Index v : s) ((parts[v] >> bit) & 1 ? s2 : s1).push_back(v);
        } else if (!s.empty()) {
            for (Index v : s) mark[v] = id;
            if (X)
                split_geo(s, s1, s2);
            else
                split_bfs(s, s1, s2, id);
        }
        if (!s.empty()) {
            for (Index v : s) mark[v] = id;
            carve(s1, s2, sep, id);
        }
        nd.separator = sep;
        std::vector<Index>().swap(s);
        const int a = id + 1, b = id + 1 + subtree_size(level + 1);
        nd.child[0] = a;
        nd.child[1] = b;
        if (level <= 6) {  // the top levels fan out as tasks; deeper subtrees run in their task
#pragma omp task default(shared) firstprivate(a, level, id) shared(s1)
            grow(std::move(s1), level + 1, id, a);
#pragma omp task default(shared) firstprivate(b, level, id) shared(s2)
            grow(std::move(s2), level + 1, id, b);
#pragma omp taskwait
        } else {
            grow(std::move(s1), level + 1, id, a);
            grow(std::move(s2), level + 1, id, b);
        }
    }
};

}  // namespace

SeparatorTree nested_dissection(const Graph& g, int L, const double* coords, int dim) {
    if (L < 1) throw std::invalid_argument("num_levels must be >= 1");
    Builder b(g, coords, dim, nullptr, L);
    std::vector<Index> all(g.n);
    std::iota(all.begin(), all.end(), 0);
    b.t.num_levels = L;
    b.t.nodes.resize(static_cast<size_t>(b.subtree_size(1)));
    b.t.root = 0;
#pragma omp parallel
#pragma omp single
    b.grow(std::move(all), 1, -1, 0);
    return std::move(b.t);
}

SeparatorTree import_partition(const Graph& g, int L, const int* parts) {
    if (L < 1) throw std::invalid_argument("num_levels must be >= 1");
    for (Index v = 0; v < g.n; ++v)
        if (parts[v] < 0 || parts[v] >= (1 << L)) throw std::invalid_argument("part id outside [0,2^L)");
    Builder b(g, nullptr, 0, parts, L);
    std::vector<Index> all(g.n);
    std::iota(all.begin(), all.end(), 0);
    b.t.num_levels = L;
    b.t.nodes.resize(static_cast<size_t>(b.subtree_size(1)));
    b.t.root = 0;
#pragma omp parallel
#pragma omp single
    b.grow(std::move(all), 1, -1, 0);
    return std::move(b.t);
}

bool ClusterHierarchy::related(int a, int b) const {  // partition.cpp:223-229
    int ta = clusters[a].tree_node, tb = clusters[b].tree_node;
    if (tree->nodes[ta].level > tree->nodes[tb].level) std::swap(ta, tb);
    while (tb != -1 && tree->nodes[tb].level > tree->nodes[ta].level) tb = tree->nodes[tb].parent;
    return ta == tb;
}

// partition.cpp:231-346.  Pieces at granularity k: separator vertices grouped
// by their set of touched level-k regions, split into connected components,
// sorted by first vertex.  Group identity is all that matters, so signatures
// are compared as sorted vectors; components are found by BFS.
ClusterHierarchy build_interfaces(const SeparatorTree& t, const Graph& g) {
    ClusterHierarchy h;
    h.num_levels = t.num_levels;
    h.tree = &t;
    const int L = t.num_levels;
    std::vector<int> owner_node(g.n, -1);
    for (size_t id = 0; id < t.nodes.size(); ++id) {
        const auto& nd = t.nodes[id];
        for (Index v : (nd.leaf() ? nd.vertices : nd.separator)) owner_node[v] = static_cast<int>(id);
    }
    for (size_t id = 0; id < t.nodes.size(); ++id) {
        const auto& nd = t.nodes[id];
        if (!nd.leaf() || nd.vertices.empty()) continue;
        ClusterHierarchy::Cluster c;
        c.tree_node = static_cast<int>(id);
        c.level = c.stage = L + 1;
        c.interior = true;
        c.cols = nd.vertices;
        h.clusters.push_back(std::move(c));
    }
    std::vector<int> seps;
    for (size_t id = 0; id < t.nodes.size(); ++id)
        if (!t.nodes[id].leaf() && !t.nodes[id].separator.empty()) seps.push_back(static_cast<int>(id));
    std::stable_sort(seps.begin(), seps.end(), [&](int a, int b) {
        return t.nodes[a].level != t.nodes[b].level ? t.nodes[a].level > t.nodes[b].level : a < b;
    });
    // pieces of every separator at every granularity, computed per separator in
    // parallel (separators are disjoint vertex sets; mark[] carries the
    // separator id so concurrent flood fills never see each other's vertices),
    // then numbered sequentially in the reference's order (partition.cpp:284-339)
    std::vector<int> grp(g.n, -1), mark(g.n, 0);
    std::vector<std::vector<std::vector<std::vector<Index>>>> all_pieces(seps.size());
#pragma omp parallel for schedule(dynamic, 1)
    for (long long si = 0; si < static_cast<long long>(seps.size()); ++si) {
        const int sid = seps[si];
        const auto& nd = t.nodes[sid];
        const int l = nd.level;
        const auto& S = nd.separator;
        const int unvisited = sid + 1, visited = -(sid + 1);
        // per separator vertex: outside neighbours' owner nodes (fixed), climbed per k
        std::vector<Index> optr(S.size() + 1, 0), onode;
        for (size_t a = 0; a < S.size(); ++a) {
            for (const Index* u = g.begin(S[a]); u != g.end(S[a]); ++u)
                if (owner_node[*u] != sid) onode.push_back(owner_node[*u]);
            optr[a + 1] = static_cast<Index>(onode.size());
        }
        std::vector<std::vector<Index>> sigs;
        auto& per_k = all_pieces[si];
        for (int k = l; k <= L + 1; ++k) {
            per_k.emplace_back();
            std::vector<std::vector<Index>>& pieces = per_k.back();
            if (k == l) {
                pieces.push_back(S);
                continue;
            }
            sigs.assign(S.size(), {});
            for (size_t a = 0; a < S.size(); ++a) {
                auto& sig = sigs[a];
                for (Index q = optr[a]; q < optr[a + 1]; ++q) {
                    int x = onode[q];
                    while (t.nodes[x].level > k) x = t.nodes[x].parent;
                    sig.push_back(x);
                }
                std::sort(sig.begin(), sig.end());
                sig.erase(std::unique(sig.begin(), sig.end()), sig.end());
            }
            std::vector<Index> ord(S.size());
            std::iota(ord.begin(), ord.end(), 0);
            std::sort(ord.begin(), ord.end(), [&](Index a, Index b) { return sigs[a] < sigs[b]; });
            int gi = -1;
            for (size_t q = 0; q < ord.size(); ++q) {
                if (q == 0 || sigs[ord[q]] != sigs[ord[q - 1]]) ++gi;
                grp[S[ord[q]]] = gi;
            }
            for (Index v : S) mark[v] = unvisited;
            for (Index s0 : S) {  // ascending seeds
                if (mark[s0] != unvisited) continue;
                mark[s0] = visited;
                std::vector<Index> comp{s0};
                for (size_t q = 0; q < comp.size(); ++q) {
                    const Index v = comp[q];
                    for (const Index* u = g.begin(v); u != g.end(v); ++u)
                        if (mark[*u] == unvisited && grp[*u] == grp[v]) {
                            mark[*u] = visited;
                            comp.push_back(*u);
                        }
                }
                std::sort(comp.begin(), comp.end());
                pieces.push_back(std::move(comp));
            }
            for (Index v : S) mark[v] = 0;
            std::sort(pieces.begin(), pieces.end(), [](const auto& a, const auto& b) { return a.front() < b.front(); });
        }
    }
    std::vector<int> piece_of(g.n, -1);
    for (size_t si = 0; si < seps.size(); ++si) {
        const int sid = seps[si];
        const int l = t.nodes[sid].level;
        for (size_t kk = 0; kk < all_pieces[si].size(); ++kk) {
            const int k = l + static_cast<int>(kk);
            std::vector<std::pair<Index, int>> next;
            for (auto& pc : all_pieces[si][kk]) {
                ClusterHierarchy::Cluster c;
                const int cid = static_cast<int>(h.clusters.size());
                c.tree_node = sid;
                c.level = k;
                c.stage = (k == l) ? l : 0;
                c.parent = (k == l) ? -1 : piece_of[pc.front()];
                for (Index v : pc) next.emplace_back(v, cid);
                c.cols = std::move(pc);
                h.clusters.push_back(std::move(c));
            }
            for (auto& [v, cid] : next) piece_of[v] = cid;
        }
    }
    h.finest_of_col.assign(g.n, -1);
    for (size_t c = 0; c < h.clusters.size(); ++c)
        if (h.clusters[c].level == L + 1)
            for (Index v : h.clusters[c].cols) h.finest_of_col[v] = static_cast<int>(c);
    return h;
}

std::vector<Index> order_columns(ClusterHierarchy& h) {  // partition.cpp:348-399
    const SeparatorTree& t = *h.tree;
    const int L = h.num_levels;
    const size_t nc = h.clusters.size();
    std::vector<Index> perm;
    perm.reserve(h.finest_of_col.size());
    for (const auto& c : h.clusters)
        if (c.interior) perm.insert(perm.end(), c.cols.begin(), c.cols.end());
    std::vector<std::vector<int>> kids(nc);
    for (size_t c = 0; c < nc; ++c)
        if (h.clusters[c].parent >= 0) kids[h.clusters[c].parent].push_back(static_cast<int>(c));
    for (auto& ks : kids)
        std::sort(ks.begin(), ks.end(), [&](int a, int b) { return h.clusters[a].cols.front() < h.clusters[b].cols.front(); });
    std::vector<int> roots;
    for (size_t c = 0; c < nc; ++c)
        if (!h.clusters[c].interior && h.clusters[c].parent < 0) roots.push_back(static_cast<int>(c));
    std::sort(roots.begin(), roots.end(), [&](int a, int b) {
        const int la = t.nodes[h.clusters[a].tree_node].level, lb = t.nodes[h.clusters[b].tree_node].level;
        return la != lb ? la > lb : h.clusters[a].tree_node < h.clusters[b].tree_node;
    });
    std::vector<int> st;
    for (int r : roots) {
        st.assign(1, r);
        while (!st.empty()) {
            const int c = st.back();
            st.pop_back();
            if (h.clusters[c].level == L + 1) {
                perm.insert(perm.end(), h.clusters[c].cols.begin(), h.clusters[c].cols.end());
                continue;
            }
            for (auto it = kids[c].rbegin(); it != kids[c].rend(); ++it) st.push_back(*it);
        }
    }
    std::vector<Index> newpos(perm.size());
    for (size_t q = 0; q < perm.size(); ++q) newpos[perm[q]] = static_cast<Index>(q);
    for (auto& c : h.clusters) {
        for (Index& v : c.cols) v = newpos[v];
        std::sort(c.cols.begin(), c.cols.end());
    }
    std::vector<int> fin(perm.size());
    for (size_t o = 0; o < perm.size(); ++o) fin[newpos[o]] = h.finest_of_col[o];
    h.finest_of_col.swap(fin);
    return perm;
}

RowMatching match_rows(const Csc& A) {  // partition.cpp:401-463
    RowMatching res;
    res.row_of_col.assign(A.n, -1);
    res.col_of_row.assign(A.m, -1);
    for (Index j = 0; j < A.n; ++j) {
        Index best = -1;
        double bv = 0.0;
        for (Index k = A.p[j]; k < A.p[j + 1]; ++k) {
            if (res.col_of_row[A.i[k]] >= 0) continue;
            const double a = std::abs(A.x[k]);
            if (a > bv) {
                bv = a;
                best = A.i[k];
            }
        }
        if (best >= 0) {
            res.row_of_col[j] = best;
            res.col_of_row[best] = j;
            ++res.size;
        }
    }
    std::vector<Index> seen(A.m, -1), from(A.m, -1), q;
    for (Index j0 = 0; j0 < A.n; ++j0) {
        if (res.row_of_col[j0] >= 0) continue;
        q.assign(1, j0);
        Index fr = -1;
        for (size_t h = 0; h < q.size() && fr < 0; ++h) {
            const Index j = q[h];
            for (Index k = A.p[j]; k < A.p[j + 1]; ++k) {
                const Index r = A.i[k];
                if (seen[r] == j0) continue;
                seen[r] = j0;
                from[r] = j;
                if (res.col_of_row[r] < 0) {
                    fr = r;
                    break;
                }
                q.push_back(res.col_of_row[r]);
            }
        }
        if (fr < 0) continue;
        for (Index r = fr;;) {
            const Index j = from[r];
            const Index prev = res.row_of_col[j];
            res.row_of_col[j] = r;
            res.col_of_row[r] = j;
            if (j == j0) break;
            r = prev;
        }
        ++res.size;
    }
    return res;
}

std::vector<int> assign_rows(const Csc& A, const ClusterHierarchy& h, const RowMatching& m) {  // :465-514
    const int Lf = h.num_levels + 1;
    std::vector<int> owner(A.m, -1);
    int root_cl = -1;
    for (size_t c = 0; c < h.clusters.size() && root_cl < 0; ++c)
        if (h.clusters[c].level == Lf && !h.clusters[c].interior && h.clusters[c].tree_node == h.tree->root)
            root_cl = static_cast<int>(c);
    for (size_t c = 0; c < h.clusters.size() && root_cl < 0; ++c)
        if (h.clusters[c].level == Lf) root_cl = static_cast<int>(c);
    // row-major pass: per row (cluster, v) pairs in column order
    std::vector<Index> rptr(A.m + 1, 0);
    for (Index k = 0; k < A.nnz(); ++k) rptr[A.i[k] + 1]++;
    for (Index r = 0; r < A.m; ++r) rptr[r + 1] += rptr[r];
    std::vector<std::pair<int, double>> ent(A.nnz());
    {
        std::vector<Index> pos(rptr.begin(), rptr.end() - 1);
        for (Index j = 0; j < A.n; ++j)
            for (Index k = A.p[j]; k < A.p[j + 1]; ++k) ent[pos[A.i[k]]++] = {h.finest_of_col[j], A.x[k]};
    }
    std::vector<std::pair<int, double>> w;
    for (Index r = 0; r < A.m; ++r) {
        if (m.col_of_row[r] >= 0) {
            owner[r] = h.finest_of_col[m.col_of_row[r]];
            continue;
        }
        if (rptr[r] == rptr[r + 1]) {
            owner[r] = root_cl;
            continue;
        }
        // accumulate v^2 per cluster in column order (std::map semantics), ascending-id argmax
        w.clear();
        for (Index k = rptr[r]; k < rptr[r + 1]; ++k) {
            auto it = std::find_if(w.begin(), w.end(), [&](const auto& e) { return e.first == ent[k].first; });
            if (it == w.end())
                w.emplace_back(ent[k].first, ent[k].second * ent[k].second);
            else
                it->second += ent[k].second * ent[k].second;
        }
        std::sort(w.begin(), w.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
        int best = -1;
        double bw = -1.0;
        for (auto& [c, ww] : w)
            if (ww > bw) {
                bw = ww;
                best = c;
            }
        owner[r] = best;
    }
    return owner;
}

}  // namespace spqr
