"""Oracle pinning: partition / sparse core against the reference's known
answers and invariants (proj/tests/test_partition.cpp, test_sparse.cpp)."""
import numpy as np
import scipy.sparse as sp

import oracle as O


def from_edges(n, edges):
    adj = [set() for _ in range(n)]
    for a, b in edges:
        adj[a].add(b)
        adj[b].add(a)
    ptr = np.zeros(n + 1, np.int32)
    flat = []
    for v in range(n):
        s = sorted(adj[v])
        flat += s
        ptr[v + 1] = len(flat)
    return ptr, np.array(flat, np.int32), [sorted(a) for a in adj]


def grid_graph(nx, ny):
    e = []
    for y in range(ny):
        for x in range(nx):
            if x + 1 < nx:
                e.append((x + nx * y, x + 1 + nx * y))
            if y + 1 < ny:
                e.append((x + nx * y, x + nx * (y + 1)))
    return from_edges(nx * ny, e)


def grid_coords(nx, ny):
    c = np.zeros((nx * ny, 2))
    for y in range(ny):
        for x in range(nx):
            c[x + nx * y] = (x, y)
    return c


def check_tree(t, adj, n, L):  # test_partition.cpp:64-114
    nodes = t.nodes()
    root = nodes[t.root]
    assert root["level"] == 1 and len(root["vertices"]) == n
    for i, nd in enumerate(nodes):
        assert np.all(np.diff(nd["vertices"]) > 0)
        if nd["child"][0] < 0:
            assert nd["level"] == L + 1 and len(nd["separator"]) == 0
            continue
        c0, c1 = nodes[nd["child"][0]], nodes[nd["child"][1]]
        assert c0["parent"] == i and c1["parent"] == i
        allv = np.sort(np.concatenate([c0["vertices"], c1["vertices"], nd["separator"]]))
        assert np.array_equal(allv, nd["vertices"])
        in0, in1 = set(c0["vertices"].tolist()), set(c1["vertices"].tolist())
        for v in c0["vertices"]:
            assert not any(u in in1 for u in adj[v])
        for s in nd["separator"]:
            assert any(u in in0 for u in adj[s]) and any(u in in1 for u in adj[s])


def test_default_num_levels_table():  # :223-232
    for n, L in [(1, 1), (64, 1), (65, 1), (128, 1), (129, 2), (256, 2), (257, 3), (4096, 6)]:
        assert O.default_num_levels(n) == L


def test_path_graph_single_vertex_separator():  # :234-242
    ptr, adj, al = from_edges(7, [(i, i + 1) for i in range(6)])
    t = O.Tree(ptr, adj, 1)
    check_tree(t, al, 7, 1)
    nodes = t.nodes()
    r = nodes[t.root]
    assert len(r["separator"]) == 1
    assert len(nodes[r["child"][0]]["vertices"]) + len(nodes[r["child"][1]]["vertices"]) == 6


def test_grid_root_separator_is_a_grid_column():  # :244-253
    ptr, adj, al = grid_graph(8, 8)
    coords = grid_coords(8, 8)
    t = O.Tree(ptr, adj, 2, coords=coords)
    check_tree(t, al, 64, 2)
    sep = t.nodes()[t.root]["separator"]
    assert len(sep) == 8
    assert np.all(coords[sep, 0] == coords[sep[0], 0])


def test_dissection_invariants_random_graphs():  # :255-272
    rng = np.random.default_rng(21)
    for _ in range(12):
        n = 20 + int(rng.integers(120))
        e = [(v - 1, v) for v in range(1, n)]
        for _ in range(n):
            a, b = int(rng.integers(n)), int(rng.integers(n))
            if a != b:
                e.append((min(a, b), max(a, b)))
        ptr, adj, al = from_edges(n, e)
        L = 1 + int(rng.integers(3))
        check_tree(O.Tree(ptr, adj, L), al, n, L)
        check_tree(O.Tree(ptr, adj, L, coords=rng.random((n, 2))), al, n, L)


def test_imported_partition_follows_bit_paths():  # :273-303
    ptr, adj, al = grid_graph(4, 4)
    parts = np.zeros(16, np.int32)
    for y in range(4):
        for x in range(4):
            parts[x + 4 * y] = (2 if y >= 2 else 0) + (1 if x >= 2 else 0)
    t = O.Tree(ptr, adj, 2, parts=parts)
    check_tree(t, al, 16, 2)
    nodes = t.nodes()

    def leaf_of(path):
        nd = t.root
        for bit in (1, 0):
            nd = nodes[nd]["child"][(path >> bit) & 1]
        return nd

    for v in range(16):
        if all(parts[u] == parts[v] for u in al[v]):
            assert v in set(nodes[leaf_of(int(parts[v]))]["vertices"].tolist())


def test_hierarchy_invariants():  # :116-177 (cluster ids, stages, nesting, column cover)
    ptr, adj, al = grid_graph(16, 16)
    t = O.Tree(ptr, adj, 3, coords=grid_coords(16, 16))
    cl = t.clusters()
    L = 3
    fin = t.finest_of_col()
    assert np.all(fin >= 0)
    for i, c in enumerate(cl):
        if c["level"] == L + 1:
            assert all(fin[v] == i for v in c["cols"])
        if c["parent"] >= 0:
            p = cl[c["parent"]]
            assert p["level"] == c["level"] - 1
            assert set(c["cols"].tolist()) <= set(p["cols"].tolist())
            assert c["stage"] == 0
        elif not c["interior"]:
            assert c["stage"] == c["level"]
    # every column is in exactly one finest cluster
    cover = np.concatenate([c["cols"] for c in cl if c["level"] == L + 1])
    assert np.array_equal(np.sort(cover), np.arange(256))
    perm = t.order()
    assert np.array_equal(np.sort(perm), np.arange(256))
    for c in t.clusters():  # contiguous ranges after ordering
        if len(c["cols"]):
            assert c["cols"][-1] - c["cols"][0] + 1 == len(c["cols"])


def kuhn(A):
    A = A.tocsc()
    m, n = A.shape
    rows_of = [A.indices[A.indptr[j]:A.indptr[j + 1]].tolist() for j in range(n)]
    mrow = [-1] * m

    def tryc(j, used):
        for r in rows_of[j]:
            if used[r]:
                continue
            used[r] = True
            if mrow[r] < 0 or tryc(mrow[r], used):
                mrow[r] = j
                return True
        return False

    return sum(tryc(j, [False] * m) for j in range(n))


def test_row_matching_maximum_cardinality():  # :399-427
    rng = np.random.default_rng(55)
    for _ in range(30):
        n = 3 + int(rng.integers(25))
        m = n + int(rng.integers(25))
        mask = rng.random((m, n)) < 0.12
        D = np.where(mask, rng.uniform(-1, 1, (m, n)), 0.0)
        A = sp.csc_matrix(D)
        rc, cr, size = O.match_rows(A)
        assert size == kuhn(A)
        paired = 0
        for j in range(n):
            if rc[j] < 0:
                continue
            paired += 1
            assert cr[rc[j]] == j and D[rc[j], j] != 0
        assert paired == size
    D = np.zeros((20, 12))
    D[np.arange(12), np.arange(12)] = 1.0 + np.arange(12)
    assert O.match_rows(sp.csc_matrix(D))[2] == 12


def test_row_assignment_rules():  # :429-449
    D = np.zeros((5, 3))
    D[0, 0], D[1, 2], D[2, 1], D[3, 0], D[3, 2] = 3.0, 2.0, 1.0, 1.0, -1.0
    A = sp.csc_matrix(D)
    ptr, adj, al = from_edges(3, [(0, 1), (1, 2)])
    t = O.Tree(ptr, adj, 1)
    own, rc, cr, size = t.assign_rows(A)
    fin = t.finest_of_col()
    assert size == 3
    assert own[0] == fin[0] and own[1] == fin[2] and own[2] == fin[1]
    assert own[3] == min(fin[0], fin[2])
    assert own[4] == fin[1]


def test_ata_graph_matches_bruteforce():  # test_sparse.cpp:233-262
    rng = np.random.default_rng(9)
    D = np.where(rng.random((30, 20)) < 0.15, rng.standard_normal((30, 20)), 0.0)
    ptr, adj = O.ata_graph(sp.csc_matrix(D))
    P = (D != 0).astype(int)
    G = (P.T @ P) > 0
    np.fill_diagonal(G, False)
    for v in range(20):
        assert adj[ptr[v]:ptr[v + 1]].tolist() == np.nonzero(G[v])[0].tolist()
