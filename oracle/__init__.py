"""ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front-end to oracle/liboracle.so, the single-threaded Eigen-free CPU
restatement of the spaQR reference (see oracle/orc_core.h for what it restates
and how it is pinned).  Only tests/, __graft_entry__.smoke() and bench.py's
CPU-baseline legs may import this module; the product package never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
# oracle/ref.py re-executes this module with _LIB_OVERRIDE set to oracle/_ref/libspaqr_ref.so:
# the reference's own sources behind the same orc_* ABI (see oracle/ref_capi.cpp).
_LIB = globals().get("_LIB_OVERRIDE") or os.path.join(_HERE, "liboracle.so")
_MAKEFILE = globals().get("_MAKEFILE_OVERRIDE") or "Makefile"
_lib = None

i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")


class SingularFrontError(RuntimeError):
    def __init__(self, cluster, msg):
        super().__init__(msg)
        self.cluster = cluster
        self.reason = msg.split("| reason: ")[-1]


def build():
    subprocess.run(["make", "-s", "-C", _HERE, "-f", _MAKEFILE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            build()
        _lib = C.CDLL(_LIB)
        L = _lib
        vp = C.c_void_p
        L.orc_pipeline_new.restype = vp
        L.orc_pipeline_new.argtypes = [C.c_int, C.c_int, i32p, i32p, f64p, vp, C.c_int, vp, C.c_int, C.c_double,
                                       C.c_int, C.c_int, C.c_int, C.c_int, C.c_char_p, C.c_int,
                                       C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_pipeline_free.argtypes = [vp]
        L.orc_pipeline_info.argtypes = [vp, i64p]
        L.orc_pipeline_times.argtypes = [vp, f64p]
        L.orc_pipeline_perm.argtypes = [vp, i32p]
        L.orc_pipeline_owner.argtypes = [vp, i32p]
        L.orc_pipeline_weights.argtypes = [vp, f64p]
        L.orc_pipeline_scaled.argtypes = [vp, i32p, i32p, f64p]
        L.orc_pipeline_rows.argtypes = [vp, i32p, i32p, i32p]
        L.orc_pipeline_cluster.argtypes = [vp, C.c_int, i32p]
        L.orc_pipeline_cluster_cols.argtypes = [vp, C.c_int, i32p]
        L.orc_pipeline_stage.argtypes = [vp, C.c_int, i64p, f64p]
        L.orc_pipeline_stage_fronts.argtypes = [vp, C.c_int, i32p, f64p]
        L.orc_pipeline_phase.argtypes = [vp, C.c_int, C.c_char_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.orc_pipeline_wfactor.argtypes = [vp, C.c_int, i32p]
        L.orc_pipeline_wfactor_data.argtypes = [vp, C.c_int, i32p, f64p, i32p, f64p, f64p]
        L.orc_pipeline_apply.argtypes = [vp, C.c_int, f64p, C.c_char_p, C.c_int]
        L.orc_pipeline_save.argtypes = [vp, C.c_char_p, C.c_char_p, C.c_int]
        L.orc_factor_file_apply.argtypes = [C.c_char_p, C.c_int, vp, C.c_longlong, i64p, C.c_char_p, C.c_int]
        L.orc_pipeline_solve.argtypes = [vp, C.c_int, f64p, f64p, C.c_double, C.c_int, C.POINTER(C.c_int),
                                         C.POINTER(C.c_int), f64p, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                         C.c_char_p, C.c_int]
        L.orc_cgls_plain.argtypes = [C.c_int, C.c_int, i32p, i32p, f64p, f64p, vp, C.c_double, C.c_int, f64p,
                                     C.POINTER(C.c_int), C.POINTER(C.c_int), f64p, C.POINTER(C.c_int)]
        L.orc_householder_qr.argtypes = [C.c_int, C.c_int, f64p, f64p, f64p, f64p, f64p]
        L.orc_apply_reflectors.argtypes = [C.c_int, C.c_int, f64p, f64p, f64p, C.c_int, C.c_int, C.c_int, f64p]
        L.orc_cpqr.argtypes = [C.c_int, C.c_int, f64p, C.c_double, C.POINTER(C.c_int), C.POINTER(C.c_double),
                               i32p, f64p, f64p, f64p, f64p]
        L.orc_tri_solve.argtypes = [C.c_int, f64p, C.c_int, C.c_int, f64p, C.c_int, C.c_int, C.c_char_p, C.c_int]
        L.orc_check_diag.argtypes = [C.c_int, f64p, C.c_char_p, C.c_int]
        L.orc_graph_tree_new.restype = vp
        L.orc_graph_tree_new.argtypes = [C.c_int, i32p, i32p, vp, C.c_int, vp, C.c_int, C.c_char_p, C.c_int,
                                         C.POINTER(C.c_int)]
        L.orc_tree_free.argtypes = [vp]
        for f in ("orc_tree_nnodes", "orc_tree_root", "orc_tree_nclusters"):
            getattr(L, f).argtypes = [vp]
        L.orc_tree_node.argtypes = [vp, C.c_int, i32p]
        L.orc_tree_node_sets.argtypes = [vp, C.c_int, i32p, i32p]
        L.orc_tree_cluster.argtypes = [vp, C.c_int, i32p]
        L.orc_tree_cluster_cols.argtypes = [vp, C.c_int, i32p]
        L.orc_tree_finest.argtypes = [vp, i32p]
        L.orc_tree_related.argtypes = [vp, C.c_int, C.c_int]
        L.orc_tree_order.argtypes = [vp, i32p]
        L.orc_tree_assign_rows.argtypes = [vp, C.c_int, C.c_int, i32p, i32p, f64p, i32p, i32p, i32p]
        L.orc_match_rows.argtypes = [C.c_int, C.c_int, i32p, i32p, f64p, i32p, i32p]
        L.orc_ata_graph.restype = C.c_longlong
        L.orc_ata_graph.argtypes = [C.c_int, C.c_int, i32p, i32p, f64p, vp, vp]
        L.orc_from_triplets.argtypes = [C.c_int, C.c_int, C.c_int, i32p, i32p, f64p, vp, vp, vp]
    return _lib


def _csc(A):
    A = A.tocsc()
    return (int(A.shape[0]), int(A.shape[1]), np.ascontiguousarray(A.indptr, np.int32),
            np.ascontiguousarray(A.indices, np.int32), np.ascontiguousarray(A.data, np.float64))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def default_num_levels(n):
    return lib().orc_default_num_levels(int(n))


SOLVERS = {"spaqr": 0, "direct": 1, "diag": 2}


class Pipeline:
    """Mirror of spaqr::Pipeline (pipeline.h:39-82) over the oracle."""

    def __init__(self, A, eps=1e-2, levels=0, skip_levels=3, store_q=False, solver="spaqr", coords=None,
                 parts=None, check_invariants=False):
        L = lib()
        m, n, p, i, x = _csc(A)
        self._keep = []
        cp = None
        dim = 0
        if coords is not None:
            cp = np.ascontiguousarray(coords, np.float64)
            dim = cp.shape[1]
            self._keep.append(cp)
        pp = None
        if parts is not None:
            pp = np.ascontiguousarray(parts, np.int32)
            self._keep.append(pp)
        err = C.create_string_buffer(512)
        code, cl = C.c_int(0), C.c_int(-1)
        self.h = L.orc_pipeline_new(m, n, p, i, x, _ptr(cp), dim, _ptr(pp), int(levels), float(eps), int(skip_levels),
                                    int(store_q), SOLVERS[solver], int(check_invariants), err, 512, C.byref(code),
                                    C.byref(cl))
        if not self.h:
            msg = err.value.decode()
            if code.value == 1:
                raise SingularFrontError(cl.value, msg)
            if code.value == 2:
                raise ValueError(msg)
            raise RuntimeError(msg)
        info = np.zeros(13, np.int64)
        L.orc_pipeline_info(self.h, info)
        (self.M, self.N, self.L, self.nclusters, self.nW, self.nQ, self.ndropped, self.ntrailing, self.nstages,
         self.nnz_w, self.nnz_A, self.violations, self.nphases) = [int(v) for v in info]

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_pipeline_free(self.h)
            self.h = None

    def times(self):
        t = np.zeros(2)
        lib().orc_pipeline_times(self.h, t)
        return {"t_partition": t[0], "t_factorize": t[1]}

    def perm(self):
        o = np.zeros(self.N, np.int32)
        lib().orc_pipeline_perm(self.h, o)
        return o

    def owner(self):
        o = np.zeros(self.M, np.int32)
        lib().orc_pipeline_owner(self.h, o)
        return o

    def weights(self):
        o = np.zeros(self.N)
        lib().orc_pipeline_weights(self.h, o)
        return o

    def scaled(self):
        import scipy.sparse as sp
        p = np.zeros(self.N + 1, np.int32)
        i = np.zeros(self.nnz_A, np.int32)
        x = np.zeros(self.nnz_A)
        lib().orc_pipeline_scaled(self.h, p, i, x)
        return sp.csc_matrix((x, i, p), shape=(self.M, self.N))

    def rows(self):
        pr = np.zeros(self.N, np.int32)
        dr = np.zeros(max(self.ndropped, 1), np.int32)
        tr = np.zeros(max(self.ntrailing, 1), np.int32)
        lib().orc_pipeline_rows(self.h, pr, dr, tr)
        return pr, dr[: self.ndropped], tr[: self.ntrailing]

    def clusters(self):
        out = []
        info = np.zeros(6, np.int32)
        for c in range(self.nclusters):
            lib().orc_pipeline_cluster(self.h, c, info)
            cols = np.zeros(max(int(info[5]), 1), np.int32)
            lib().orc_pipeline_cluster_cols(self.h, c, cols)
            out.append(dict(tree_node=int(info[0]), level=int(info[1]), parent=int(info[2]), stage=int(info[3]),
                            interior=bool(info[4]), cols=cols[: int(info[5])].copy()))
        return out

    def stages(self):
        out = []
        o = np.zeros(5, np.int64)
        t = np.zeros(5)
        for s in range(self.nstages):
            lib().orc_pipeline_stage(self.h, s, o, t)
            nf = int(o[1])
            fc = np.zeros(max(nf, 1), np.int32)
            fa = np.zeros(max(nf, 1))
            lib().orc_pipeline_stage_fronts(self.h, s, fc, fa)
            out.append(dict(stage=int(o[0]), front_cols=fc[:nf].copy(), front_aspect=fa[:nf].copy(),
                            top_rows=int(o[2]), top_cols=int(o[3]), nnz_w=int(o[4]),
                            t_eliminate=t[0], t_reassign=t[1], t_scale=t[2], t_sparsify=t[3], t_merge=t[4]))
        return out

    def phases(self):
        out = []
        buf = C.create_string_buffer(32)
        st, de = C.c_int(), C.c_int()
        for i in range(self.nphases):
            lib().orc_pipeline_phase(self.h, i, buf, 32, C.byref(st), C.byref(de))
            out.append((buf.value.decode(), st.value, de.value))
        return out

    def wfactors(self):
        """List of ('tri', cols, R, coupled, C) / ('rot', cols, V, tau, sign)."""
        out = []
        info = np.zeros(3, np.int32)
        for f in range(self.nW):
            lib().orc_pipeline_wfactor(self.h, f, info)
            kind, c, d = int(info[0]), int(info[1]), int(info[2])
            cols = np.zeros(max(c, 1), np.int32)
            if kind == 0:
                R = np.zeros(max(c * c, 1))
                cp = np.zeros(max(d, 1), np.int32)
                Cm = np.zeros(max(c * d, 1))
                lib().orc_pipeline_wfactor_data(self.h, f, cols, R, cp, Cm, np.zeros(1))
                out.append(("tri", cols[:c].copy(), R[: c * c].reshape(c, c, order="F").copy(), cp[:d].copy(),
                            Cm[: c * d].reshape(c, d, order="F").copy()))
            else:
                V = np.zeros(max(c * d, 1))
                tau = np.zeros(max(d, 1))
                sg = np.zeros(max(d, 1))
                lib().orc_pipeline_wfactor_data(self.h, f, cols, V, np.zeros(1, np.int32), tau, sg)
                out.append(("rot", cols[:c].copy(), V[: c * d].reshape(c, d, order="F").copy(), tau[:d].copy(),
                            sg[:d].copy()))
        return out

    def _apply(self, mode, z):
        z = np.ascontiguousarray(z, np.float64).copy()
        err = C.create_string_buffer(256)
        rc = lib().orc_pipeline_apply(self.h, mode, z, err, 256)
        if rc:
            raise RuntimeError(err.value.decode())
        return z

    def save(self, path):
        """save_factorization (transforms.cpp:206-240): SPQRFW01 file."""
        err = C.create_string_buffer(512)
        if lib().orc_pipeline_save(self.h, str(path).encode(), err, 512):
            raise RuntimeError(err.value.decode())

    def w_apply(self, z): return self._apply(0, z)
    def w_solve(self, z): return self._apply(1, z)
    def wt_apply(self, z): return self._apply(2, z)
    def wt_solve(self, z): return self._apply(3, z)
    def q_apply_t(self, y): return self._apply(4, y)
    def q_apply(self, y): return self._apply(5, y)

    def solve(self, b, tol=-1.0, maxit=-1, direct=False):
        b = np.ascontiguousarray(b, np.float64)
        x = np.zeros(self.N)
        mi = maxit if maxit > 0 else 500
        hist = np.zeros(mi + 4)
        it, cv, nh = C.c_int(), C.c_int(), C.c_int()
        ts = C.c_double()
        err = C.create_string_buffer(256)
        rc = lib().orc_pipeline_solve(self.h, int(direct), b, x, float(tol), int(maxit), C.byref(it), C.byref(cv),
                                      hist, C.byref(nh), C.byref(ts), err, 256)
        if rc:
            raise RuntimeError(err.value.decode())
        return x, dict(iterations=it.value, converged=bool(cv.value), residual_history=hist[: nh.value].copy(),
                       t_solve=ts.value, dropped_rows=self.ndropped)


def cgls_plain(A, b, tol=1e-12, maxit=500, weights=None):
    m, n, p, i, x = _csc(A)
    b = np.ascontiguousarray(b, np.float64)
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    u = np.zeros(n)
    hist = np.zeros(maxit + 2)
    it, cv, nh = C.c_int(), C.c_int(), C.c_int()
    lib().orc_cgls_plain(m, n, p, i, x, b, _ptr(w), tol, maxit, u, C.byref(it), C.byref(cv), hist, C.byref(nh))
    return u, dict(iterations=it.value, converged=bool(cv.value), residual_history=hist[: nh.value].copy())


# ------------------------------------------------------------ dense kernels
def householder_qr(B):
    B = np.asfortranarray(B, np.float64)
    m, n = B.shape
    V = np.zeros(m * n)
    tau = np.zeros(max(n, 1))
    sg = np.zeros(max(n, 1))
    R = np.zeros(max(n * n, 1))
    lib().orc_householder_qr(m, n, np.ascontiguousarray(B.ravel(order="F")), V, tau, sg, R)
    return V.reshape(m, n, order="F"), tau[:n], sg[:n], R[: n * n].reshape(n, n, order="F")


def apply_reflectors(V, tau, sign, X, mode):
    """mode: 'left_t' (H^T X), 'left' (H X), 'right' (X H), 'right_t' (X H^T)."""
    V = np.asfortranarray(V, np.float64)
    m, k = V.shape
    X = np.asfortranarray(X, np.float64)
    xr, xc = X.shape
    flat = np.array(X.ravel(order="F"), dtype=np.float64, copy=True)
    md = {"left_t": 0, "left": 1, "right": 2, "right_t": 3}[mode]
    lib().orc_apply_reflectors(m, k, np.ascontiguousarray(V.ravel(order="F")), np.ascontiguousarray(tau, np.float64),
                               np.ascontiguousarray(sign, np.float64), md, xr, xc, flat)
    return flat.reshape(xr, xc, order="F")


def cpqr(B, eps):
    B = np.asfortranarray(B, np.float64)
    m, n = B.shape
    kmax = max(min(m, n), 1)
    rank, r11 = C.c_int(), C.c_double()
    perm = np.zeros(kmax, np.int32)
    R = np.zeros(kmax * max(n, 1))
    V = np.zeros(max(m, 1) * kmax)
    tau = np.zeros(kmax)
    sg = np.zeros(kmax)
    lib().orc_cpqr(m, n, np.ascontiguousarray(B.ravel(order="F")) if B.size else np.zeros(1), float(eps),
                   C.byref(rank), C.byref(r11), perm, R, V, tau, sg)
    r = rank.value
    return dict(rank=r, r11=r11.value, perm=perm[:r].copy(), R=R[: r * n].reshape(r, n, order="F").copy(),
                V=V[: m * r].reshape(m, r, order="F").copy(), tau=tau[:r].copy(), sign=sg[:r].copy())


def tri_solve_upper(R, B, side="left", transpose=False):
    R = np.asfortranarray(R, np.float64)
    B = np.asfortranarray(B, np.float64)
    flat = np.array(B.ravel(order="F"), dtype=np.float64, copy=True)
    err = C.create_string_buffer(256)
    rc = lib().orc_tri_solve(R.shape[0], np.ascontiguousarray(R.ravel(order="F")), B.shape[0], B.shape[1], flat,
                             int(side == "right"), int(transpose), err, 256)
    if rc == 1:
        raise SingularFrontError(-1, err.value.decode())
    return flat.reshape(B.shape, order="F")


def check_diag_invertible(R):
    R = np.asfortranarray(R, np.float64)
    err = C.create_string_buffer(256)
    rc = lib().orc_check_diag(R.shape[0], np.ascontiguousarray(R.ravel(order="F")), err, 256)
    if rc == 1:
        raise SingularFrontError(-1, err.value.decode())


# ------------------------------------------------------------ partition
def ata_graph(A):
    m, n, p, i, x = _csc(A)
    tot = lib().orc_ata_graph(m, n, p, i, x, None, None)
    ptr = np.zeros(n + 1, np.int32)
    adj = np.zeros(max(tot, 1), np.int32)
    lib().orc_ata_graph(m, n, p, i, x, _ptr(ptr), _ptr(adj))
    return ptr, adj[:tot]


class Tree:
    """nested_dissection / import_partition + build_interfaces (+ order_columns)."""

    def __init__(self, adjptr, adj, L, coords=None, parts=None):
        n = len(adjptr) - 1
        self.n = n
        self._keep = [np.ascontiguousarray(adjptr, np.int32), np.ascontiguousarray(adj, np.int32)]
        cp = pp = None
        dim = 0
        if coords is not None:
            cp = np.ascontiguousarray(coords, np.float64)
            dim = cp.shape[1]
        if parts is not None:
            pp = np.ascontiguousarray(parts, np.int32)
        self._keep += [cp, pp]
        err = C.create_string_buffer(256)
        code = C.c_int()
        self.h = lib().orc_graph_tree_new(n, self._keep[0], self._keep[1], _ptr(cp), dim, _ptr(pp), int(L), err,
                                          256, C.byref(code))
        if not self.h:
            raise ValueError(err.value.decode())

    def __del__(self):
        if getattr(self, "h", None):
            lib().orc_tree_free(self.h)
            self.h = None

    @property
    def root(self):
        return lib().orc_tree_root(self.h)

    def nodes(self):
        out = []
        info = np.zeros(6, np.int32)
        for i in range(lib().orc_tree_nnodes(self.h)):
            lib().orc_tree_node(self.h, i, info)
            v = np.zeros(max(int(info[4]), 1), np.int32)
            s = np.zeros(max(int(info[5]), 1), np.int32)
            lib().orc_tree_node_sets(self.h, i, v, s)
            out.append(dict(level=int(info[0]), parent=int(info[1]), child=(int(info[2]), int(info[3])),
                            vertices=v[: int(info[4])].copy(), separator=s[: int(info[5])].copy()))
        return out

    def clusters(self):
        out = []
        info = np.zeros(6, np.int32)
        for c in range(lib().orc_tree_nclusters(self.h)):
            lib().orc_tree_cluster(self.h, c, info)
            cols = np.zeros(max(int(info[5]), 1), np.int32)
            lib().orc_tree_cluster_cols(self.h, c, cols)
            out.append(dict(tree_node=int(info[0]), level=int(info[1]), parent=int(info[2]), stage=int(info[3]),
                            interior=bool(info[4]), cols=cols[: int(info[5])].copy()))
        return out

    def finest_of_col(self):
        o = np.zeros(self.n, np.int32)
        lib().orc_tree_finest(self.h, o)
        return o

    def related(self, a, b):
        return bool(lib().orc_tree_related(self.h, a, b))

    def order(self):
        o = np.zeros(self.n, np.int32)
        lib().orc_tree_order(self.h, o)
        return o

    def assign_rows(self, A):
        m, n, p, i, x = _csc(A)
        own = np.zeros(m, np.int32)
        rc = np.zeros(n, np.int32)
        cr = np.zeros(m, np.int32)
        size = lib().orc_tree_assign_rows(self.h, m, n, p, i, x, own, rc, cr)
        return own, rc, cr, size


def match_rows(A):
    m, n, p, i, x = _csc(A)
    rc = np.zeros(n, np.int32)
    cr = np.zeros(m, np.int32)
    size = lib().orc_match_rows(m, n, p, i, x, rc, cr)
    return rc, cr, size


def factor_file_apply(path, mode, z=None):
    """load_factorization (transforms.cpp:242-289) of an SPQRFW01 file, then one sweep:
    mode 'w_apply' | 'w_solve' | 'wt_apply' | 'wt_solve' (z of length N) or 'q_apply_t' | 'q_apply'
    (length M, store_q files).  Returns (M, N, nW) and the transformed copy of z (None when z is
    None)."""
    md = {"w_apply": 0, "w_solve": 1, "wt_apply": 2, "wt_solve": 3, "q_apply_t": 4, "q_apply": 5}[mode]
    dims = np.zeros(3, np.int64)
    err = C.create_string_buffer(512)
    v = None if z is None else np.array(z, np.float64, copy=True)
    rc = lib().orc_factor_file_apply(str(path).encode(), md, None if v is None else v.ctypes.data_as(C.c_void_p),
                                     0 if v is None else len(v), dims, err, 512)
    if rc:
        raise RuntimeError(err.value.decode())
    return tuple(int(d) for d in dims), v
