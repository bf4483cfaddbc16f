"""Python mirror of the reference's public API over the C ABI.

Names, argument meaning and error behaviour follow proj/include/spaqr:
Pipeline(A, opt, coords, parts) (pipeline.h:39-44), Pipeline.solve /
solve_direct (:46-52), Factorization.w_apply/w_solve/wt_apply/wt_solve
(transforms.h:66-69), SingularFrontError{cluster, reason} (types.h:24-31).
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import lib, require_gpu

SOLVERS = {"spaqr": 0, "direct": 1, "diag": 2}


class SingularFrontError(RuntimeError):
    def __init__(self, cluster, msg):
        super().__init__(msg)
        self.cluster = cluster
        self.reason = msg.split("| reason: ")[-1]


def _csc(A):
    A = A.tocsc()
    return (int(A.shape[0]), int(A.shape[1]), np.ascontiguousarray(A.indptr, np.int32),
            np.ascontiguousarray(A.indices, np.int32), np.ascontiguousarray(A.data, np.float64))


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


class _EngineView(C.Structure):  # spqr_engine_view (include/spaqr_b200.h)
    _fields_ = [("nfronts", C.c_int), ("front_cluster", C.POINTER(C.c_int)), ("rows_ptr", C.POINTER(C.c_int)),
                ("rows", C.POINTER(C.c_int)), ("keys_ptr", C.POINTER(C.c_int)), ("keys", C.POINTER(C.c_int)),
                ("key_width", C.POINTER(C.c_int)), ("block_off", C.POINTER(C.c_longlong)),
                ("values", C.POINTER(C.c_double)), ("nclusters", C.c_int), ("cols_ptr", C.POINTER(C.c_int)),
                ("cols", C.POINTER(C.c_int)), ("nwave", C.c_int), ("wave", C.POINTER(C.c_int)),
                ("pivots", C.c_longlong), ("dropped", C.c_longlong), ("trailing", C.c_longlong)]


_OBSERVER_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_char_p, C.c_int, C.c_int, C.POINTER(_EngineView))


def _arr(p, n, dt):
    return np.ctypeslib.as_array(p, shape=(n,)).astype(dt, copy=True) if n > 0 else np.zeros(0, dt)


def _observer(fn):
    """Wrap fn(phase, stage, detail, view) — FactorizeObserver::on_phase (factorize.h:40-43) —
    as the C callback; view = dict(fronts={cluster: dict(rows, blocks={key: ndarray})},
    cols=[active columns per cluster], wave, pivots, dropped, trailing) copied to numpy."""
    if fn is None:
        return None

    def cb(user, phase, stage, detail, vp_):
        v = vp_.contents
        nf = v.nfronts
        rp = _arr(v.rows_ptr, nf + 1, np.int64)
        kp = _arr(v.keys_ptr, nf + 1, np.int64)
        fc = _arr(v.front_cluster, nf, np.int64)
        nkeys = int(kp[-1]) if nf else 0
        rows = _arr(v.rows, int(rp[-1]) if nf else 0, np.int64)
        keys = _arr(v.keys, nkeys, np.int64)
        kw = _arr(v.key_width, nkeys, np.int64)
        bo = _arr(v.block_off, nkeys, np.int64)
        have_vals = bool(v.values)
        nval = int(bo[-1] + kw[-1] * (rp[-1] - rp[-2])) if (nkeys and have_vals) else 0
        vals = _arr(v.values, nval, np.float64) if have_vals else None
        fronts = {}
        for f in range(nf):
            nr = int(rp[f + 1] - rp[f])
            blocks = {}
            for b in range(int(kp[f]), int(kp[f + 1])):
                w = int(kw[b])
                blocks[int(keys[b])] = (vals[bo[b]: bo[b] + nr * w].reshape(w, nr).T.copy() if vals is not None
                                        else np.zeros((nr, w)))  # SPQR_OBSERVE_STRUCTURE_ONLY
            fronts[int(fc[f])] = dict(rows=rows[rp[f]: rp[f + 1]].copy(), blocks=blocks)
        cp = _arr(v.cols_ptr, v.nclusters + 1, np.int64)
        cols_all = _arr(v.cols, int(cp[-1]), np.int64)
        cols = [cols_all[cp[c]: cp[c + 1]] for c in range(v.nclusters)]
        fn(phase.decode(), stage, detail, dict(fronts=fronts, cols=cols, wave=_arr(v.wave, v.nwave, np.int64).tolist(),
                                               pivots=v.pivots, dropped=v.dropped, trailing=v.trailing))
    return _OBSERVER_FN(cb)


_SEND_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_longlong)
_RECV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_int, C.c_void_p, C.c_longlong)


def _transport(group):
    """The blocking byte transport of spqr_pipeline_create_dist over a torch.distributed group
    (CPU tensors: a gloo group; under an NCCL default group pass dist.new_group(backend="gloo"))."""
    import torch
    import torch.distributed as dist

    def send(user, dst, buf, n):
        try:
            a = np.ctypeslib.as_array(C.cast(buf, C.POINTER(C.c_uint8)), shape=(int(n),))
            dist.send(torch.from_numpy(a.copy()), dst, group=group)
            return 0
        except Exception:
            return 1

    def recv(user, src, buf, n):
        try:
            t = torch.empty(int(n), dtype=torch.uint8)
            dist.recv(t, src, group=group)
            C.memmove(buf, t.numpy().ctypes.data, int(n))
            return 0
        except Exception:
            return 1

    return _SEND_FN(send), _RECV_FN(recv)


class Pipeline:
    """spqr_pipeline_create / _solve / _apply (include/spaqr_b200.h).  observer: an optional
    fn(phase, stage, detail, view) called after every engine phase (pipeline.h:39-41)."""

    def __init__(self, A, eps=1e-2, levels=0, skip_levels=3, solver="spaqr", coords=None, parts=None, device=0,
                 observer=None, store_q=False, ranks=1, dist_group=None):
        require_gpu()
        L = lib()
        m, n, p, i, x = _csc(A)
        if coords is not None and np.asarray(coords).shape[0] != n:  # pipeline.cpp:39-40
            raise ValueError("coordinate row count does not match column count")
        if parts is not None and len(parts) != n:
            raise ValueError("partition length does not match column count")
        cp = None if coords is None else np.ascontiguousarray(coords, np.float64)
        pp = None if parts is None else np.ascontiguousarray(parts, np.int32)
        dim = 0 if cp is None else cp.shape[1]
        err = C.create_string_buffer(512)
        cl = C.c_int(-1)
        h = C.c_void_p()
        cb = _observer(observer)
        if dist_group is not None:  # spqr_pipeline_create_dist: one factorization across the group's ranks
            if solver != "spaqr" or store_q or observer is not None:
                raise ValueError("a distributed pipeline takes the spaqr solver without store_q / observer")
            import torch.distributed as dist
            rank, size = dist.get_rank(dist_group), dist.get_world_size(dist_group)
            self._tp = _transport(dist_group)
            rc = L.spqr_pipeline_create_dist(m, n, p, i, x, _ptr(cp), dim, _ptr(pp), int(levels), float(eps),
                                             int(skip_levels), int(device), rank, size,
                                             C.cast(self._tp[0], C.c_void_p), C.cast(self._tp[1], C.c_void_p), None,
                                             C.byref(h), err, 512, C.byref(cl))
        else:
            rc = L.spqr_pipeline_create_ex(m, n, p, i, x, _ptr(cp), dim, _ptr(pp), int(levels), float(eps),
                                           int(skip_levels), SOLVERS[solver], int(bool(store_q)), int(ranks),
                                           int(device), C.cast(cb, C.c_void_p) if cb else None, None, C.byref(h),
                                           err, 512, C.byref(cl))
        if rc != 0:
            msg = err.value.decode()
            if rc == 1:
                raise SingularFrontError(cl.value, msg)
            if rc == 2:
                raise ValueError(msg)
            raise RuntimeError(msg)
        self.h = h
        info = np.zeros(16, np.int64)
        L.spqr_pipeline_info(self.h, info)
        (self.M, self.N, self.L, self.nclusters, self.nW, self.ndropped, self.ntrailing, self.nstages, self.nnz_w,
         self.nnz_A, self.nbatches, self.launches, self.syncs, self.h2d_bytes, self.d2h_bytes,
         self.sweep_launches) = [int(v) for v in info]
        self.nQ = int(L.spqr_pipeline_nq(self.h))  # -1: no Q kept
        di = np.zeros(3)
        L.spqr_pipeline_dist_info(self.h, di)
        self.is_root = di[0] == 0.0  # False on ranks > 0 of a distributed factorization
        self.dist_exchange_s, self.dist_bytes = float(di[1]), int(di[2])

    def __del__(self):
        if getattr(self, "h", None):
            lib().spqr_pipeline_destroy(self.h)
            self.h = None

    def times(self):
        t = np.zeros(24)
        lib().spqr_pipeline_times(self.h, t)
        return dict(t_partition=t[0], t_factorize=t[1], t_upload=t[2], qr_ms=t[3], qr_flops=t[4], qr_bytes=t[5],
                    cpqr_flops=t[6], cpqr_bytes=t[7], qr_launches=int(t[8]), factorize_event_ms=t[9],
                    solve_event_ms=t[10], solve_launches=int(t[11]), elim_waves=int(t[12]),
                    cpqr_redundant_bytes=t[13], cpqr_redundant_flops=t[14], sweep_ms=t[15], sweeps=int(t[16]),
                    sweep_bytes=t[17], solve_plan_s=t[18], w_solve_levels=int(t[19]), wt_solve_levels=int(t[20]))

    KERNELS = ("assemble", "stats", "front_qr", "trsm", "cpqr", "scatter")

    def kernel_stats(self):
        ms, by, n = np.zeros(6), np.zeros(6), np.zeros(6, np.int64)
        lib().spqr_pipeline_kernel_stats(self.h, ms, by, n)
        return {k: dict(ms=float(ms[i]), bytes=float(by[i]), launches=int(n[i])) for i, k in enumerate(self.KERNELS)}

    def solve(self, b, tol=-1.0, maxit=-1, direct=False):
        b = np.ascontiguousarray(b, np.float64)
        if b.ndim != 1 or b.shape[0] != self.M:  # pipeline.cpp:71,84
            raise ValueError("right-hand side length mismatch")
        x = np.zeros(self.N)
        hist = np.zeros((maxit if maxit > 0 else 500) + 4)
        it, cv, nh = C.c_int(), C.c_int(), C.c_int()
        ts = C.c_double()
        err = C.create_string_buffer(256)
        rc = lib().spqr_pipeline_solve(self.h, int(direct), b, x, float(tol), int(maxit), C.byref(it), C.byref(cv),
                                       hist, C.byref(nh), C.byref(ts), err, 256)
        if rc:
            raise RuntimeError(err.value.decode())
        return x, dict(iterations=it.value, converged=bool(cv.value), residual_history=hist[: nh.value].copy(),
                       t_solve=ts.value, dropped_rows=self.ndropped)

    def _apply(self, mode, z):
        z = np.array(z, dtype=np.float64, copy=True)
        if z.ndim != 1 or z.shape[0] != (self.M if mode >= 4 else self.N):
            raise ValueError("vector length does not match the factorization")
        if mode >= 4 and self.nQ < 0:
            raise RuntimeError("the factorization holds no Q (create the pipeline with store_q=True)")
        if lib().spqr_pipeline_apply(self.h, mode, z):
            raise RuntimeError("spqr_pipeline_apply failed")
        return z

    def q_apply_t(self, y): return self._apply(4, y)  # transforms.cpp:113-119
    def q_apply(self, y): return self._apply(5, y)    # transforms.cpp:121-127

    def w_apply(self, z): return self._apply(0, z)
    def w_solve(self, z): return self._apply(1, z)
    def wt_apply(self, z): return self._apply(2, z)
    def wt_solve(self, z): return self._apply(3, z)

    def rank_stats(self):
        """Subtree-split accounting of a pipeline created with ranks=G > 1:
        flops[stage, rank], cross[stage, phase] bytes (phases: stack rows, R to holders,
        sparsify_cols holder blocks, merges), owner per cluster."""
        L = lib()
        ns = C.c_int()
        G = L.spqr_pipeline_rank_stats(self.h, C.byref(ns), None, None, None)
        if G <= 1:
            return None
        fl = np.zeros((ns.value, G))
        cr = np.zeros((ns.value, 4))
        ow = np.zeros(self.nclusters, np.int32)
        L.spqr_pipeline_rank_stats(self.h, C.byref(ns), fl.ctypes.data_as(C.c_void_p), cr.ctypes.data_as(C.c_void_p),
                                   ow.ctypes.data_as(C.c_void_p))
        return dict(ranks=G, flops=fl, cross=cr, owner=ow)

    def perm(self):
        o = np.zeros(self.N, np.int32)
        lib().spqr_pipeline_perm(self.h, o)
        return o

    def owner(self):
        o = np.zeros(self.M, np.int32)
        lib().spqr_pipeline_owner(self.h, o)
        return o

    def weights(self):
        o = np.zeros(self.N)
        lib().spqr_pipeline_weights(self.h, o)
        return o

    def rows(self):
        pr = np.zeros(self.N, np.int32)
        dr = np.zeros(max(self.ndropped, 1), np.int32)
        tr = np.zeros(max(self.ntrailing, 1), np.int32)
        lib().spqr_pipeline_rows(self.h, pr, dr, tr)
        return pr, dr[: self.ndropped], tr[: self.ntrailing]

    def clusters(self):
        out = []
        info = np.zeros(6, np.int32)
        for c in range(self.nclusters):
            lib().spqr_pipeline_cluster(self.h, c, info)
            cols = np.zeros(max(int(info[5]), 1), np.int32)
            lib().spqr_pipeline_cluster_cols(self.h, c, cols)
            out.append(dict(tree_node=int(info[0]), level=int(info[1]), parent=int(info[2]), stage=int(info[3]),
                            interior=bool(info[4]), cols=cols[: int(info[5])].copy()))
        return out

    def stages(self):
        out = []
        o = np.zeros(5, np.int64)
        t = np.zeros(5)
        for s in range(self.nstages):
            lib().spqr_pipeline_stage(self.h, s, o, t)
            nf = int(o[1])
            fc = np.zeros(max(nf, 1), np.int32)
            fa = np.zeros(max(nf, 1))
            lib().spqr_pipeline_stage_fronts(self.h, s, fc, fa)
            out.append(dict(stage=int(o[0]), front_cols=fc[:nf].copy(), front_aspect=fa[:nf].copy(),
                            top_rows=int(o[2]), top_cols=int(o[3]), nnz_w=int(o[4]), t_eliminate=t[0],
                            t_reassign=t[1], t_scale=t[2], t_sparsify=t[3], t_merge=t[4]))
        return out

    def save(self, path):
        """save_factorization (transforms.cpp:206-240): SPQRFW01 file of this factorization."""
        err = C.create_string_buffer(512)
        if lib().spqr_pipeline_save(self.h, str(path).encode(), err, 512):
            raise RuntimeError(err.value.decode())

    def scaled(self):
        """Pipeline::scaled() (pipeline.h:62): the column-scaled, permuted A the engine factors."""
        import scipy.sparse as sp
        p = np.zeros(self.N + 1, np.int32)
        i = np.zeros(self.nnz_A, np.int32)
        x = np.zeros(self.nnz_A)
        lib().spqr_pipeline_scaled(self.h, p, i, x)
        return sp.csc_matrix((x, i, p), shape=(self.M, self.N))

    def hierarchy(self):
        """Pipeline::hierarchy() (pipeline.h:59) as the flat description spaqr_factorize takes."""
        nt = lib().spqr_pipeline_tree(self.h, None, None)
        par = np.zeros(nt, np.int32)
        root = C.c_int()
        lib().spqr_pipeline_tree(self.h, par.ctypes.data_as(C.c_void_p), C.byref(root))
        fin = np.zeros(self.N, np.int32)
        lib().spqr_pipeline_finest(self.h, fin)
        return dict(num_levels=self.L, clusters=self.clusters(), finest_of_col=fin, tree_parent=par,
                    tree_root=root.value)

    def wfactors(self):
        out = []
        info = np.zeros(4, np.int32)
        for f in range(self.nW):
            lib().spqr_pipeline_wfactor(self.h, f, info)
            kind, c, d = int(info[0]), int(info[1]), int(info[2])
            cols = np.zeros(max(c, 1), np.int32)
            if kind == 0:
                R = np.zeros(max(c * c, 1))
                cp = np.zeros(max(d, 1), np.int32)
                Cm = np.zeros(max(c * d, 1))
                lib().spqr_pipeline_wfactor_data(self.h, f, cols, R, cp, Cm, np.zeros(1))
                out.append(("tri", cols[:c].copy(), R[: c * c].reshape(c, c, order="F").copy(), cp[:d].copy(),
                            Cm[: c * d].reshape(c, d, order="F").copy()))
            else:
                V = np.zeros(max(c * d, 1))
                tau = np.zeros(max(d, 1))
                sg = np.zeros(max(d, 1))
                lib().spqr_pipeline_wfactor_data(self.h, f, cols, V, np.zeros(1, np.int32), tau, sg)
                out.append(("rot", cols[:c].copy(), V[: c * d].reshape(c, d, order="F").copy(), tau[:d].copy(),
                            sg[:d].copy()))
        return out


def qr_apply_batched(A, n):
    """A: (nb, m, ntot) float64 (each block column-major when viewed as A[b].T.ravel()).
    Returns (A_out, tau, sign, info) with R/V in the first n columns and H^T X after."""
    require_gpu()
    A = np.asarray(A, np.float64)
    nb, m, ntot = A.shape
    buf = np.array(A.transpose(0, 2, 1), dtype=np.float64, order='C', copy=True).ravel()  # column-major per block
    tau = np.zeros(max(nb * n, 1))
    sg = np.zeros(max(nb * n, 1))
    info = np.zeros(max(nb, 1), np.int32)
    rc = lib().spqr_qr_apply_batched(nb, m, n, ntot, buf, tau, sg, info)
    if rc:
        raise RuntimeError(f"spqr_qr_apply_batched failed ({rc})")
    out = buf.reshape(nb, ntot, m).transpose(0, 2, 1).copy()
    return out, tau[: nb * n].reshape(nb, n), sg[: nb * n].reshape(nb, n), info[:nb]


def cpqr_batched(A, eps):
    """A: (nb, m, n).  Returns list of dicts like oracle.cpqr."""
    require_gpu()
    A = np.asarray(A, np.float64)
    nb, m, n = A.shape
    k = max(min(m, n), 1)
    buf = np.array(A.transpose(0, 2, 1), dtype=np.float64, order='C', copy=True).ravel()
    rank = np.zeros(nb, np.int32)
    r11 = np.zeros(nb)
    perm = np.zeros(nb * k, np.int32)
    R = np.zeros(nb * k * max(n, 1))
    V = np.zeros(nb * max(m, 1) * k)
    tau = np.zeros(nb * k)
    sg = np.zeros(nb * k)
    rc = lib().spqr_cpqr_batched(nb, m, n, buf, float(eps), rank, r11, perm, R, V, tau, sg)
    if rc:
        raise RuntimeError(f"spqr_cpqr_batched failed ({rc})")
    out = []
    for b in range(nb):
        r = int(rank[b])
        Rb = R[b * k * n:(b + 1) * k * n].reshape(n, k).T[:r]
        Vb = V[b * m * k:(b + 1) * m * k].reshape(k, m).T[:, :r]
        out.append(dict(rank=r, r11=float(r11[b]), perm=perm[b * k:b * k + r].copy(), R=Rb.copy(), V=Vb.copy(),
                        tau=tau[b * k:b * k + r].copy(), sign=sg[b * k:b * k + r].copy()))
    return out


def trsm_right_batched(B, R):
    """B (nb, nrows, n) <- B R^{-1} with R (nb, n, n) upper triangular."""
    require_gpu()
    B = np.asarray(B, np.float64)
    nb, nrows, n = B.shape
    bb = np.array(B.transpose(0, 2, 1), dtype=np.float64, order='C', copy=True).ravel()
    rr = np.ascontiguousarray(np.asarray(R, np.float64).transpose(0, 2, 1)).ravel()
    rc = lib().spqr_trsm_right_batched(nb, nrows, n, bb, rr)
    if rc:
        raise RuntimeError(f"spqr_trsm_right_batched failed ({rc})")
    return bb.reshape(nb, n, nrows).transpose(0, 2, 1).copy()


class Factorization:
    """spaqr::Factorization (transforms.h:53-72) with W resident on the GPU: made by
    spaqr_factorize or Factorization.load; w_apply / w_solve / wt_apply / wt_solve
    (transforms.h:66-69), save (transforms.h:75)."""

    def __init__(self, handle):
        self.h = handle
        info = np.zeros(8, np.int64)
        lib().spqr_factorization_info(self.h, info)
        (self.M, self.N, self.nW, self.nnz_w, self.ndropped, self.ntrailing, self.nstages,
         self.levels) = [int(v) for v in info]
        self.nQ = int(lib().spqr_factorization_nq(self.h))  # -1: no Q kept

    def __del__(self):
        if getattr(self, "h", None):
            lib().spqr_factorization_destroy(self.h)
            self.h = None

    @classmethod
    def load(cls, path, device=0):
        """load_factorization (transforms.cpp:242-289) straight onto the GPU."""
        require_gpu()
        h = C.c_void_p()
        err = C.create_string_buffer(512)
        rc = lib().spqr_factorization_load(str(path).encode(), int(device), C.byref(h), err, 512)
        if rc:
            raise (ValueError if rc == 2 else RuntimeError)(err.value.decode())
        return cls(h)

    def save(self, path):
        err = C.create_string_buffer(512)
        if lib().spqr_factorization_save(self.h, str(path).encode(), err, 512):
            raise RuntimeError(err.value.decode())

    def rows(self):
        pr = np.zeros(max(self.N, 1), np.int32)
        dr = np.zeros(max(self.ndropped, 1), np.int32)
        tr = np.zeros(max(self.ntrailing, 1), np.int32)
        lib().spqr_factorization_rows(self.h, pr, dr, tr)
        return pr[: self.N], dr[: self.ndropped], tr[: self.ntrailing]

    def stages(self):
        out = []
        o = np.zeros(5, np.int64)
        for s in range(self.nstages):
            lib().spqr_factorization_stage(self.h, s, o)
            fc = np.zeros(max(int(o[1]), 1), np.int32)
            lib().spqr_factorization_stage_fronts(self.h, s, fc)
            out.append(dict(stage=int(o[0]), front_cols=fc[: int(o[1])].copy(), top_rows=int(o[2]),
                            top_cols=int(o[3]), nnz_w=int(o[4])))
        return out

    def _apply(self, mode, z):
        z = np.array(z, dtype=np.float64, copy=True)
        if z.ndim != 1 or z.shape[0] != (self.M if mode >= 4 else self.N):
            raise ValueError("vector length does not match the factorization")
        if mode >= 4 and self.nQ < 0:
            raise RuntimeError("the factorization holds no Q (factorize with store_q=True)")
        if lib().spqr_factorization_apply(self.h, mode, z):
            raise RuntimeError("spqr_factorization_apply failed")
        return z

    def q_apply_t(self, y): return self._apply(4, y)  # transforms.cpp:113-119
    def q_apply(self, y): return self._apply(5, y)    # transforms.cpp:121-127

    def w_apply(self, z): return self._apply(0, z)
    def w_solve(self, z): return self._apply(1, z)
    def wt_apply(self, z): return self._apply(2, z)
    def wt_solve(self, z): return self._apply(3, z)


def spaqr_factorize(A, hierarchy, row_owner, eps=1e-2, skip_levels=3, device=0, observer=None, store_q=False):
    """spaqr_factorize(A, h, row_owner, opt) (factorize.h:51-53) on the GPU.  A: the scaled,
    permuted matrix; hierarchy: the dict Pipeline.hierarchy() returns (clusters with tree_node,
    level, parent, stage, interior, cols; finest_of_col; tree_parent; tree_root; num_levels)."""
    require_gpu()
    m, n, p, i, x = _csc(A)
    owner = np.ascontiguousarray(row_owner, np.int32)
    if owner.shape[0] != m:  # factorize.cpp:800-801
        raise ValueError("row_owner size mismatch")
    cl = hierarchy["clusters"]
    info = np.ascontiguousarray([[c["tree_node"], c["level"], c["parent"], c["stage"], int(c["interior"])]
                                 for c in cl], np.int32).ravel()
    cptr = np.zeros(len(cl) + 1, np.int32)
    cptr[1:] = np.cumsum([len(c["cols"]) for c in cl])
    ccols = np.ascontiguousarray(np.concatenate([np.asarray(c["cols"], np.int32) for c in cl])
                                 if cl else np.zeros(0, np.int32), np.int32)
    if ccols.size == 0:
        ccols = np.zeros(1, np.int32)
    fin = np.ascontiguousarray(hierarchy["finest_of_col"], np.int32)
    tpar = np.ascontiguousarray(hierarchy["tree_parent"], np.int32)
    h = C.c_void_p()
    err = C.create_string_buffer(512)
    ecl = C.c_int(-1)
    cb = _observer(observer)
    rc = lib().spqr_factorize_ex(m, n, p, i, x, int(hierarchy["num_levels"]), len(cl), info, cptr, ccols, fin,
                                 len(tpar), tpar, int(hierarchy["tree_root"]), owner, float(eps), int(skip_levels),
                                 int(bool(store_q)), int(device), C.cast(cb, C.c_void_p) if cb else None, None,
                                 C.byref(h), err, 512, C.byref(ecl))
    if rc:
        msg = err.value.decode()
        if rc == 1:
            raise SingularFrontError(ecl.value, msg)
        if rc == 2:
            raise ValueError(msg)
        raise RuntimeError(msg)
    return Factorization(h)


def cgls(A, W, b, tol=1e-12, maxit=500, weights=None, device=0):
    """cgls(A, W, b, u, opt, weights) (solve.h:30-31) on the GPU: right-preconditioned CGLS on A
    (in W's column coordinates) with W a Factorization or None.  Returns (u, report)."""
    require_gpu()
    m, n, p, i, x = _csc(A)
    b = np.ascontiguousarray(b, np.float64)
    if b.shape[0] != m:
        raise ValueError("right-hand side length mismatch")
    if W is not None and W.N != n:
        raise ValueError("factorization column count does not match A")
    w = None if weights is None else np.ascontiguousarray(weights, np.float64)
    if w is not None and w.shape[0] != n:
        raise ValueError("weights length does not match column count")
    u = np.zeros(n)
    hist = np.zeros(int(maxit if maxit > 0 else 500) + 4)
    it, cv, nh = C.c_int(), C.c_int(), C.c_int()
    ts = C.c_double()
    err = C.create_string_buffer(512)
    rc = lib().spqr_cgls(m, n, p, i, x, None if W is None else W.h, b, u, float(tol), int(maxit), _ptr(w),
                         int(device), C.byref(it), C.byref(cv), hist, C.byref(nh), C.byref(ts), err, 512)
    if rc:
        raise (ValueError if rc == 2 else RuntimeError)(err.value.decode())
    return u, dict(iterations=it.value, converged=bool(cv.value), residual_history=hist[: nh.value].copy(),
                   t_solve=ts.value)


def rank_plan(A, nranks, levels=0, coords=None, parts=None):
    """spqr_rank_plan (include/spaqr_b200.h): the owner rank of every cluster for an
    nranks = 2^g GPU subtree split of the pipeline's partition of A (host only, no GPU)."""
    L = lib()
    m, n, p, i, x = _csc(A)
    cp = None if coords is None else np.ascontiguousarray(coords, np.float64)
    pp = None if parts is None else np.ascontiguousarray(parts, np.int32)
    dim = 0 if cp is None else cp.shape[1]
    ncl, nt = C.c_int(), C.c_int()
    err = C.create_string_buffer(512)
    args = (m, n, p, i, x, _ptr(cp), dim, _ptr(pp), int(levels), int(nranks), C.byref(ncl), C.byref(nt))
    rc = L.spqr_rank_plan(*args, None, None, None, None, None, err, 512)
    if rc:
        raise (ValueError if rc == 2 else RuntimeError)(err.value.decode())
    out = dict(owner=np.zeros(ncl.value, np.int32), cluster_node=np.zeros(ncl.value, np.int32),
               cluster_level=np.zeros(ncl.value, np.int32), tree_parent=np.zeros(nt.value, np.int32),
               tree_level=np.zeros(nt.value, np.int32))
    rc = L.spqr_rank_plan(*args, *[out[k].ctypes.data_as(C.c_void_p) for k in ("owner", "cluster_node", "cluster_level",
                                                                               "tree_parent", "tree_level")], err, 512)
    if rc:
        raise RuntimeError(err.value.decode())
    return out
