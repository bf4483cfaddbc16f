"""ctypes binding of libspaqr_b200.so (the C ABI declared in include/spaqr_b200.h).

The product path has no CPU fallback: if the CUDA library is missing this
raises, and every compute entry point needs a visible B200.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libspaqr_b200.so")
_lib = None

i32p = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")
f64p = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
i64p = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
vp = C.c_void_p

# every symbol include/spaqr_b200.h declares -> (restype, argtypes)
SIGNATURES = {
    "spqr_version": (C.c_char_p, []),
    "spqr_device_count": (C.c_int, []),
    "spqr_pipeline_create": (C.c_int, [C.c_int, C.c_int, i32p, i32p, f64p, vp, C.c_int, vp, C.c_int, C.c_double,
                                       C.c_int, C.c_int, C.c_int, C.POINTER(vp), C.c_char_p, C.c_int,
                                       C.POINTER(C.c_int)]),
    "spqr_pipeline_destroy": (None, [vp]),
    "spqr_pipeline_info": (None, [vp, i64p]),
    "spqr_pipeline_times": (None, [vp, f64p]),
    "spqr_pipeline_kernel_stats": (None, [vp, f64p, f64p, i64p]),
    "spqr_pipeline_solve": (C.c_int, [vp, C.c_int, f64p, f64p, C.c_double, C.c_int, C.POINTER(C.c_int),
                                      C.POINTER(C.c_int), f64p, C.POINTER(C.c_int), C.POINTER(C.c_double),
                                      C.c_char_p, C.c_int]),
    "spqr_pipeline_apply": (C.c_int, [vp, C.c_int, f64p]),
    "spqr_pipeline_perm": (None, [vp, i32p]),
    "spqr_pipeline_owner": (None, [vp, i32p]),
    "spqr_pipeline_weights": (None, [vp, f64p]),
    "spqr_pipeline_rows": (None, [vp, i32p, i32p, i32p]),
    "spqr_pipeline_cluster": (None, [vp, C.c_int, i32p]),
    "spqr_pipeline_cluster_cols": (None, [vp, C.c_int, i32p]),
    "spqr_pipeline_stage": (None, [vp, C.c_int, i64p, f64p]),
    "spqr_pipeline_stage_fronts": (None, [vp, C.c_int, i32p, f64p]),
    "spqr_pipeline_wfactor": (None, [vp, C.c_int, i32p]),
    "spqr_pipeline_wfactor_data": (C.c_int, [vp, C.c_int, i32p, f64p, i32p, f64p, f64p]),
    "spqr_pipeline_save": (C.c_int, [vp, C.c_char_p, C.c_char_p, C.c_int]),
    "spqr_pipeline_tree": (C.c_int, [vp, vp, vp]),
    "spqr_pipeline_finest": (None, [vp, i32p]),
    "spqr_pipeline_scaled": (None, [vp, i32p, i32p, f64p]),
    "spqr_factorize": (C.c_int, [C.c_int, C.c_int, i32p, i32p, f64p, C.c_int, C.c_int, i32p, i32p, i32p, i32p,
                                 C.c_int, i32p, C.c_int, i32p, C.c_double, C.c_int, C.c_int, vp, vp,
                                 C.POINTER(vp), C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
    "spqr_pipeline_create_observed": (C.c_int, [C.c_int, C.c_int, i32p, i32p, f64p, vp, C.c_int, vp, C.c_int,
                                                C.c_double, C.c_int, C.c_int, C.c_int, vp, vp, C.POINTER(vp),
                                                C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
    "spqr_factorize_ex": (C.c_int, [C.c_int, C.c_int, i32p, i32p, f64p, C.c_int, C.c_int, i32p, i32p, i32p, i32p,
                                    C.c_int, i32p, C.c_int, i32p, C.c_double, C.c_int, C.c_int, C.c_int, vp, vp,
                                    C.POINTER(vp), C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
    "spqr_pipeline_create_ex": (C.c_int, [C.c_int, C.c_int, i32p, i32p, f64p, vp, C.c_int, vp, C.c_int,
                                          C.c_double, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, vp, vp,
                                          C.POINTER(vp), C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
    "spqr_pipeline_rank_stats": (C.c_int, [vp, C.POINTER(C.c_int), vp, vp, vp]),
    "spqr_pipeline_create_dist": (C.c_int, [C.c_int, C.c_int, i32p, i32p, f64p, vp, C.c_int, vp, C.c_int, C.c_double,
                                            C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, C.POINTER(vp),
                                            C.c_char_p, C.c_int, C.POINTER(C.c_int)]),
    "spqr_pipeline_dist_info": (None, [vp, f64p]),
    "spqr_rank_plan": (C.c_int, [C.c_int, C.c_int, i32p, i32p, f64p, vp, C.c_int, vp, C.c_int, C.c_int,
                                 C.POINTER(C.c_int), C.POINTER(C.c_int), vp, vp, vp, vp, vp, C.c_char_p, C.c_int]),
    "spqr_pipeline_nq": (C.c_longlong, [vp]),
    "spqr_factorization_nq": (C.c_longlong, [vp]),
    "spqr_factorization_destroy": (None, [vp]),
    "spqr_factorization_info": (None, [vp, i64p]),
    "spqr_factorization_rows": (None, [vp, i32p, i32p, i32p]),
    "spqr_factorization_stage": (C.c_int, [vp, C.c_int, i64p]),
    "spqr_factorization_stage_fronts": (C.c_int, [vp, C.c_int, i32p]),
    "spqr_factorization_apply": (C.c_int, [vp, C.c_int, f64p]),
    "spqr_factorization_save": (C.c_int, [vp, C.c_char_p, C.c_char_p, C.c_int]),
    "spqr_factorization_load": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(vp), C.c_char_p, C.c_int]),
    "spqr_cgls": (C.c_int, [C.c_int, C.c_int, i32p, i32p, f64p, vp, f64p, f64p, C.c_double, C.c_int, vp, C.c_int,
                            C.POINTER(C.c_int), C.POINTER(C.c_int), f64p, C.POINTER(C.c_int),
                            C.POINTER(C.c_double), C.c_char_p, C.c_int]),
    "spqr_qr_apply_batched": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, f64p, f64p, f64p, i32p]),
    "spqr_qr_apply_batched_dev": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_int, vp, vp, vp, vp,
                                            C.POINTER(C.c_float)]),
    "spqr_cpqr_batched_dev": (C.c_int, [C.c_int, C.c_int, C.c_int, vp, C.c_double, vp, C.POINTER(C.c_float)]),
    "spqr_cpqr_batched": (C.c_int, [C.c_int, C.c_int, C.c_int, f64p, C.c_double, i32p, f64p, i32p, f64p, f64p,
                                    f64p, f64p]),
    "spqr_trsm_right_batched": (C.c_int, [C.c_int, C.c_int, C.c_int, f64p, f64p]),
}


def build():
    subprocess.run(["make", "-s", "-j8", "-C", _HERE], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"spaqr_b200: CUDA library {LIB_PATH} is missing (run __graft_entry__.build()); "
                               "there is no CPU fallback")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def require_gpu():
    n = lib().spqr_device_count()
    if n <= 0:
        raise RuntimeError("spaqr_b200: no CUDA device visible; the product path runs only on the GPU")
    return n
