"""spaqr_b200 — B200-native (sm_100a) implementation of the spaQR hot path.

Mirrors the reference's API (proj/include/spaqr): Pipeline (factorize + CGLS /
CSNE), Factorization sweeps, and the batched dense kernels.  All FP64 front
work and the W sweeps run on the GPU through libspaqr_b200.so (C ABI in
include/spaqr_b200.h); partitioning is host C++ inside the same library.
"""
from .api import (Factorization, Pipeline, SingularFrontError, cgls, cpqr_batched, qr_apply_batched,  # noqa: F401
                  rank_plan, spaqr_factorize, trsm_right_batched)
from ._lib import LIB_PATH, build, lib, require_gpu  # noqa: F401
from .profile import make_profile, validate_profile  # noqa: F401
