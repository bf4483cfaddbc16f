"""CPU checks of the boundary: the CUDA C-ABI library loads without a GPU and
exports every symbol include/spaqr_b200.h declares; the Python binding
declares a signature for each; compute entry points refuse to run without a
device (no CPU fallback)."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_symbols():
    txt = open(os.path.join(ROOT, "include", "spaqr_b200.h")).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(spqr_[a-z0-9_]+)\s*\(", txt)))


def test_library_exports_every_header_symbol():
    import paper_2102_09878_b200 as P
    lib = ctypes.CDLL(P.LIB_PATH)
    syms = header_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_declares_every_symbol():
    from paper_2102_09878_b200._lib import SIGNATURES
    assert set(header_symbols()) == set(SIGNATURES)


def test_no_cpu_fallback():
    import paper_2102_09878_b200 as P
    if P.lib().spqr_device_count() > 0:
        pytest.skip("a GPU is visible")
    import scipy.sparse as sp
    with pytest.raises(RuntimeError):
        P.Pipeline(sp.identity(4, format="csc"), eps=0.0, levels=1)


def test_partition_levels_default_matches_reference_table():
    import oracle as O
    for n, L in [(1, 1), (64, 1), (65, 1), (128, 1), (129, 2), (256, 2), (257, 3), (4096, 6)]:
        assert O.default_num_levels(n) == L
