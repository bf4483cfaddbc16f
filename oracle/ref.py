"""ORACLE — TEST INFRASTRUCTURE ONLY.

The spaQR reference itself, as a checker: /root/reference/proj/src/*.cpp compiled
UNMODIFIED against the in-repo Eigen API shim (oracle/eigen_shim/) into
oracle/_ref/libspaqr_ref.so by oracle/Makefile.ref, exposed through the same orc_*
C ABI and the same Python front-end as the restatement.  Usage mirrors `oracle`:

    from oracle import ref
    if ref.available():
        p = ref.Pipeline(A, eps=1e-2, levels=8, coords=xy)

The .so is built where /root/reference exists (this container: __graft_entry__.build())
and travels to the GPU box as a prebuilt, git-ignored file.
"""
import importlib.util
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
PATH = os.path.join(_HERE, "_ref", "libspaqr_ref.so")


def available():
    return os.path.exists(PATH) or os.path.isdir("/root/reference/proj/src")


def _load():
    spec = importlib.util.spec_from_file_location("oracle._ref_frontend", os.path.join(_HERE, "__init__.py"))
    mod = importlib.util.module_from_spec(spec)
    mod.__dict__["_LIB_OVERRIDE"] = PATH
    mod.__dict__["_MAKEFILE_OVERRIDE"] = "Makefile.ref"
    spec.loader.exec_module(mod)
    return mod


_mod = _load()
globals().update({k: v for k, v in _mod.__dict__.items() if not k.startswith("__") and k not in ("_HERE",)})
