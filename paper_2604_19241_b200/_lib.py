"""Loader for libeplab_b200.so (the in-tree CUDA library). There is no fallback:
if the library or a CUDA device is missing, every data-path call fails loudly."""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("EPLAB_LIB") or os.path.join(_HERE, "libeplab_b200.so")  # EPLAB_LIB: A/B experiments
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"libeplab_b200.so not built at {LIB_PATH}; run __graft_entry__.build()")
        _lib = ctypes.CDLL(LIB_PATH)
    return _lib
