"""ctypes loader for libtreetrain_b200.so (the C-ABI in include/treetrain_b200.h).

The product path has no fallback: if the library is missing, every call fails loudly.
"""
import ctypes
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtreetrain_b200.so")
_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        _lib = ctypes.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def _declare(L):
    c = ctypes
    L.tt_last_error.restype = c.c_char_p
    L.tt_debug_gemm.argtypes = [c.c_void_p, c.c_long, c.c_int, c.c_void_p, c.c_long, c.c_int, c.c_int, c.c_int,
                                c.c_int, c.c_int, c.c_void_p, c.c_void_p, c.c_void_p, c.c_long, c.c_int, c.c_void_p,
                                c.c_void_p, c.c_int]
