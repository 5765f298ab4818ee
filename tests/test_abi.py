"""The C-ABI library loads without a GPU and exports every entry point include/*.h declares."""
import ctypes
import os
import re

from paper_2602_00482_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    names = set()
    inc = os.path.join(ROOT, "include")
    for f in os.listdir(inc):
        if f.endswith(".h"):
            src = open(os.path.join(inc, f)).read()
            names |= set(re.findall(r"^\s*(?:int|const char\*)\s+(tt_\w+)\s*\(", src, re.M))
    return names


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(_native.LIB_PATH)
    names = declared_symbols()
    assert len(names) >= 25
    missing = [n for n in sorted(names) if not hasattr(lib, n)]
    assert not missing, missing


def test_python_binding_covers_header():
    assert declared_symbols() <= set(_native.EXPORTS)


def test_error_reporting_without_gpu():
    import paper_2602_00482_b200 as tt

    cfg = tt.ModelConfig(64, 32, 4, 2, 64, 128)
    assert cfg.param_count() == 64 * 32 * 2 + 2 * (2 * 32 + 4 * 32 * 32 + 2 * 32 * 64) + 32
    bad = tt.ModelConfig(64, 30, 4, 2, 64, 128)  # d_model not divisible by n_heads
    try:
        tt.Engine(bad)
        raised = None
    except (ValueError, RuntimeError) as e:
        raised = e
    assert raised is not None
