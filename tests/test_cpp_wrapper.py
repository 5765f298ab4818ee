"""The header-only C++ wrapper (include/treetrain_b200.hpp) compiles, links against the C-ABI
library and mirrors the reference's results and exception types (no GPU needed)."""
import os
import subprocess

import pytest

from oracle import treetrain_oracle as O
from paper_2602_00482_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_cpp_wrapper_tree_and_partition(tmp_path):
    exe = str(tmp_path / "demo")
    libdir = os.path.dirname(_native.LIB_PATH)
    r = subprocess.run(["g++", "-std=c++17", "-O1", "-I", os.path.join(ROOT, "include"),
                        os.path.join(ROOT, "tests", "cpp", "wrapper_demo.cpp"), "-L", libdir, "-ltreetrain_b200",
                        f"-Wl,-rpath,{libdir}", "-o", exe], capture_output=True, text=True)
    if r.returncode != 0:
        pytest.fail(r.stderr)
    out = subprocess.run([exe], capture_output=True, text=True, check=True).stdout
    seqs = [O.TokenSequence(i, t, [1.0] * len(t)) for i, t in enumerate([[1, 2, 3], [1, 2, 4], [1, 2], [7, 7, 7, 7]])]
    root = O.order_children(O.build_prefix_tree(seqs), "subtree_tokens_desc")
    expect = f"TOKENS {O.tree_token_count(root)}\n" + O.serialize_tree(root) + O.dfs_trace(root)
    assert out.startswith(expect)
    assert f"MAXCOST {O.partition_contiguous(seqs, 2).max_cost}" in out
    assert "INVALID_ARGUMENT" in out
