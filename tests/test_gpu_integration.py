"""The C++ drop-in: the reference's own objects and libfsgg.so in one binary
(oracle/ref/adapter_check.cpp via include/fsgg/fsg_adapter.hpp), comparing
fsg::build_similarity_graph (CPU, exact) with the adapter (GPU)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "oracle", "_ref", "adapter_check")

pytestmark = pytest.mark.gpu


def test_cpp_adapter_matches_reference_binary():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/adapter_check not built (needs /root/reference at build time)")
    out = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(out.stdout, out.stderr)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "adapter ok" in out.stdout
