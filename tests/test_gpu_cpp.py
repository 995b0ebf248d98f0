"""GPU: the C++ drop-in layer (include/dso/batch.hpp) against the reference's own
brute_force_config, through tests/cpp/test_batch (built by __graft_entry__.build()
where the reference headers exist; the binary travels to the GPU box)."""

import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "tests", "cpp", "test_batch")


def test_cpp_batch_layer():
    assert os.path.exists(BIN), "tests/cpp/test_batch not built (run __graft_entry__.build())"
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=300)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
