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


MLP_BIN = os.path.join(ROOT, "tests", "cpp", "test_mlp_batch")


def test_cpp_mlp_batch_layer():
    """include/dso/batch_mlp.hpp (predict_params / forward_raw / featurize / as_vector /
    load_dcgm_samples / analytic_gradients / mse_loss / fit_model / cross_validate /
    train, incl. a one-rank NCCL data-parallel run) against the C restatement."""
    assert os.path.exists(MLP_BIN), "tests/cpp/test_mlp_batch not built (run __graft_entry__.build())"
    r = subprocess.run([MLP_BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "PASS" in r.stdout
