"""GPU parity: predictor inference (predict_params / forward_raw) vs the oracle.

FP32 on the device against the reference's double MLP.  Tolerance (written
here): |gpu - ref| <= 1e-5 * |ref| + 1e-6 * target_std — i.e.
1e-5 relative, with an absolute floor of a millionth of the target's spread for
outputs that cross zero (a pure relative bound is ill-posed there).  The clamp
flag must agree except where the raw output is within that tolerance of 0."""

import types

import numpy as np
import pytest
import torch

from paper_2407_13096_b200 import init_mlp, MlpModel

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("engine")]


def fused_dev(x):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(x, np.float32).T)).cuda()


def stats_model(port, seed=424242, n=4096):
    """Golden-initialised net with target stats of the synthetic truth params, so the
    outputs live on the scale of real DVFS parameters."""
    m = init_mlp(seed=seed)
    params = port.gen_stream(0xC0FFEE, n, want=("params",))["params"]
    mean, std, _ = port.target_stats(params)
    m.target_mean, m.target_std = mean, std
    return m


def check_params(got, want, std):
    tol = 1e-5 * np.abs(want) + 1e-6 * std[None, :]
    err = np.abs(got - want)
    assert (err <= tol).all(), f"worst {np.max(err / tol):.3f} x tolerance"


def test_golden_forward(ctx, golden_json):
    g = golden_json("mlp_forward_golden.json")
    m = init_mlp(g["layer_sizes"], g["seed"])
    ctx.set_model(m)
    x = np.array([[(i % 13) / 13.0 for i in range(134)]])
    params, clamped, raw = ctx.predict_params(fused_dev(x), want_raw=True)
    raw = raw.cpu().numpy()[:, 0]
    want = np.array(g["outputs"])
    assert np.all(np.abs(raw - want) <= 1e-5 * np.abs(want) + 1e-6)


def test_predict_vs_oracle(ctx, port):
    m = stats_model(port)
    ctx.set_model(m)
    n = 65_536 + 77
    fused = port.gen_stream(0xD50B201, n, want=("fused",))["fused"]
    rng = np.random.default_rng(1)
    fused[: n // 4] = rng.uniform(0, 1, size=(n // 4, 134))   # off-distribution inputs too
    p, cl, raw = ctx.predict_params(fused_dev(fused), want_raw=True)
    want_raw = port.forward_raw(m, fused.astype(np.float32).astype(np.float64))
    want_p, want_cl = port.predict_params(m, fused.astype(np.float32).astype(np.float64))
    check_params(raw.cpu().numpy().T, want_raw, m.target_std)
    check_params(p.cpu().numpy().T, want_p, m.target_std)
    cl = cl.cpu().numpy()
    near0 = (np.abs(want_raw) <= 1e-5 * np.abs(want_raw) + 1e-6 * m.target_std).any(1)
    assert ((cl == want_cl) | near0).all()


def test_constant_net_and_clamp(ctx, port):
    """test_mlp.cpp:41-54 (constant net reproduces the means) and :228-241 (clamp)."""
    m = init_mlp(seed=1)
    m.weights = [np.zeros_like(w) for w in m.weights]
    m.biases = [np.zeros_like(b) for b in m.biases]
    m.target_mean = np.array([10, 5, 2, 3, 1, 8, 6], float)
    ctx.set_model(m)
    for t in range(3):
        p, cl, _ = ctx.predict_params(fused_dev(np.full((5, 134), 0.1 * t)))
        np.testing.assert_array_equal(p.cpu().numpy().T, np.tile(m.target_mean, (5, 1)))
        assert not cl.cpu().numpy().any()
    m = init_mlp(seed=6)
    m.target_mean = np.full(7, -100.0)
    ctx.set_model(m)
    p, cl, _ = ctx.predict_params(fused_dev(np.zeros((3, 134))))
    p = p.cpu().numpy().T
    assert cl.cpu().numpy().all()
    assert (p[:, :6] == 0).all() and np.all(p[:, 6] == np.float32(1e-12))


def test_set_model_validation(ctx):
    from paper_2407_13096_b200 import DsoError, ErrorKind
    m = init_mlp(seed=3)
    m.target_std = np.zeros(7)
    with pytest.raises(DsoError) as e:
        ctx.set_model(m)
    assert e.value.kind == ErrorKind.InvalidModel
    # any chain within the generic engine's limits is accepted (mlp_gen.cu) ...
    ctx.set_model(init_mlp([4, 3, 2], seed=1))
    assert ctx.n_model_params == 4 * 3 + 3 * 2 + 3 + 2
    # ... wider chains are not
    with pytest.raises(DsoError) as e:
        ctx.set_model(init_mlp([4, 300, 2], seed=1))
    assert e.value.kind == ErrorKind.InvalidModel
