"""GPU parity: predictor training step vs the oracle (analytic_gradients, mse_loss,
sgd update — reference proj/src/mlp.cpp:84-112, 259-289).

FP32 on the device vs double in the oracle.  Tolerances:
per-layer max |g_gpu - g_ref| <= 2e-5 * max|g_ref| (entries summed over the
batch in FP32 per CTA, then in double across CTAs); loss within 1e-5
relative; 20 SGD steps leave the weights within 1e-4 relative (max-norm)."""

import numpy as np
import pytest
import torch

from paper_2407_13096_b200 import init_mlp
from paper_2407_13096_b200.train import DataParallelTrainer, target_stats

pytestmark = pytest.mark.gpu


def batch(port, n, root=0xACCE5505):
    g = port.gen_stream(root, n, want=("params", "fused"))
    mean, std, _ = target_stats(g["params"])
    y = (g["params"] - mean) / std
    return g["fused"], y, mean, std


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.float32).T)).cuda()


def f32model(m):
    """The model the device actually holds (weights rounded to float)."""
    m2 = m.copy()
    m2.weights = [w.astype(np.float32).astype(np.float64) for w in m.weights]
    m2.biases = [b.astype(np.float32).astype(np.float64) for b in m.biases]
    return m2


@pytest.mark.parametrize("n", [1, 63, 64, 1000, 20_000])
def test_gradient_vs_oracle(ctx, port, n):
    x, y, mean, std = batch(port, n)
    m = init_mlp(seed=424242)
    m.target_mean, m.target_std = mean, std
    ctx.set_model(m)
    grad, loss = ctx.train_grad(dev(x), dev(y))
    grad = grad.cpu().numpy().astype(np.float64) / (n * 7)
    x32 = x.astype(np.float32).astype(np.float64)
    y32 = y.astype(np.float32).astype(np.float64)
    mr = f32model(m)
    gw, gb = port.analytic_gradients(mr, x32, y32)
    off = 0
    for w in gw:
        got = grad[off:off + w.size].reshape(w.shape)
        off += w.size
        assert np.abs(got - w).max() <= 2e-5 * np.abs(w).max() + 1e-12
    for b in gb:
        got = grad[off:off + b.size]
        off += b.size
        assert np.abs(got - b).max() <= 2e-5 * np.abs(b).max() + 1e-12
    want_loss = port.mse_loss(mr, x32, y32)
    assert float(loss.item()) / (n * 7) == pytest.approx(want_loss, rel=1e-5)


def test_sgd_trajectory_vs_oracle(ctx, port):
    """20 steps of W -= lr * g on fixed batches (batch 256) vs the oracle in double."""
    n, B, lr = 256 * 20, 256, 0.3
    x, y, mean, std = batch(port, n, root=77)
    m = init_mlp(seed=5)
    m.target_mean, m.target_std = mean, std
    ctx.set_model(m)
    tr = DataParallelTrainer(ctx, lr=lr)
    ref = f32model(m)
    for s in range(20):
        xs, ys = x[s * B:(s + 1) * B], y[s * B:(s + 1) * B]
        loss = tr.step(dev(xs), dev(ys), B, B)
        x32 = xs.astype(np.float32).astype(np.float64)
        y32 = ys.astype(np.float32).astype(np.float64)
        want = port.mse_loss(ref, x32, y32)
        assert float(loss.item()) == pytest.approx(want, rel=1e-4)
        gw, gb = port.analytic_gradients(ref, x32, y32)
        ref.weights = [w - lr * g for w, g in zip(ref.weights, gw)]
        ref.biases = [b - lr * g for b, g in zip(ref.biases, gb)]
    got = ctx.get_model()
    for a, b in zip(got.weights + got.biases, ref.weights + ref.biases):
        assert np.abs(a - b).max() <= 1e-4 * np.abs(b).max()
    # the inference kernels see the trained weights (device repack)
    p, cl, raw = ctx.predict_params(dev(x[:500]), want_raw=True)
    want_raw = port.forward_raw(got, x[:500].astype(np.float32).astype(np.float64))
    assert np.abs(raw.cpu().numpy().T - want_raw).max() <= 1e-5 * np.abs(want_raw).max()


def test_training_reduces_loss(ctx, port):
    """SGD on 50k synthetic kernels at a GPU batch size: epoch losses must be
    non-increasing (test_mlp.cpp:174-193 analogue; large batches converge slowly,
    so only the trend is asserted, as in the reference test)."""
    n, B = 50_000, 1024
    x, y, mean, std = batch(port, n, root=99)
    m = init_mlp(seed=3)
    m.target_mean, m.target_std = mean, std
    ctx.set_model(m)
    tr = DataParallelTrainer(ctx, lr=0.5)
    X, Y = dev(x), dev(y)
    losses = []
    for epoch in range(6):
        tot = 0.0
        for s in range(0, n, B):
            b = min(B, n - s)
            tot += float(tr.step(X[:, s:s + b].contiguous(), Y[:, s:s + b].contiguous(), b, b))
        losses.append(tot)
    assert all(b <= a * (1 + 1e-9) for a, b in zip(losses, losses[1:])), losses
    assert losses[-1] < 0.99 * losses[0], losses


# ---- orchestration: fit_model / cross_validate / train (mlp.cpp:115-130, 348-437) ----

def _oracle_fit(port, feats, targets, sizes, mean, std, lr, batch, epochs, seed):
    """fit_model restated on the double oracle (sgd_epoch, init_mlp)."""
    from paper_2407_13096_b200.train import fork
    ws, bs = port.init_mlp(sizes, seed)
    m = init_mlp(list(sizes), seed=seed)
    m.weights, m.biases = ws, bs
    m.target_mean, m.target_std = mean, std
    state = fork(seed, 0x5D0)
    trace = []
    for _ in range(epochs):
        loss, m.weights, m.biases, state = port.sgd_epoch(m, feats, targets, mean, std, lr,
                                                          batch, state)
        trace.append(loss)
        if np.isnan(loss):
            break
    return m, trace


def _corpus(port, n, root):
    g = port.gen_stream(root, n, want=("params", "fused"))
    return g["fused"], g["params"]


def test_fit_model_vs_oracle(ctx, port):
    from paper_2407_13096_b200.train import canonicalize, fit_model, target_stats as ts
    f, t = canonicalize(*_corpus(port, 40, 0xACCE5505))
    sizes = [134, 100, 50, 25, 7]
    mean, std, _ = ts(t)
    got, trace = fit_model(ctx, f, t, sizes, mean, std, 0.05, 8, 6, 1234)
    want, wtrace = _oracle_fit(port, f, t, sizes, mean, std, 0.05, 8, 6, 1234)
    assert len(trace) == len(wtrace) == 6
    np.testing.assert_allclose(trace, wtrace, rtol=2e-4)
    for a, b in zip(got.weights + got.biases, want.weights + want.biases):
        assert np.abs(a - b).max() <= 2e-4 * np.abs(b).max()


def test_cross_validate_and_train_vs_oracle(ctx, port):
    """3 folds x 2 cells: per-fold validation MAPEs within 1e-3 relative of the
    double oracle's, the same winning cell, and the final model's trace."""
    from paper_2407_13096_b200.train import (canonicalize, cross_validate, fork,
                                             shuffled_order, target_stats as ts, train)
    f0, t0 = _corpus(port, 30, 0xACCE5506)
    grid = [(0.05, 8), (0.02, 16)]
    seed, epochs = 99, 8
    cv = cross_validate(ctx, f0, t0, grid, seed, epochs)
    f, t = canonicalize(f0, t0)
    order, _ = shuffled_order(len(f), fork(seed, 0xF01D))
    fold_of = np.empty(len(f), np.int64)
    fold_of[order] = np.arange(len(f)) % 3
    sizes = [134, 100, 50, 25, 7]
    for ci, (lr, bs) in enumerate(grid):
        for fold in range(3):
            tr, va = fold_of != fold, fold_of == fold
            mean, std, _ = ts(t[tr])
            m, _ = _oracle_fit(port, f[tr], t[tr], sizes, mean, std, lr, bs, epochs,
                               seed + 1000003 * fold + 29 * ci)
            pred = port.forward_raw(m, f[va])
            mape = 100 * np.mean(np.abs(pred - t[va]) / np.maximum(np.abs(t[va]), 1e-9))
            assert cv["table"][ci][2][fold] == pytest.approx(mape, rel=1e-3)
    means = [row[3] for row in cv["table"]]
    assert cv["best"] == grid[int(np.argmin(means))]
    res = train(ctx, f0, t0, grid, seed, epochs)
    assert res["cv"]["best"] == cv["best"]
    assert len(res["epoch_loss"]) == epochs


def test_train_errors(ctx):
    from paper_2407_13096_b200 import DsoError, ErrorKind
    from paper_2407_13096_b200.train import cross_validate, train
    f, t = np.random.rand(2, 134), np.random.rand(2, 7)
    with pytest.raises(DsoError) as e:
        train(ctx, f, t, [(0.1, 8)], 1, 1)
    assert e.value.kind == ErrorKind.DatasetTooSmall
    f, t = np.random.rand(5, 134), np.random.rand(5, 7)
    t[2, 3] = np.nan
    with pytest.raises(DsoError) as e:
        train(ctx, f, t, [(0.1, 8)], 1, 1)
    assert e.value.kind == ErrorKind.InvalidArgument
    with pytest.raises(DsoError) as e:
        cross_validate(ctx, np.random.rand(5, 134), np.random.rand(5, 7), [], 1, 1)
    assert e.value.kind == ErrorKind.InvalidArgument


def test_fit_model_restores_context_stream(ctx, port):
    """fit_model captures its epochs on a side stream; the context must be back on
    the caller's stream afterwards (later launches race with torch otherwise)."""
    import ctypes as C
    from paper_2407_13096_b200.train import canonicalize, fit_model, target_stats as ts
    f, t = canonicalize(*_corpus(port, 20, 0xACCE5505))
    mean, std, _ = ts(t)
    fit_model(ctx, f, t, [134, 100, 50, 25, 7], mean, std, 0.05, 8, 4, 3)
    x = torch.from_numpy(np.random.default_rng(0).uniform(size=(134, 4096)).astype(np.float32)).cuda()
    for _ in range(3):
        p1, _, _ = ctx.predict_params(x)
        a = p1.cpu().numpy()
        p2, _, _ = ctx.predict_params(x)
        np.testing.assert_array_equal(a, p2.cpu().numpy())
