"""Non-default layer chains on the device (TrainConfig.layer_sizes, mlp.hpp:87-89;
init_mlp / validate accept any chain, mlp.cpp:184-226) and the 64-bit-count
feature stage (KernelInstructionCounts are std::uint64_t, ptx_features.hpp:31-37).

The reference's own gradient checks use the probe net {4, 3, 3, 3, 2}
(test_mlp.cpp:79-113, acceptance AC4); here the device gradient of such chains
is compared with the oracle's analytic gradient (itself pinned to central finite
differences in tests/test_oracle.py) and with the oracle's finite differences."""

import numpy as np
import pytest
import torch

from helpers import check_index_rule
from paper_2407_13096_b200 import DsoError, ErrorKind, config_domain, init_mlp
from paper_2407_13096_b200.train import fit_model, fork, train

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.float32).T)).cuda()


def f32model(m):
    m2 = m.copy()
    m2.weights = [w.astype(np.float32).astype(np.float64) for w in m.weights]
    m2.biases = [b.astype(np.float32).astype(np.float64) for b in m.biases]
    return m2


def chain_model(sizes, seed):
    m = init_mlp(list(sizes), seed=seed)
    m.target_mean = np.linspace(0.5, 2.0, sizes[-1])
    m.target_std = np.linspace(1.0, 3.0, sizes[-1])
    return m


@pytest.mark.parametrize("sizes", [[4, 3, 3, 3, 2], [134, 7], [134, 64, 32, 7], [10, 256, 5]])
@pytest.mark.parametrize("n", [1, 65, 3000])
def test_generic_gradient_vs_oracle(ctx, port, sizes, n):
    rng = np.random.default_rng(n + len(sizes))
    x = rng.uniform(0, 1, (n, sizes[0]))
    y = rng.normal(0, 1, (n, sizes[-1]))
    m = chain_model(sizes, seed=17 + n)
    ctx.set_model(m)
    grad, loss = ctx.train_grad(dev(x), dev(y))
    grad = grad.cpu().numpy().astype(np.float64) / (n * sizes[-1])
    x32, y32 = x.astype(np.float32).astype(np.float64), y.astype(np.float32).astype(np.float64)
    mr = f32model(m)
    gw, gb = port.analytic_gradients(mr, x32, y32)
    off = 0
    for want in list(gw) + list(gb):
        got = grad[off:off + want.size].reshape(want.shape)
        off += want.size
        assert np.abs(got - want).max() <= 2e-5 * np.abs(want).max() + 1e-12
    assert off == grad.size == ctx.n_model_params
    assert float(loss.item()) / (n * sizes[-1]) == pytest.approx(port.mse_loss(mr, x32, y32),
                                                                  rel=1e-5)


def test_probe_net_vs_finite_differences(ctx, port):
    """AC4 shape: {4,3,3,3,2} on one sample, device gradient vs central differences."""
    rng = np.random.default_rng(4)
    x, y = rng.uniform(0, 1, (1, 4)), rng.normal(0, 1, (1, 2))
    m = chain_model([4, 3, 3, 3, 2], seed=99)
    ctx.set_model(m)
    grad, _ = ctx.train_grad(dev(x), dev(y))
    grad = grad.cpu().numpy().astype(np.float64) / 2
    nw, nb = port.numeric_gradients(f32model(m), x.astype(np.float32).astype(np.float64),
                                    y.astype(np.float32).astype(np.float64), 1e-6)
    want = np.concatenate([a.ravel() for a in list(nw) + list(nb)])
    assert np.abs(grad - want).max() <= 1e-5 * max(np.abs(want).max(), 1e-3)


@pytest.mark.parametrize("sizes", [[134, 7], [134, 64, 32, 7], [8, 16, 3]])
def test_generic_forward_and_predict(ctx, port, sizes):
    rng = np.random.default_rng(sum(sizes))
    n = 5003
    x = rng.uniform(0, 1, (n, sizes[0]))
    m = chain_model(sizes, seed=5)
    m.target_mean = np.abs(m.target_mean)
    ctx.set_model(m)
    params, clamped, raw = ctx.predict_params(dev(x), want_raw=True)
    raw = raw.cpu().numpy().T.astype(np.float64)
    want = port.forward_raw(f32model(m), x.astype(np.float32).astype(np.float64))
    scale = np.asarray(m.target_std)[None, :]
    assert (np.abs(raw - want) <= 1e-5 * np.abs(want) + 1e-6 * scale).all()
    if sizes[-1] == 7:
        wp, wc = port.predict_params(f32model(m), x.astype(np.float32).astype(np.float64))
        p = params.cpu().numpy().T.astype(np.float64)
        assert (np.abs(p - wp) <= 1e-5 * np.abs(wp) + 1e-6 * scale).all()
        assert (clamped.cpu().numpy() == wc).mean() >= 0.999
    else:
        assert params is None and clamped is None


@pytest.mark.parametrize("csr", [False, True])
def test_generic_pipeline_vs_oracle(ctx, port, csr):
    """A 134-64-32-7 predictor through dso_pipeline / dso_pipeline_csr (staged on
    the generic engine) vs the oracle pipeline, under the index rule."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    m = init_mlp([134, 64, 32, 7], seed=31)
    p = port.gen_stream(0xC0FFEE, 4096, want=("params",))["params"]
    m.target_mean, m.target_std = p.mean(0), p.std(0)
    ctx.set_model(m)
    n = 20_011
    if csr:
        g = ctx.gen_synthetic_csr(n, root=0xD50B2)
        out = ctx.pipeline_csr(g["row_ptr"], g["entries"], g["dcgm"], 0.8, want_params=True)
    else:
        g = ctx.gen_synthetic(n, root=0xD50B2, params=False)
        out = ctx.pipeline(g["counts"], g["dcgm"], 0.8, want_params=True)
    host = port.gen_stream(0xD50B2, n, want=("counts", "dcgm"))
    d = dom.dev.as_array()
    st, want = port.pipeline(host["counts"], host["dcgm"].astype(np.float32).astype(np.float64),
                             f32model(m), dom.core_freqs_mhz, dom.mem_freqs_mhz, d, 0.8,
                             dom.dev.pmax_w)
    assert st == 0
    got = out["params"].cpu().numpy().T.astype(np.float64)
    tol = 1e-5 * np.abs(want["params"]) + 1e-6 * m.target_std[None, :]
    assert (np.abs(got - want["params"]) <= tol).all()
    rule = check_index_rule(got, want["params"], out["idx"].cpu().numpy(), want["idx"],
                            dom.core_freqs_mhz, dom.mem_freqs_mhz, d, 0.8, dom.dev.pmax_w)
    assert rule["mismatches"] <= n // 1000


def test_generic_fit_model_vs_oracle(ctx, port):
    """fit_model with a layer_sizes override: device epochs vs the oracle's sgd_epoch."""
    sizes = [134, 32, 7]
    g = port.gen_stream(0xACCE5505, 200, want=("params", "fused"))
    f, t = g["fused"], g["params"]
    mean, std, _ = port.target_stats(t)
    seed, lr, batch, epochs = 11, 0.05, 16, 4
    model, trace = fit_model(ctx, f, t, sizes, mean, std, lr, batch, epochs, seed)
    cur = init_mlp(sizes, seed=seed)
    cur.target_mean, cur.target_std = mean, std
    cur = f32model(cur)
    st, want = fork(seed, 0x5D0), []
    ff = f.astype(np.float32).astype(np.float64)
    for _ in range(epochs):
        loss, ws, bs, st = port.sgd_epoch(cur, ff, t, mean, std, lr, batch, st)
        cur.weights, cur.biases = ws, bs
        want.append(loss)
    np.testing.assert_allclose(trace, want, rtol=2e-4)
    for a, b in zip(model.weights, cur.weights):
        assert np.abs(a - b).max() <= 2e-4 * np.abs(b).max()


def test_train_with_layer_sizes(ctx, port):
    """train() with TrainConfig.layer_sizes = [in, 16, out] runs end to end on the GPU."""
    g = port.gen_stream(0xACCE5505, 60, want=("params", "fused"))
    res = train(ctx, g["fused"], g["params"], [(0.05, 8)], seed=3, epochs=3, sizes=[134, 16, 7])
    assert res["model"].layer_sizes == [134, 16, 7]
    assert len(res["epoch_loss"]) == 3 and np.isfinite(res["epoch_loss"]).all()


def test_generic_limits(ctx):
    m = init_mlp([4, 300, 2], seed=1)
    m.target_mean, m.target_std = np.zeros(2), np.ones(2)
    with pytest.raises(DsoError) as e:
        ctx.set_model(m)
    assert e.value.kind == ErrorKind.InvalidModel


def test_featurize_u64(ctx, port):
    """64-bit counts: equal to dso_featurize on 32-bit-range counts, and the
    reference's double quotient (rounded to float) on counts beyond 2^32."""
    n = 3001
    g = ctx.gen_synthetic(n, root=71, params=False)
    c32 = g["counts"].cpu().numpy().view(np.uint32).astype(np.uint64)
    a = ctx.featurize(g["counts"], g["dcgm"]).cpu().numpy()
    b = ctx.featurize_u64(torch.from_numpy(c32.view(np.int64)).cuda(), g["dcgm"]).cpu().numpy()
    np.testing.assert_array_equal(a, b)
    rng = np.random.default_rng(2)
    big = (rng.integers(0, 1 << 40, size=(126, n), dtype=np.uint64) *
           (rng.uniform(size=(126, n)) < 0.2))
    got = ctx.featurize_u64(torch.from_numpy(big.view(np.int64)).cuda(), g["dcgm"]).cpu().numpy()
    cats = [(0, 101), (101, 118), (118, 126)]
    for lo, hi in cats:
        tot = big[lo:hi].sum(axis=0).astype(np.float64)
        want = np.where(tot > 0, big[lo:hi].astype(np.float64) / np.where(tot > 0, tot, 1), 0.0)
        np.testing.assert_array_equal(got[8 + lo:8 + hi], want.astype(np.float32))
    np.testing.assert_array_equal(got[:8], g["dcgm"].cpu().numpy())
