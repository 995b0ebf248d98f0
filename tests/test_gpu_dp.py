"""Data-parallel training inside the library (GPU): dso_train_step (gradient ->
NCCL allreduce -> update) and dso_fit_model (fit_model's epoch loop,
mlp.cpp:84-130) against the two-call path and the oracle.

The box has one GPU, so the communicator here is a one-rank NCCL communicator
made by the library (dso_nccl_unique_id / dso_nccl_comm_init): the collective
runs for real (an allreduce over one rank is the identity) and the results must
equal the communicator-free path bit for bit.  The multi-rank arithmetic (shares
of a batch summed, one update on every replica) is covered on CPU by
tests/test_dp_gloo.py."""

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2407_13096_b200 import _lib, init_mlp
from paper_2407_13096_b200.train import fork, shuffled_order

pytestmark = pytest.mark.gpu


class OneRankComm:
    def __init__(self, device=0):
        L = _lib.lib()
        uid = (C.c_uint8 * 128)()
        assert L.dso_nccl_unique_id(uid) == 0
        h = C.c_void_p()
        assert L.dso_nccl_comm_init(1, uid, 0, device, C.byref(h)) == 0
        self.handle, self.L = h, L

    def close(self):
        self.L.dso_nccl_comm_destroy(self.handle)


@pytest.fixture(scope="module")
def comm():
    v = C.c_int32()
    if _lib.lib().dso_nccl_version(C.byref(v)) != 0:
        pytest.fail("libnccl.so.2 is not loadable on the GPU box")
    c = OneRankComm()
    yield c
    c.close()


def data(port, n, seed=5):
    g = port.gen_stream(seed, n, want=("params", "fused"))
    mean, std, _ = port.target_stats(g["params"])
    y = (g["params"] - mean) / std
    x = torch.from_numpy(np.ascontiguousarray(g["fused"].T.astype(np.float32))).cuda()
    yt = torch.from_numpy(np.ascontiguousarray(y.T.astype(np.float32))).cuda()
    return x, yt, g, mean, std


def model(mean, std, seed=424242):
    m = init_mlp(seed=seed)
    m.target_mean, m.target_std = mean, std
    return m


def test_train_step_equals_grad_apply(ctx, port, comm):
    x, y, _, mean, std = data(port, 3000)
    m = model(mean, std)
    ctx.set_model(m)
    g, loss = ctx.train_grad(x, y)
    ctx.train_apply(g, 0.1, 1.0 / (3000 * 7))
    want = ctx.get_model().flat()
    want_loss = float(loss.item()) / (3000 * 7)
    for c in (None, comm):
        ctx.set_model(m)
        got_loss = ctx.train_step(x, y, 0.1, 3000, comm=c)
        got = ctx.get_model().flat()
        for a, b in zip(got, want):
            np.testing.assert_array_equal(a, b)
        assert got_loss == want_loss


def test_train_step_shares_sum_to_the_batch(ctx, port):
    """Two 'ranks' run in sequence on one device: the sum of their share gradients
    applied once equals the whole-batch step (the DP identity the allreduce uses)."""
    x, y, _, mean, std = data(port, 2048, seed=6)
    m = model(mean, std)
    ctx.set_model(m)
    ga, la = ctx.train_grad(x[:, :1000].contiguous(), y[:, :1000].contiguous())
    ga = ga.clone()
    gb, lb = ctx.train_grad(x[:, 1000:].contiguous(), y[:, 1000:].contiguous())
    ctx.train_apply(ga + gb, 0.1, 1.0 / (2048 * 7))
    split = ctx.get_model().flat()
    ctx.set_model(m)
    ctx.train_step(x, y, 0.1, 2048, want_loss=False)
    whole = ctx.get_model().flat()
    for a, b in zip(split, whole):
        np.testing.assert_allclose(a, b, rtol=0, atol=2e-6)


def test_fit_model_graph_comm_and_oracle(ctx, port, comm):
    """dso_fit_model: the CUDA-graph path (no communicator) == the launch-by-launch
    path with a one-rank NCCL communicator, bit for bit; both follow the oracle's
    sgd_epoch (mlp.cpp:84-112) over 5 epochs."""
    n, batch, epochs, seed = 301, 16, 5, 77
    x, y, g, mean, std = data(port, n, seed=8)
    m = model(mean, std, seed=seed)
    runs = []
    for c in (None, comm):
        ctx.set_model(m)
        trace = ctx.fit_model(x, y, 0.05, batch, epochs, seed, comm=c)
        runs.append((trace, ctx.get_model().flat()))
    assert runs[0][0] == runs[1][0]
    for a, b in zip(runs[0][1], runs[1][1]):
        np.testing.assert_array_equal(a, b)
    # oracle: the same epochs in double (targets already standardized: mean 0, std 1)
    feats = x.cpu().numpy().T.astype(np.float64)
    targ = y.cpu().numpy().T.astype(np.float64)
    cur, st, want = m.copy(), fork(seed, 0x5D0), []
    for _ in range(epochs):
        loss, ws, bs, st = port.sgd_epoch(cur, feats, targ, np.zeros(7), np.ones(7), 0.05, batch, st)
        cur.weights, cur.biases = ws, bs
        want.append(loss)
    np.testing.assert_allclose(runs[0][0], want, rtol=2e-4)
    W = cur.flat()[0]
    np.testing.assert_allclose(runs[0][1][0], W, rtol=0, atol=2e-4 * np.abs(W).max())
    # the order used is the reference's: the shuffle state advanced epochs times
    order, _ = shuffled_order(n, fork(seed, 0x5D0))
    assert sorted(order) == list(range(n))


def test_fit_model_errors(ctx, port):
    from paper_2407_13096_b200 import DsoError, ErrorKind
    x, y, _, mean, std = data(port, 10)
    ctx.set_model(model(mean, std))
    with pytest.raises(DsoError) as e:
        ctx.fit_model(x, y, 0.1, 0, 3, 1)
    assert e.value.kind == ErrorKind.InvalidArgument
    with pytest.raises(DsoError) as e:
        ctx.fit_model(x, y, 0.1, 4, 3, 1, nranks=2)  # no communicator
    assert e.value.kind == ErrorKind.InvalidArgument
