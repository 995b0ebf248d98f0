"""GPU parity: synthetic generator, feature stage and DCGM mean vs the oracle.

Integer/byte work is bit-exact: generated PTX counts equal the host generator's;
fractions and DCGM means equal the reference's double results rounded once to
float (the reference computes in double; see DESIGN.md §4.1 for why the FP32
correctly-rounded quotient is that value)."""

import numpy as np
import pytest
import torch

from paper_2407_13096_b200 import DsoError, ErrorKind

pytestmark = pytest.mark.gpu


def test_gen_synthetic_bit_exact(ctx, port):
    n = 4096
    for root, salt, first in ((0xD50B203, 0, 0), (0xACCE5506, 0x7e57000, 0), (99, 0, 123_456)):
        g = ctx.gen_synthetic(n, root=root, salt_base=salt, first=first)
        o = port.gen_stream(root, n, first=first, salt_base=salt)
        np.testing.assert_array_equal(g["counts"].cpu().numpy().T.view(np.uint32), o["counts"])
        np.testing.assert_array_equal(g["params"].cpu().numpy().T, o["params"].astype(np.float32))
        np.testing.assert_array_equal(g["dcgm"].cpu().numpy().T, o["dcgm"].astype(np.float32))


def test_featurize_bit_exact_on_generated(ctx, port):
    n = 8192
    g = ctx.gen_synthetic(n, root=5)
    fused = ctx.featurize(g["counts"], g["dcgm"]).cpu().numpy().T
    counts = g["counts"].cpu().numpy().T.view(np.uint32)
    want = port.featurize(counts).astype(np.float32)
    np.testing.assert_array_equal(fused[:, 8:], want)
    np.testing.assert_array_equal(fused[:, :8], g["dcgm"].cpu().numpy().T)


def test_featurize_random_counts_and_edges(ctx, port):
    rng = np.random.default_rng(3)
    n = 4096
    c = rng.integers(0, 50_000, size=(n, 126)).astype(np.uint32)
    c[::5] = rng.integers(0, 3, size=(len(c[::5]), 126))   # tiny totals
    c[1::7, :101] = 0                                          # zero instr total
    c[2::11, 101:118] = 0                                      # zero dtype total
    c[3] = 0                                                   # all zero
    c[4, 0] = 1 << 25                                          # total >= 2^24 (FP64 path)
    c[6, 101:118] = (1 << 23) + rng.integers(0, 1000, 17)       # large dtype total
    dc = rng.uniform(0, 1, size=(n, 8)).astype(np.float32)
    ct = torch.from_numpy(c.T.copy().view(np.int32)).cuda()
    dt = torch.from_numpy(dc.T.copy()).cuda()
    fused = ctx.featurize(ct, dt).cpu().numpy().T
    want = port.featurize(c).astype(np.float32)
    np.testing.assert_array_equal(fused[:, 8:], want)
    assert fused[3].sum() == dc[3].sum()
    # KATs (test_ptx_features.cpp:63-91)
    k = np.zeros((3, 126), np.uint32)
    k[0, 0] = k[0, 71] = k[0, 103] = 1
    k[1, 111], k[1, 103] = 3, 1
    f = ctx.featurize(torch.from_numpy(k.T.copy().view(np.int32)).cuda(),
                      torch.zeros((8, 3), device="cuda")).cpu().numpy().T
    assert f[0, 8 + 0] == 0.5 and f[0, 8 + 71] == 0.5 and f[0, 8 + 103] == 1.0
    assert f[1, 8 + 111] == 0.75 and f[1, 8 + 103] == 0.25 and f[2].sum() == 0


def test_dcgm_mean(ctx, port):
    rng = np.random.default_rng(4)
    rows, n = 37, 1000
    s = rng.uniform(0, 1, size=(rows, 8, n))
    mean, bad = ctx.dcgm_mean(torch.from_numpy(s).cuda())
    mean = mean.cpu().numpy()
    for k in range(0, n, 97):
        st, v, _ = port.dcgm_mean(s[:, :, k])
        assert st == 0
        np.testing.assert_array_equal(mean[:, k], v.astype(np.float32))
    assert (bad.cpu().numpy() == 0).all()
    s[5, 3, 17] = 1.3
    with pytest.raises(DsoError) as e:
        ctx.dcgm_mean(torch.from_numpy(s).cuda())
    assert e.value.kind == ErrorKind.OutOfRange and "row 6" in e.value.message
