"""GPU parity: dso_optimal_config vs the reference's own optimal_config
(proj/src/optimizer.cpp:119-205 via oracle/_ref), bit for bit on every output:
best pair, cost, energy, time, candidates_evaluated, fallback, presnap."""

import numpy as np
import pytest
import torch

from paper_2407_13096_b200 import DsoError, DvfsDomain, DeviceConstants, ErrorKind

pytestmark = pytest.mark.gpu

DOMAINS = ["toy", "c1", "c1_literal", "c2", "c3", "grid10x10"]


def _params(g, name, rng, n):
    base = g[f"{name}/params"]
    extra = np.column_stack([rng.uniform(40, 90, n), rng.uniform(5, 15, n),
                             rng.uniform(0.004, 0.02, n), rng.uniform(0.002, 0.0055, n),
                             rng.uniform(0.04, 0.3, n), rng.uniform(1, 440, n),
                             rng.uniform(1, 440, n)])
    extra[::7, 5] = 0.0                       # alpha = 0: knee at infinity
    extra[3::11, 6] = 0.0                     # beta = 0: knee at zero -> fallback
    extra[5::13, 6] = extra[5::13, 5] * 1e-3  # knee below the core table -> fallback
    extra[1::17, 0] = np.nan                  # passes validate(), like the reference
    extra[2::19, 1] = -1.0                    # invalid -> InvalidArgument
    bad = ~(extra[:, 5] + extra[:, 6] > 0)
    extra[bad, 6] = 1.0
    return np.concatenate([base, extra])


def _same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return np.array_equal(a, b, equal_nan=True) if a.dtype.kind == "f" else np.array_equal(a, b)


@pytest.mark.parametrize("name", DOMAINS)
@pytest.mark.parametrize("eta", [0.0, 0.5, 0.8, 1.0])
def test_optimal_config_bit_exact(ctx, ref, golden_sweep, name, eta):
    g = golden_sweep
    core, mem, dev = g[f"{name}/core"], g[f"{name}/mem"], g[f"{name}/dev"]
    ctx.set_domain(DvfsDomain(core, mem, DeviceConstants(*dev)))
    pmax = float(dev[1]) if name != "toy" else 200.0
    p = _params(g, name, np.random.default_rng(sum(map(ord, name))), 20_000)
    want = ref.optimal_config(p, core, mem, dev, eta, pmax)
    for where in ("device", "host"):
        arg = torch.from_numpy(p).cuda() if where == "device" else p
        got = ctx.optimal_config(arg, eta, pmax)
        got = {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in got.items()}
        np.testing.assert_array_equal(got["kstatus"], want["kstatus"])
        ok = want["kstatus"] == 0
        assert _same(got["idx"][ok], want["idx"][ok]), where
        for k in ("cost", "energy", "time", "candidates"):
            assert _same(got[k][ok], want[k][ok]), (k, where)
        assert _same(got["fallback"][ok].astype(bool), want["fallback"][ok]), where
        assert _same(got["presnap"][ok], want["presnap"][ok]), where
    assert want["fallback"][ok].any()


def test_optimal_config_errors(ctx):
    ctx.set_domain(DvfsDomain([705.0, 900.0, 1380.0], [438.0, 877.0]))
    p = np.array([[10.0, 5.0, 2.0, 3.0, 1.0, 8.0, 6.0]])
    for eta in (1.5, -0.1, float("nan")):
        with pytest.raises(DsoError) as e:
            ctx.optimal_config(p, eta)
        assert e.value.kind == ErrorKind.EtaOutOfRange
    r = ctx.optimal_config(np.zeros((0, 7)), 0.5)
    assert r["idx"].shape == (0,)
