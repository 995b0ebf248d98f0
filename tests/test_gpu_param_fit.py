"""GPU parity: dso_param_fit (batched fit_power / fit_time) vs the param_fit
restatement in the oracle (itself pinned to the reference's unit tests,
tests/test_oracle_param_fit.py).  FP64 both sides; the device applies the QR
solve operator as a matrix, so coefficients agree to ~1e-12 relative; flags,
iteration counts and statuses agree exactly."""

import numpy as np
import pytest
import torch

from test_oracle_param_fit import KTRUTH, power_of, time_of

pytestmark = pytest.mark.gpu


def measure(truths, cfg, noise, rng):
    """measure_sweep (sim_harness.cpp:145-170): multiplicative noise per sample."""
    P = np.array([[power_of(p, *c) for c in cfg] for p in truths]).T    # [S, n]
    T = np.array([[time_of(p, c[1], c[2]) for c in cfg] for p in truths]).T
    if noise:
        P = P * (1 + noise * rng.uniform(-1, 1, P.shape))
        T = T * (1 + noise * rng.uniform(-1, 1, T.shape))
    return np.ascontiguousarray(P), np.ascontiguousarray(T)


def grid_cfg(core, mem, dev=(0.5, 300.0, 0.55, 2.10, 1000.0)):
    out = []
    for fc in core:
        d = fc / dev[4] - dev[0]
        vc = 2.0 * d * d + dev[0]
        for fm in mem:
            out.append([vc, fc, fm])
    return np.array(out)


def truths_of(rng, n):
    t = np.column_stack([rng.uniform(40, 90, n), rng.uniform(5, 15, n),
                         rng.uniform(0.004, 0.02, n), rng.uniform(0.002, 0.0055, n),
                         rng.uniform(0.04, 0.3, n), rng.uniform(40, 400, n),
                         rng.uniform(40, 400, n)])
    t[::9, 6] = 1e-3     # memory-bound everywhere -> partial identifiability
    t[4::9, 5] = 1e-3    # core-bound everywhere
    return t


@pytest.mark.parametrize("grid", ["default14x3", "c3_128x4", "toy4x4"])
@pytest.mark.parametrize("noise", [0.0, 0.01, 0.05])
def test_param_fit_vs_oracle(ctx, port, grid, noise):
    rng = np.random.default_rng(7)
    if grid == "default14x3":
        cfg = grid_cfg([705.0 + 52 * k for k in range(13)] + [1380.0], [438.0, 658.0, 877.0])
        n = 400
    elif grid == "c3_128x4":
        cfg = grid_cfg(list(705 + 675 * np.arange(128) / 127), list(438 + 439 * np.arange(4) / 3))
        n = 60
    else:
        cfg = np.array([[1.0, fc, fm] for fc in (1.0, 2.0, 3.0, 4.0) for fm in (1.0, 2.0, 3.0, 4.0)])
        n = 200
    truths = truths_of(rng, n)
    if grid == "toy4x4":
        truths[:, 5:7] = np.column_stack([rng.uniform(2, 20, n), rng.uniform(2, 20, n)])
    P, T = measure(truths, cfg, noise, rng)
    T[:, 5] *= -1                      # one kernel with a non-positive time
    P[0, 6] = 0.0                      # one kernel with a non-positive power
    for where in ("device", "host"):
        if where == "device":
            got = ctx.param_fit(cfg, torch.from_numpy(P).cuda(), torch.from_numpy(T).cuda())
            got = {k: v.cpu().numpy() for k, v in got.items()}
        else:
            got = ctx.param_fit(cfg, P, T)
        for k in range(n):
            st, want = port.fit_power(cfg, P[:, k])
            assert got["pstatus"][k] == st, (where, k)
            if st == 0:
                np.testing.assert_allclose(got["pfit"][:4, k], want[:4], rtol=1e-9,
                                           atol=1e-12 * np.abs(want[:4]).max())
                assert got["pfit"][4, k] == pytest.approx(want[4], rel=1e-6, abs=1e-9)
                assert got["pfit"][5, k] == want[5]
            st, want, _ = port.fit_time(cfg, T[:, k])
            assert got["tstatus"][k] == st, (where, k)
            if st == 0:
                np.testing.assert_allclose(got["tfit"][:3, k], want[:3], rtol=1e-8,
                                           atol=1e-12 * np.abs(want[:3]).max())
                assert got["tfit"][3, k] == pytest.approx(want[3], rel=1e-6, abs=1e-9)
                np.testing.assert_array_equal(got["tfit"][4:7, k], want[4:7])


def test_param_fit_reference_kats(ctx):
    """The reference's own unit-test cases (test_param_fit.cpp) through the GPU path."""
    cfg = np.array([[vc, fc, fm] for vc in (0.8, 1.2) for fc in (600.0, 1100.0)
                    for fm in (400.0, 800.0)])
    P = np.array([[power_of(KTRUTH, *c)] for c in cfg])
    r = ctx.param_fit(cfg, P)
    assert r["pstatus"][0] == 0
    np.testing.assert_allclose(r["pfit"][:4, 0], KTRUTH[:4], rtol=1e-9)
    # single voltage level: RankDeficient; fewer than 4 samples: RankDeficient
    cfgc = np.array([[1.0, fc, fm] for fc in (600.0, 800.0) for fm in (400.0, 700.0)])
    r = ctx.param_fit(cfgc, np.array([[power_of(KTRUTH, *c)] for c in cfgc]))
    assert r["pstatus"][0] == 9
    r = ctx.param_fit(cfgc[:3], np.array([[power_of(KTRUTH, *c)] for c in cfgc[:3]]))
    assert r["pstatus"][0] == 9
    # 4x4 time grid: both branches; fm = 1e9: memory never binds
    cfgt = np.array([[1.0, fc, fm] for fc in (1.0, 2.0, 3.0, 4.0) for fm in (1.0, 2.0, 3.0, 4.0)])
    r = ctx.param_fit(cfgt, time=np.array([[time_of(KTRUTH, c[1], c[2])] for c in cfgt]))
    np.testing.assert_allclose(r["tfit"][:3, 0], [1.0, 8.0, 6.0], rtol=1e-6)
    assert r["tfit"][5, 0] == 0
    cfg1 = np.array([[1.0, fc, 1e9] for fc in (1.0, 2.0, 3.0, 4.0)])
    r = ctx.param_fit(cfg1, time=np.array([[time_of(KTRUTH, c[1], c[2])] for c in cfg1]))
    assert r["tfit"][5, 0] == 1 and r["tfit"][1, 0] == 0.0
    np.testing.assert_allclose(r["tfit"][[0, 2], 0], [1.0, 6.0], rtol=1e-6)
    cfg2 = np.array([[1.0, fc, 1.0] for fc in (1.0, 2.0)])
    r = ctx.param_fit(cfg2, time=np.array([[time_of(KTRUTH, c[1], c[2])] for c in cfg2]))
    assert r["tstatus"][0] == 10  # Underdetermined
