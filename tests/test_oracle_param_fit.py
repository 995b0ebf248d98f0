"""Pin the param_fit restatement (oracle/dso_oracle.c orc_fit_power / orc_fit_time)
against the reference's own unit tests (proj/tests/unit/test_param_fit.cpp) and
acceptance checks (proj/tests/acceptance/acceptance_main.cpp:150-200).  The
reference needs Eigen (absent), so these expectations are the pin."""

import numpy as np
import pytest

KTRUTH = [10.0, 5.0, 2.0, 3.0, 1.0, 8.0, 6.0]  # test_param_fit.cpp:46


def power_of(p, vc, fc, fm):  # dvfs_model.hpp:81-84
    return ((p[0] + p[1] * vc) + p[2] * fm) + ((p[3] * vc) * vc) * fc


def time_of(p, fc, fm):  # dvfs_model.hpp:88-90
    a, b = p[5] / fm, p[6] / fc
    return p[4] + (b if a < b else a)


def power_grid(p, vcs, fcs, fms):
    cfg = np.array([[vc, fc, fm] for vc in vcs for fc in fcs for fm in fms])
    return cfg, np.array([power_of(p, *c) for c in cfg])


def time_grid(p, fcs, fms, noise=0.0, rng=None):
    cfg = np.array([[1.0, fc, fm] for fc in fcs for fm in fms])
    t = np.array([time_of(p, c[1], c[2]) for c in cfg])
    if rng is not None:
        t = t * (1.0 + noise * rng.uniform(-1, 1, len(t)))
    return cfg, t


def test_fit_power_exact(port):
    cfg, w = power_grid(KTRUTH, [0.8, 1.2], [600.0, 1100.0], [400.0, 800.0])
    st, f = port.fit_power(cfg, w)
    assert st == 0
    np.testing.assert_allclose(f[:4], KTRUTH[:4], rtol=1e-9)
    assert f[4] == pytest.approx(0.0, abs=1e-9) and f[5] == 0


def test_fit_power_constant_and_errors(port):
    cfg = np.array([[vc, fc, fm] for vc in (0.8, 1.0, 1.3) for fc in (500.0, 900.0)
                    for fm in (300.0, 700.0)])
    st, f = port.fit_power(cfg, np.full(len(cfg), 42.0))
    assert st == 0 and f[0] == pytest.approx(42.0, rel=1e-9)
    assert np.abs(f[1:4]).max() <= 1e-6
    cfg3, w3 = power_grid(KTRUTH, [1.0], [600.0, 800.0, 1000.0], [400.0])
    assert port.fit_power(cfg3[:3], w3[:3])[0] == 9          # RankDeficient (< 4 samples)
    cfgc, wc = power_grid(KTRUTH, [1.0], [600.0, 800.0], [400.0, 700.0])
    assert port.fit_power(cfgc, wc)[0] == 9                  # collinear vc column
    cfgn, wn = power_grid(KTRUTH, [0.8, 1.2], [600.0, 1100.0], [400.0, 800.0])
    wn[3] = -1.0
    assert port.fit_power(cfgn, wn)[0] == 12                 # InvalidArgument


def test_fit_power_random_recovery(port):
    from oracle import port as _p  # noqa: F401
    rng = np.random.default_rng(31)
    for _ in range(30):
        p = [rng.uniform(5, 80), rng.uniform(1, 30), rng.uniform(0.001, 0.05),
             rng.uniform(0.0005, 0.01), 1.0, 1.0, 1.0]
        cfg, w = power_grid(p, [0.7, 1.1, 1.9], [700.0, 1000.0, 1350.0], [450.0, 650.0, 880.0])
        st, f = port.fit_power(cfg, w)
        assert st == 0
        np.testing.assert_allclose(f[:4], p[:4], rtol=1e-6)


def test_fit_time_both_branches(port):
    cfg, t = time_grid(KTRUTH, [1.0, 2.0, 3.0, 4.0], [1.0, 2.0, 3.0, 4.0])
    st, f, _ = port.fit_time(cfg, t)
    assert st == 0
    assert f[0] == pytest.approx(1.0, rel=1e-6)
    assert f[1] == pytest.approx(8.0, rel=1e-6)
    assert f[2] == pytest.approx(6.0, rel=1e-6)
    assert f[5] == 0 and f[3] == pytest.approx(0.0, abs=1e-9)


def test_fit_time_single_branch_and_errors(port):
    cfg, t = time_grid(KTRUTH, [1.0, 2.0, 3.0, 4.0], [1e9])
    st, f, _ = port.fit_time(cfg, t)
    assert st == 0 and f[5] == 1 and f[1] == 0.0
    assert f[0] == pytest.approx(1.0, rel=1e-6) and f[2] == pytest.approx(6.0, rel=1e-6)
    cfg2, t2 = time_grid(KTRUTH, [1.0, 2.0], [1.0])
    assert port.fit_time(cfg2, t2)[0] == 10                  # Underdetermined
    cfg3, t3 = time_grid(KTRUTH, [1.0, 2.0, 3.0], [1.0])
    t3[1] = 0.0
    assert port.fit_time(cfg3, t3)[0] == 12                  # InvalidArgument


def test_fit_time_noise_and_scaling(port):
    rng = np.random.default_rng(47)
    cfg, t = time_grid(KTRUTH, [1.0, 2.0, 3.0, 4.0], [1.0, 2.0, 3.0, 4.0], 0.01, rng)
    st, f, _ = port.fit_time(cfg, t)
    assert st == 0 and f[3] <= 2.0
    cfg, t = time_grid(KTRUTH, [1.0, 2.0, 3.0, 4.0], [1.0, 2.0, 3.0, 4.0])
    _, base, _ = port.fit_time(cfg, t)
    _, big, _ = port.fit_time(cfg, 3.7 * t)
    np.testing.assert_allclose(big[:3], 3.7 * base[:3], rtol=1e-9)


def test_acceptance_noiseless_recovery(port):
    """acceptance_main.cpp:150-190: 25 random truths, 3x3x3 power grid and 4x4 time
    grid with alpha/beta within [0.5, 2] of each other: recovery within 1e-6."""
    rng = np.random.default_rng(1)
    for _ in range(25):
        beta = rng.uniform(2, 20)
        p = [rng.uniform(5, 80), rng.uniform(1, 30), rng.uniform(0.001, 0.05),
             rng.uniform(0.0005, 0.01), rng.uniform(0.05, 0.5), beta * rng.uniform(0.5, 2), beta]
        cfg, w = power_grid(p, [0.7, 1.1, 1.9], [700.0, 1000.0, 1350.0], [450.0, 650.0, 880.0])
        st, f = port.fit_power(cfg, w)
        assert st == 0
        np.testing.assert_allclose(f[:4], p[:4], rtol=1e-6)
        cfg, t = time_grid(p, [1.0, 2.0, 3.0, 4.0], [1.0, 2.0, 3.0, 4.0])
        st, f, _ = port.fit_time(cfg, t)
        assert st == 0
        np.testing.assert_allclose(f[:3], [p[4], p[5], p[6]], rtol=1e-6)
