"""Pin the CPU oracle (test infrastructure) before trusting it.

The C restatement (oracle/dso_oracle.c) is checked against
  * the reference itself: brute_force_config / optimal_config / Rng compiled
    from /root/reference/proj into oracle/_ref, frozen in tests/golden/*;
  * the reference's own golden file (mlp_forward_golden.json) and recorded
    acceptance KATs (proj/test_output.txt);
  * the reference unit tests' hand values (test_dvfs_model.cpp, test_ptx_features.cpp,
    test_telemetry.cpp, test_sim_harness.cpp, test_mlp.cpp).
"""

import ctypes as C
import types

import numpy as np
import pytest

KREF = [10.0, 5.0, 2.0, 3.0, 1.0, 8.0, 6.0]


def model_ns(sizes, ws, bs, mean=None, std=None):
    out = sizes[-1]
    return types.SimpleNamespace(layer_sizes=sizes, weights=ws, biases=bs,
                                 target_mean=np.zeros(out) if mean is None else mean,
                                 target_std=np.ones(out) if std is None else std)


# ---- RNG (rng.hpp) ------------------------------------------------------------------
def test_rng_matches_reference(port, golden_json):
    g = golden_json("rng_golden.json")
    assert [int(v) for v in port.rng_u64(42, 16)] == g["u64_seed_42"]
    assert list(port.rng_uniform01(7, 16)) == g["uniform01_seed_7"]
    assert [int(v) for v in port.rng_below(3, 10, 32)] == g["below_seed_3_m_10"]
    assert [int(v) for v in port.fork_seeds(0xACCE5506, 0x7e57000, 20)] == \
        g["fork_seeds_0xACCE5506_0x7e57000"]
    assert [int(v) for v in port.shuffled_indices(99, 20)] == g["shuffled_seed_99_n_20"]


# ---- DVFS model (test_dvfs_model.cpp:15-69) ---------------------------------------
def test_dvfs_hand_values(port):
    assert port.power(KREF, 1.0, 4.0, 2.0) == pytest.approx(31.0, rel=1e-12)
    assert port.exec_time(KREF, 1.0, 3.0, 2.0) == pytest.approx(5.0)
    assert port.exec_time(KREF, 1.0, 3.0, 4.0) == pytest.approx(3.0)
    e = port.power(KREF, 1.0, 3.0, 4.0) * port.exec_time(KREF, 1.0, 3.0, 4.0)
    assert e == pytest.approx(96.0)
    T = port.exec_time(KREF, 1.0, 3.0, 4.0)
    P = port.power(KREF, 1.0, 3.0, 4.0)
    for eta, want in ((1.0, 96.0), (0.0, 120.0), (0.5, 108.0)):
        assert (eta * P + (1 - eta) * 40.0) * T == pytest.approx(want)


def test_dvfs_matches_reference_header(port, ref):
    rng = np.random.default_rng(5)
    for _ in range(200):
        p = [rng.uniform(1, 50), rng.uniform(0.1, 20), rng.uniform(0.001, 0.05),
             rng.uniform(0.001, 0.01), rng.uniform(0.01, 0.5), rng.uniform(10, 400),
             rng.uniform(10, 400)]
        vc, fc, fm = rng.uniform(0.6, 2.0), rng.uniform(700, 1400), rng.uniform(400, 900)
        assert port.power(p, vc, fc, fm) == ref.model_eval("power", p, vc, fc, fm)[1]
        assert port.exec_time(p, vc, fc, fm) == ref.model_eval("exec_time", p, vc, fc, fm)[1]
        fcm = rng.uniform(705, 1380)
        assert port.required_voltage_mhz(fcm, [0.5, 300, 0.55, 2.1, 1000]) == \
            ref.vf_eval("required_voltage_mhz", fcm, [0.5, 300, 0.55, 2.1, 1000])[1]


# ---- sweep: bit-exact against the reference brute_force_config ---------------------
DOMAINS = ["toy", "c1", "c1_literal", "c2", "c3", "grid10x10"]
ETAS = [0.0, 0.2, 0.5, 0.8, 1.0]


@pytest.mark.parametrize("name", DOMAINS)
@pytest.mark.parametrize("eta", ETAS)
def test_port_sweep_bit_exact(port, golden_sweep, name, eta):
    g = golden_sweep
    core, mem, dev = g[f"{name}/core"], g[f"{name}/mem"], g[f"{name}/dev"]
    params = g[f"{name}/params"]
    key = f"{name}/eta{eta}"
    st, r = port.brute_force(params, core, mem, dev, eta, float(g[key + "/pmax"][0]), threads=4)
    assert st == 0
    ok = g[key + "/kstatus"] == 0
    np.testing.assert_array_equal(r["kstatus"], g[key + "/kstatus"])
    np.testing.assert_array_equal(r["idx"][ok], g[key + "/idx"][ok])
    for f in ("cost", "energy", "time"):
        np.testing.assert_array_equal(r[f][ok], g[key + "/" + f][ok])


def test_sweep_structural_cases(port):
    """test_optimizer.cpp:67-83, 176-197."""
    dev = [0.5, 300.0, 0.55, 2.10, 1000.0]
    core = [900.0]
    st, r = port.brute_force([KREF], core, [600.0], dev, 0.5, 300.0)
    assert st == 0 and r["idx"][0] == 0
    # alpha = 0: the lowest memory clock wins at eta = 1
    c1 = [705.0 + 52.0 * k for k in range(13)] + [1380.0]
    st, r = port.brute_force([[20.0, 5.0, 0.01, 0.002, 0.05, 0.0, 200.0]], c1,
                             [438.0, 658.0, 877.0], dev, 1.0, 300.0)
    assert r["idx"][0] % 3 == 0
    # eta outside [0, 1] -> EtaOutOfRange (status 6)
    st, _ = port.brute_force([KREF], c1, [438.0], dev, 1.5, 300.0)
    assert st == 6


def test_validate_domain_kinds(port, ref):
    """test_optimizer.cpp:199-214: the same error kind from port and reference."""
    dev = np.array([0.5, 300.0, 0.55, 2.10, 1000.0])
    c1 = np.array([705.0 + 52.0 * k for k in range(13)] + [1380.0])
    m = np.array([438.0, 658.0, 877.0])
    cases = [
        (c1, m, dev),
        (np.array([900.0, 900.0]), m, dev),
        (c1, np.array([]), dev),
        (c1, m, np.array([0.5, 300.0, 0.55, 0.6, 1000.0])),
        (np.array([400.0, 900.0]), m, dev),
        (c1, m, np.array([0.6, 300.0, 0.55, 2.1, 1000.0])),
        (c1, m, np.array([0.5, -1.0, 0.55, 2.1, 1000.0])),
    ]
    for core, mem, d in cases:
        assert port.validate_domain(core, mem, d) == ref.validate_domain(core, mem, d)


# ---- optimal_config KATs (acceptance AC1/AC2, test_output.txt:15-16) -----------------
def test_ac1_fallbacks_and_equality(golden_sweep, golden_json, port):
    g = golden_sweep
    kat = golden_json("kat.json")
    fb = g["ac1/fallback"]
    # "pre-snap knee identity on 103 results" = the non-fallback runs
    assert int((~fb).sum()) == kat["ac2_non_fallback"]
    # AC1: optimizer equals oracle on 200/200 -> brute force cost equals optimal cost
    core, mem, dev = g["c1/core"], g["c1/mem"], g["c1/dev"]
    for i in range(200):
        st, r = port.brute_force(g["ac1/params"][i:i + 1], core, mem, dev,
                                 float(g["ac1/eta"][i]), 300.0, threads=1)
        assert r["idx"][0] == g["ac1/idx"][i]
        assert abs(r["cost"][0] - g["ac1/opt_cost"][i]) <= 1e-9 * r["cost"][0]


# ---- generator + AC6 KAT ------------------------------------------------------------
def test_generator_endpoints_and_determinism(port):
    """test_sim_harness.cpp:13-51."""
    st, k = port.gen_kernel_rho(5, 1.0)
    assert st == 0 and k["params"][5] < 50.0 and k["dcgm"][3] < 0.1 and k["dcgm"][5] > 0.7
    st, k = port.gen_kernel_rho(5, 0.0)
    assert k["params"][6] < 50.0 and k["dcgm"][3] > 0.7 and k["dcgm"][5] < 0.2
    a = port.gen_seeded(np.array([1234], np.uint64))
    b = port.gen_seeded(np.array([1234], np.uint64))
    c = port.gen_seeded(np.array([1235], np.uint64))
    np.testing.assert_array_equal(a["fused"], b["fused"])
    assert a["params"][0, 5] != c["params"][0, 5]
    g = port.gen_stream(2, 500)
    for p in g["params"]:
        assert port.validate_params(p) == 0
    f = g["fused"]
    assert (f >= 0).all() and (f <= 1).all()
    for lo, hi in ((8, 109), (109, 126), (126, 134)):
        np.testing.assert_allclose(f[:, lo:hi].sum(1), 1.0, atol=1e-9)


def test_generator_slots_match_reference_categories(port, golden_json):
    cats = golden_json("categories.json")
    c = port.gen_stream(11, 64)["counts"]
    nz = np.flatnonzero(c.sum(0))
    names = [("instr", cats["instr"][i]) if i < 101 else
             ("dtype", cats["dtype"][i - 101]) if i < 118 else ("memspace", cats["memspace"][i - 118])
             for i in nz]
    # sim_harness.cpp:70-95 fills exactly these keys
    want = {("instr", s) for s in ("add", "mul", "fma", "ld", "st", "mov", "setp", "bra", "cvt",
                                   "bar", "ret")}
    want |= {("dtype", s) for s in (".f32", ".s32", ".u32", ".b32", ".f64", ".u64", ".b64")}
    want |= {("memspace", s) for s in (".global", ".shared", ".param", ".reg", ".local",
                                       ".const")}
    assert set(names) == want


def _campaign_savings(port, params, core, mem, dev, eta):
    st, r = port.brute_force(params, core, mem, dev, eta, dev[1])
    vdef = port.required_voltage_mhz(core[-1], dev)
    sav, loss = [], []
    for i, p in enumerate(params):
        t_def = port.exec_time(p, vdef, core[-1], mem[-1])
        e_def = port.power(p, vdef, core[-1], mem[-1]) * t_def
        fi, fj = divmod(int(r["idx"][i]), len(mem))
        vc = port.required_voltage_mhz(core[fi], dev)
        t = port.exec_time(p, vc, core[fi], mem[fj])
        e = port.power(p, vc, core[fi], mem[fj]) * t
        sav.append(100 * (e_def - e) / e_def)
        loss.append(100 * (t - t_def) / t_def)
    return np.mean(sav), np.mean(loss)


def test_ac6_kat(port, golden_json):
    """Oracle-predictor campaign at eta = 0.8 (acceptance_main.cpp:272-313): the
    recorded run says 24.1 % saving at 2.00 % loss (test_output.txt:20)."""
    kat = golden_json("kat.json")
    seeds = port.fork_seeds(kat["ac6_seed"], 0x7e57000, 20)
    params = port.gen_seeded(seeds)["params"]
    core = np.array([705.0 + 52.0 * k for k in range(13)] + [1380.0])
    mem = np.array([438.0, 658.0, 877.0])
    dev = np.array([0.5, 300.0, 0.55, 2.10, 1000.0])
    s, l = _campaign_savings(port, params, core, mem, dev, 0.8)
    assert round(s, 1) == kat["ac6_saving_pct_1dp"]
    assert round(l, 2) == kat["ac6_loss_pct_2dp"]
    assert s == pytest.approx(24.1042218, abs=1e-6) and l == pytest.approx(2.0001302, abs=1e-6)
    s0, l0 = _campaign_savings(port, params, core, mem, dev, 0.0)
    assert l0 == 0.0  # eta = 0 keeps the default-level time (test_sim_harness.cpp:103-104)


# ---- features (test_ptx_features.cpp:63-91, 221-256; test_telemetry.cpp) ------------
def test_featurize_kats(port):
    c = np.zeros(126, np.uint32)
    c[0] = 1      # add
    c[71] = 1     # bra
    c[101 + 2] = 1  # .s32
    v = port.featurize(c)[0]
    assert v[0] == 0.5 and v[71] == 0.5 and v[101 + 2] == 1.0 and v[118:].sum() == 0
    c = np.zeros(126, np.uint32)
    c[101 + 10], c[101 + 2] = 3, 1
    v = port.featurize(c)[0]
    assert v[101 + 10] == 0.75 and v[101 + 2] == 0.25
    assert port.featurize(np.zeros(126, np.uint32)).sum() == 0.0
    rng = np.random.default_rng(29)
    cc = rng.integers(0, 1000, size=(50, 126)).astype(np.uint32)
    cc[::7, :101] = 0
    v = port.featurize(cc)
    for lo, hi in ((0, 101), (101, 118), (118, 126)):
        tot = cc[:, lo:hi].astype(np.float64).sum(1)
        s = v[:, lo:hi].sum(1)
        assert np.all((np.abs(s) <= 1e-12) | (np.abs(s - 1) <= 1e-12))
        np.testing.assert_allclose(v[:, lo:hi] * tot[:, None], cc[:, lo:hi], rtol=1e-9)


def test_dcgm_mean_kats(port):
    st, v, _ = port.dcgm_mean([[0.8, 0, 0, 0, 0, 0, 0, 0]])
    assert st == 0 and v[0] == pytest.approx(0.8)
    st, v, _ = port.dcgm_mean([[0.6, 0.1, 0, 0.2, 0, 0.5, 0, 0.3],
                               [0.8, 0.3, 0, 0.4, 0, 0.7, 0, 0.1]])
    np.testing.assert_allclose(v[[0, 1, 3, 5, 7]], [0.7, 0.2, 0.3, 0.6, 0.2])
    st, _, row = port.dcgm_mean([[0.5, 0, 0, 1.3, 0, 0, 0, 0]])
    assert st == 3 and row == 1  # OutOfRange, "row 1"
    st, _, _ = port.dcgm_mean(np.zeros((0, 8)))
    assert st == 2  # EmptyTrace
    a = np.array([[0.2, 0.1, 0, 0.9, 0, 0.4, 0, 0.6], [0.6, 0.5, 0, 0.1, 0, 0.2, 0, 0.2],
                  [0.4, 0.3, 0, 0.5, 0, 0.9, 0, 0.1]])
    _, va, _ = port.dcgm_mean(a)
    _, vb, _ = port.dcgm_mean(a[[2, 0, 1]])
    _, vd, _ = port.dcgm_mean(np.concatenate([a, a]))
    np.testing.assert_allclose(va, vb, rtol=1e-15)
    np.testing.assert_allclose(vd, va, rtol=1e-12)


# ---- MLP (test_mlp.cpp) -------------------------------------------------------------
def test_mlp_golden_forward(port, golden_json):
    """mlp_forward_golden.json: the reference is bit-exact with Eigen's GEMV
    order; the naive-order restatement lands within 4 ulp (measured: <= 2)."""
    g = golden_json("mlp_forward_golden.json")
    sizes = g["layer_sizes"]
    ws, bs = port.init_mlp(sizes, g["seed"])
    x = np.array([(i % 13) / 13.0 for i in range(134)])
    out = port.forward_raw(model_ns(sizes, ws, bs), x)[0]
    ulps = np.abs(out.view(np.int64) - np.array(g["outputs"]).view(np.int64))
    assert ulps.max() <= 4


def test_constant_net_and_clamp(port):
    """test_mlp.cpp:41-54 and 228-241."""
    sizes = [134, 100, 50, 25, 7]
    ws, bs = port.init_mlp(sizes, 1)
    ws = [np.zeros_like(w) for w in ws]
    bs = [np.zeros_like(b) for b in bs]
    means = np.array([10, 5, 2, 3, 1, 8, 6], float)
    m = model_ns(sizes, ws, bs, means, np.ones(7))
    for t in range(3):
        np.testing.assert_allclose(port.forward_raw(m, np.full(134, 0.1 * t))[0], means,
                                   rtol=1e-15)
    ws, bs = port.init_mlp(sizes, 6)
    m = model_ns(sizes, ws, bs, np.full(7, -100.0), np.ones(7))
    p, cl = port.predict_params(m, np.zeros(134))
    assert cl[0] and port.validate_params(p[0]) == 0 and p[0, 6] == 1e-12


def test_gradient_check(port):
    """acceptance AC4 (acceptance_main.cpp:226-252): < 1e-6, mutation 4.76e-02."""
    x = np.array([0.1, 0.7, 0.3, 0.9])
    y = np.array([0.4, -0.6])
    sizes = [4, 3, 3, 3, 2]

    def rel(a, b):
        worst = 0.0
        for ga, gb in zip(a[0] + a[1], b[0] + b[1]):
            d = np.maximum(np.abs(ga) + np.abs(gb), 1e-12)
            worst = max(worst, float((np.abs(ga - gb) / d).max()))
        return worst

    worst = 0.0
    for seed in range(1, 6):
        ws, bs = port.init_mlp(sizes, seed)
        m = model_ns(sizes, ws, bs)
        worst = max(worst, rel(port.analytic_gradients(m, x, y), port.numeric_gradients(m, x, y)))
    assert worst < 1e-6
    ws, bs = port.init_mlp(sizes, 6)
    m = model_ns(sizes, ws, bs)
    a = port.analytic_gradients(m, x, y)
    n = port.numeric_gradients(m, x, y)
    a[0][2][1, 1] *= 1.10
    assert round(rel(a, n), 4) == pytest.approx(0.0476, abs=1e-4)


def test_sgd_loss_trend(port):
    """test_mlp.cpp:174-193: 20-epoch moving average non-increasing (lr 0.1, B 8)."""
    rng_state = 21
    xs, ys = [], []
    s = C.c_uint64(rng_state)
    for _ in range(30):
        x = [port.lib.orc_rng_uniform01(C.byref(s)) for _ in range(4)]
        xs.append(x)
        ys.append([3 * x[0] + x[1] * x[2], 10 - 2 * x[3]])
    xs, ys = np.array(xs), np.array(ys)
    sizes = [4, 10, 2]
    ws, bs = port.init_mlp(sizes, 31)
    mean, std, deg = port.target_stats(ys)
    m = model_ns(sizes, ws, bs, mean, std)
    state = int(port.lib.orc_rng_fork(C.byref(C.c_uint64(31)), 0x5d0))
    losses = []
    for _ in range(400):
        loss, ws, bs, state = port.sgd_epoch(m, xs, ys, mean, std, 0.1, 8, state)
        m = model_ns(sizes, ws, bs, mean, std)
        losses.append(loss)
    w = [np.mean(losses[s:s + 20]) for s in range(0, 400, 20)]
    assert all(b <= a * (1 + 1e-9) for a, b in zip(w, w[1:]))
