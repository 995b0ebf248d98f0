"""GPU parity: grid sweep + eta objective + argmin vs the reference brute_force_config.

Bars (BASELINE.json north_star):
  * FP32 path (dso_sweep / dso_eta_sweep): chosen index equal to the reference's
    except on objective near-ties within 1e-6 relative (judged in double with the
    reference's formula); cost, energy, time within 1e-5 relative.
  * FP64 path (dso_sweep_f64): bit-identical idx, cost, energy, time, kstatus.
Reference outputs come from tests/golden/sweep_golden.npz (the reference's own
optimizer.cpp, via oracle/_ref) and, for large batches, from oracle/_ref directly.
"""

import numpy as np
import pytest
import torch

from helpers import check_argmin, rel_err
from paper_2407_13096_b200 import DsoError, DvfsDomain, DeviceConstants, ErrorKind, config_domain

pytestmark = pytest.mark.gpu

DOMAINS = ["toy", "c1", "c1_literal", "c2", "c3", "grid10x10"]
ETAS = [0.0, 0.2, 0.5, 0.8, 1.0]


def set_golden_domain(ctx, g, name):
    core, mem, dev = g[f"{name}/core"], g[f"{name}/mem"], g[f"{name}/dev"]
    ctx.set_domain(DvfsDomain(core, mem, DeviceConstants(*dev)))
    return core, mem, dev


def soa(params, ld=None):
    params = np.asarray(params, np.float64)
    n = len(params)
    ld = n if ld is None else ld
    t = torch.zeros((7, ld), dtype=torch.float32)
    t[:, :n] = torch.from_numpy(params.T.astype(np.float32))
    return t.cuda()


@pytest.mark.parametrize("name", DOMAINS)
@pytest.mark.parametrize("eta", ETAS)
def test_sweep_f32_vs_reference(ctx, golden_sweep, name, eta):
    g = golden_sweep
    core, mem, dev = set_golden_domain(ctx, g, name)
    params = g[f"{name}/params"]
    key = f"{name}/eta{eta}"
    pmax = float(g[key + "/pmax"][0])
    r = ctx.brute_force_config(soa(params), eta, pmax)
    ks = r["kstatus"].cpu().numpy()
    np.testing.assert_array_equal(ks, g[key + "/kstatus"])
    ok = ks == 0
    idx = r["idx"].cpu().numpy()
    assert (idx[~ok] == -1).all()
    # the reference at the f32-rounded inputs is what the GPU sees; judge ties in double
    p32 = params.astype(np.float32).astype(np.float64)
    finite = ok & np.isfinite(g[key + "/cost"])
    check_argmin(p32[finite], idx[finite], g[key + "/idx"][finite], core, mem, dev, eta, pmax)
    same = finite & (idx == g[key + "/idx"])
    for f in ("cost", "energy", "time"):
        got = r[f].cpu().numpy()
        assert rel_err(got[same], g[key + "/" + f][same]).max(initial=0) <= 1e-5, f
    # NaN params (pass validation, dvfs_model.hpp:51) keep pair 0 like the reference
    nan_k = ok & ~np.isfinite(g[key + "/cost"])
    np.testing.assert_array_equal(idx[nan_k], g[key + "/idx"][nan_k])


@pytest.mark.parametrize("name", DOMAINS)
@pytest.mark.parametrize("eta", ETAS)
@pytest.mark.parametrize("where", ["device", "host"])
def test_sweep_f64_bit_exact(ctx, golden_sweep, name, eta, where):
    g = golden_sweep
    set_golden_domain(ctx, g, name)
    params = g[f"{name}/params"]
    key = f"{name}/eta{eta}"
    pmax = float(g[key + "/pmax"][0])
    arg = torch.from_numpy(params).cuda() if where == "device" else params
    r = ctx.brute_force_config_exact(arg, eta, pmax)
    r = {k: (v.cpu().numpy() if isinstance(v, torch.Tensor) else v) for k, v in r.items()}
    np.testing.assert_array_equal(r["kstatus"], g[key + "/kstatus"])
    ok = r["kstatus"] == 0
    np.testing.assert_array_equal(r["idx"][ok], g[key + "/idx"][ok])
    for f in ("cost", "energy", "time"):
        np.testing.assert_array_equal(r[f][ok], g[key + "/" + f][ok])


def test_sweep_large_vs_reference(ctx, ref):
    """200k generated kernels on the 128x4 grid against the reference itself."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    n = 200_000
    gen = ctx.gen_synthetic(n, root=0xD50B203, counts=False, dcgm=False)
    p32 = np.ascontiguousarray(gen["params"].cpu().numpy().T.astype(np.float64))
    dev = dom.dev.as_array()
    for eta in (0.0, 0.5, 0.8, 1.0):
        r = ctx.brute_force_config(gen["params"], eta)
        want = ref.brute_force_config(p32, dom.core_freqs_mhz, dom.mem_freqs_mhz, dev, eta,
                                      dom.dev.pmax_w)
        idx = r["idx"].cpu().numpy()
        nbad, gap = check_argmin(p32, idx, want["idx"], dom.core_freqs_mhz, dom.mem_freqs_mhz,
                                 dev, eta, dom.dev.pmax_w)
        assert nbad <= n * 1e-3
        same = idx == want["idx"]
        for f in ("cost", "energy", "time"):
            assert rel_err(r[f].cpu().numpy()[same], want[f][same]).max() <= 1e-5
        e = ctx.brute_force_config_exact(torch.from_numpy(p32).cuda(), eta)
        np.testing.assert_array_equal(e["idx"].cpu().numpy(), want["idx"])
        np.testing.assert_array_equal(e["cost"].cpu().numpy(), want["cost"])


def test_eta_sweep_matches_single_eta(ctx, ref):
    """C4 shape on a slice: 101 etas in one pass == dso_sweep per eta, bit for bit."""
    dom = config_domain("c4")
    ctx.set_domain(dom)
    n = 20_000
    gen = ctx.gen_synthetic(n, root=0xD50B204, counts=False, dcgm=False)
    etas = np.arange(101) / 100.0
    idx, cost = ctx.eta_sweep(gen["params"], etas)
    idx, cost = idx.cpu().numpy(), cost.cpu().numpy()
    p32 = np.ascontiguousarray(gen["params"].cpu().numpy().T.astype(np.float64))
    for e in (0, 1, 17, 50, 80, 99, 100):
        r = ctx.brute_force_config(gen["params"], float(etas[e]))
        np.testing.assert_array_equal(idx[e], r["idx"].cpu().numpy())
        np.testing.assert_array_equal(cost[e], r["cost"].cpu().numpy())
    for e in (0, 33, 80, 100):
        want = ref.brute_force_config(p32, dom.core_freqs_mhz, dom.mem_freqs_mhz,
                                      dom.dev.as_array(), float(etas[e]), dom.dev.pmax_w)
        check_argmin(p32, idx[e], want["idx"], dom.core_freqs_mhz, dom.mem_freqs_mhz,
                     dom.dev.as_array(), float(etas[e]), dom.dev.pmax_w)


def test_shards_equal_whole(ctx):
    """Kernel sharding: slices passed as base+offset with the batch ld give
    bit-identical results (the multi-GPU contract)."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    n = 50_001
    gen = ctx.gen_synthetic(n, root=7, counts=False, dcgm=False)
    whole = ctx.brute_force_config(gen["params"], 0.8)
    bounds = [0, 12_345, 30_000, n]
    for a, b in zip(bounds, bounds[1:]):
        sl = gen["params"][:, a:].contiguous()  # ld changes; values identical
        part = ctx.brute_force_config(sl, 0.8, n=b - a)
        np.testing.assert_array_equal(part["idx"].cpu().numpy()[:b - a],
                                      whole["idx"].cpu().numpy()[a:b])


def test_sweep_errors(ctx):
    ctx.set_domain(config_domain("c1"))
    p = soa([[10.0, 5.0, 2.0, 3.0, 1.0, 8.0, 6.0]])
    for eta in (1.5, -0.1, float("nan")):
        with pytest.raises(DsoError) as e:
            ctx.brute_force_config(p, eta)
        assert e.value.kind == ErrorKind.EtaOutOfRange
    with pytest.raises(DsoError) as e:
        ctx.brute_force_config(p.double(), 0.5)
    assert e.value.kind == ErrorKind.InvalidArgument
    bad = DvfsDomain([900.0, 900.0], [438.0])
    with pytest.raises(DsoError) as e:
        ctx.set_domain(bad)
    assert e.value.kind == ErrorKind.InvalidArgument
    r = ctx.brute_force_config(soa(np.zeros((0, 7)), ld=1), 0.5, n=0)
    assert r["idx"].shape[0] == 1


def _tie_params(rng, n):
    """Random params plus kernels built to tie: equal costs across core levels
    (kp = c = g = b = 0), coarse values, zeros, huge and non-finite entries."""
    base = np.column_stack([rng.uniform(40, 90, n), rng.uniform(5, 15, n),
                            rng.uniform(0.004, 0.02, n), rng.uniform(0.002, 0.0055, n),
                            rng.uniform(0.04, 0.3, n), rng.uniform(40, 400, n),
                            rng.uniform(40, 400, n)])
    q = n // 8
    base[:q, [1, 2, 3, 6]] = 0.0                       # cost constant along fc
    base[q:2 * q] = np.round(base[q:2 * q])            # coarse values
    base[2 * q:3 * q, 0:4] = 0.0                       # P == 0 -> C = K*T
    base[3 * q:3 * q + 8, 5] = 3e13                    # beyond the fast-path bound
    base[3 * q + 8:3 * q + 16, 4] = np.inf
    base[3 * q + 16:3 * q + 24, 0] = np.nan
    base[3 * q + 24:3 * q + 32, 1] = -1.0              # invalid -> kstatus
    return base


@pytest.mark.parametrize("name", ["toy", "c1", "c1_literal", "c2", "c3", "grid10x10"])
def test_fast_sweep_bit_identical(ctx, golden_sweep, name):
    """The group-minimum sweep (default) equals the pair-by-pair lexicographic
    scan bit for bit: idx, cost, energy, time, kstatus — including exact ties."""
    g = golden_sweep
    set_golden_domain(ctx, g, name)
    rng = np.random.default_rng(11)
    params = np.concatenate([g[f"{name}/params"], _tie_params(rng, 40_000)])
    p = soa(params)
    try:
        for eta in (0.0, 0.3, 0.8, 1.0):
            ctx.set_option("fast_sweep", 1)
            a = {k: v.cpu().numpy() for k, v in ctx.brute_force_config(p, eta).items()}
            ctx.set_option("fast_sweep", 0)
            b = {k: v.cpu().numpy() for k, v in ctx.brute_force_config(p, eta).items()}
            for k in ("idx", "kstatus"):
                np.testing.assert_array_equal(a[k], b[k], err_msg=f"{k} eta={eta}")
            for k in ("cost", "energy", "time"):
                np.testing.assert_array_equal(a[k].view(np.uint32), b[k].view(np.uint32),
                                              err_msg=f"{k} eta={eta}")
    finally:
        ctx.set_option("fast_sweep", 1)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "grid10x10"])
def test_fast_eta_sweep_bit_identical(ctx, golden_sweep, name):
    g = golden_sweep
    set_golden_domain(ctx, g, name)
    rng = np.random.default_rng(12)
    params = np.concatenate([g[f"{name}/params"], _tie_params(rng, 8_000)])
    p = soa(params)
    etas = np.arange(101) / 100.0
    try:
        ctx.set_option("fast_sweep", 1)
        ia, ca = (x.cpu().numpy() for x in ctx.eta_sweep(p, etas))
        ctx.set_option("fast_sweep", 0)
        ib, cb = (x.cpu().numpy() for x in ctx.eta_sweep(p, etas))
    finally:
        ctx.set_option("fast_sweep", 1)
    np.testing.assert_array_equal(ia, ib)
    np.testing.assert_array_equal(ca.view(np.uint32), cb.view(np.uint32))
    # and each row equals the single-eta sweep
    for e in (0, 7, 50, 100):
        r = ctx.brute_force_config(p, float(etas[e]))
        np.testing.assert_array_equal(ia[e], r["idx"].cpu().numpy())


def _eta_runs(ctx, p, etas, opts):
    out = []
    try:
        for fast, prune in opts:
            ctx.set_option("fast_sweep", fast)
            ctx.set_option("eta_prune", prune)
            i, c = (x.cpu().numpy() for x in ctx.eta_sweep(p, etas))
            out.append((i, c.view(np.uint32)))
    finally:
        ctx.set_option("fast_sweep", 1)
        ctx.set_option("eta_prune", 1)
    return out


@pytest.mark.parametrize("dom", ["c4", "nm2", "nm3", "tail", "close"])
def test_pruned_eta_sweep_bit_identical(ctx, dom):
    """The pruned eta sweep (candidate set of nc + nm points, sweep.cu) equals the
    unpruned group-minimum sweep and the pair-by-pair scan bit for bit (domains
    are strictly increasing by validate(DvfsDomain); "close" has levels whose f32
    tables are equal), with tie-built, huge, non-finite and invalid params among
    realistic ones."""
    base = config_domain("c4")
    core, mem, dev = base.core_freqs_mhz, base.mem_freqs_mhz, base.dev
    if dom == "close":                   # adjacent levels whose f32 tables coincide
        core = np.sort(np.concatenate([core[:60], core[:60] * (1 + 1e-9)]))
        mem = np.array([mem[0], mem[0] * (1 + 1e-9), mem[2]])
    elif dom == "nm2":
        mem = mem[:2].copy()
    elif dom == "nm3":
        core, mem = core[::3].copy(), mem[:3].copy()
    elif dom == "tail":                  # nc not a multiple of the 8-level group
        core = core[:77].copy()
    ctx.set_domain(DvfsDomain(core, mem, dev))
    rng = np.random.default_rng(21)
    gen = ctx.gen_synthetic(6_000, root=0xD50B204, counts=False, dcgm=False)
    params = np.concatenate([gen["params"].cpu().numpy().T.astype(np.float64),
                             _tie_params(rng, 6_000)])
    p = soa(params)
    etas = np.concatenate([np.arange(101) / 100.0, [0.0, 1.0, 0.55]])
    runs = _eta_runs(ctx, p, etas, [(1, 1), (1, 0), (0, 0)])
    for i, c in runs[1:]:
        np.testing.assert_array_equal(runs[0][0], i)
        np.testing.assert_array_equal(runs[0][1], c)


def test_set_option_errors(ctx):
    with pytest.raises(DsoError) as e:
        ctx.set_option("no_such_option", 1)
    assert e.value.kind == ErrorKind.InvalidArgument
