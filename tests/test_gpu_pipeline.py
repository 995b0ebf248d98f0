"""GPU parity: the fused pipeline (counts + DCGM -> features -> MLP -> sweep ->
argmin) vs the oracle pipeline (featurize + predict_params + brute_force_config
in double), and vs its own stage-by-stage composition (bit-exact)."""

import numpy as np
import pytest
import torch

from helpers import check_argmin, check_index_rule, rel_err
from paper_2407_13096_b200 import config_domain, init_mlp

pytestmark = [pytest.mark.gpu, pytest.mark.usefixtures("engine")]


def stats_model(port, seed=424242):
    m = init_mlp(seed=seed)
    params = port.gen_stream(0xC0FFEE, 4096, want=("params",))["params"]
    mean, std, _ = port.target_stats(params)
    m.target_mean, m.target_std = mean, std
    return m


@pytest.mark.parametrize("cfg", ["c1", "c1_literal", "c2", "c3"])
def test_pipeline_vs_oracle(ctx, port, cfg):
    dom = config_domain(cfg)
    ctx.set_domain(dom)
    m = stats_model(port)
    ctx.set_model(m)
    n = 20_000 + 3
    g = ctx.gen_synthetic(n, root=0xD50B200 + len(cfg), params=False)
    eta = 0.8
    out = ctx.pipeline(g["counts"], g["dcgm"], eta, want_params=True)
    counts = g["counts"].cpu().numpy().T.view(np.uint32)
    dcgm = g["dcgm"].cpu().numpy().T.astype(np.float64)
    dev = dom.dev.as_array()
    st, want = port.pipeline(counts, dcgm, m, dom.core_freqs_mhz, dom.mem_freqs_mhz, dev, eta,
                             dom.dev.pmax_w)
    assert st == 0
    p = out["params"].cpu().numpy().T.astype(np.float64)
    tol = 1e-5 * np.abs(want["params"]) + 1e-6 * m.target_std[None, :]
    assert (np.abs(p - want["params"]) <= tol).all()
    idx = out["idx"].cpu().numpy()
    # the GPU's choice must be optimal (to 1e-6) for the parameters it predicted ...
    r = port.brute_force(p, dom.core_freqs_mhz, dom.mem_freqs_mhz, dev, eta, dom.dev.pmax_w)[1]
    check_argmin(p, idx, r["idx"], dom.core_freqs_mhz, dom.mem_freqs_mhz, dev, eta,
                 dom.dev.pmax_w)
    # ... and agree with the all-double oracle pipeline except on near-ties, the
    # oracle-side gap at every mismatch bounded by the parameter error (helpers)
    rule = check_index_rule(p, want["params"], idx, want["idx"], dom.core_freqs_mhz,
                            dom.mem_freqs_mhz, dev, eta, dom.dev.pmax_w)
    print(f"index rule {cfg}: {rule}")
    same = idx == want["idx"]
    for f in ("cost", "energy", "time"):
        assert rel_err(out[f].cpu().numpy()[same], want[f][same]).max() <= 2e-5


def test_pipeline_equals_staged_kernels(ctx, port):
    dom = config_domain("c3")
    ctx.set_domain(dom)
    ctx.set_model(stats_model(port))
    n = 30_001
    g = ctx.gen_synthetic(n, root=17, params=False)
    fused = ctx.featurize(g["counts"], g["dcgm"])
    params, clamped, _ = ctx.predict_params(fused)
    staged = ctx.brute_force_config(params, 0.8)
    out = ctx.pipeline(g["counts"], g["dcgm"], 0.8, want_params=True)
    np.testing.assert_array_equal(out["params"].cpu().numpy(), params.cpu().numpy())
    np.testing.assert_array_equal(out["clamped"].cpu().numpy().astype(bool), clamped.cpu().numpy())
    for f in ("idx", "cost", "energy", "time"):
        np.testing.assert_array_equal(out[f].cpu().numpy(), staged[f].cpu().numpy())


def test_pipeline_host_buffers_equal_device(ctx, port):
    """DSO_HOST: pinned host in, host out, chunked + overlapped inside the call."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    ctx.set_model(stats_model(port))
    n = (1 << 20) + 12_345  # more than one staging chunk
    g = ctx.gen_synthetic(n, root=23, params=False)
    dev_out = ctx.pipeline(g["counts"], g["dcgm"], 0.5, want_params=True)
    hc = g["counts"].cpu().pin_memory()
    hd = g["dcgm"].cpu().pin_memory()
    host_out = ctx.pipeline(hc, hd, 0.5, want_params=True)
    for f in ("idx", "cost", "energy", "time", "params", "clamped"):
        np.testing.assert_array_equal(host_out[f].numpy(), dev_out[f].cpu().numpy())


def test_pipeline_shards_equal_whole(ctx, port):
    dom = config_domain("c2")
    ctx.set_domain(dom)
    ctx.set_model(stats_model(port))
    n = 10_000
    g = ctx.gen_synthetic(n, root=31, params=False)
    whole = ctx.pipeline(g["counts"], g["dcgm"], 0.8)
    # shards generated independently with `first` offsets == slices of the whole
    for a, b in ((0, 3333), (3333, 7000), (7000, n)):
        part = ctx.gen_synthetic(b - a, root=31, first=a, params=False)
        r = ctx.pipeline(part["counts"], part["dcgm"], 0.8)
        np.testing.assert_array_equal(r["idx"].cpu().numpy(), whole["idx"].cpu().numpy()[a:b])
        np.testing.assert_array_equal(r["cost"].cpu().numpy(), whole["cost"].cpu().numpy()[a:b])


# ---- sparse (CSR) input ---------------------------------------------------------------
def csr_from_dense(counts, rng=None, dup=False):
    """counts [n, 126] uint32 -> (row_ptr, entries) with entries (count << 7) | slot."""
    rp, ent = [0], []
    for k, row in enumerate(counts):
        nz = np.flatnonzero(row)
        items = [(int(row[s]) << 7) | int(s) for s in nz]
        if dup and len(nz):  # split the first count over two entries (duplicates add)
            s0 = int(nz[0])
            c0 = int(row[s0])
            items[0] = ((c0 // 2) << 7) | s0
            items.append(((c0 - c0 // 2) << 7) | s0)
        if rng is not None:
            rng.shuffle(items)
        ent.extend(items)
        rp.append(len(ent))
    return np.array(rp, np.int64), np.array(ent, np.uint32)


def test_gen_csr_matches_dense(ctx):
    n = 5000
    d = ctx.gen_synthetic(n, root=41, params=False)
    s = ctx.gen_synthetic_csr(n, root=41)
    np.testing.assert_array_equal(s["dcgm"].cpu().numpy(), d["dcgm"].cpu().numpy())
    rp = s["row_ptr"].cpu().numpy()
    ent = s["entries"].cpu().numpy().view(np.uint32)
    assert (rp == 24 * np.arange(n + 1)).all()
    dense = np.zeros((n, 126), np.uint64)
    for k in range(n):
        for e in ent[rp[k]:rp[k + 1]]:
            dense[k, e & 127] += e >> 7
    np.testing.assert_array_equal(dense, d["counts"].cpu().numpy().T.view(np.uint32))


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3"])
def test_pipeline_csr_equals_dense(ctx, port, cfg):
    dom = config_domain(cfg)
    ctx.set_domain(dom)
    ctx.set_model(stats_model(port))
    n = 20_000 + 37
    d = ctx.gen_synthetic(n, root=43, params=False)
    s = ctx.gen_synthetic_csr(n, root=43)
    a = ctx.pipeline(d["counts"], d["dcgm"], 0.8, want_params=True)
    b = ctx.pipeline_csr(s["row_ptr"], s["entries"], s["dcgm"], 0.8, want_params=True)
    for f in ("idx", "cost", "energy", "time", "params", "clamped"):
        np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())


def test_pipeline_csr_irregular(ctx, port):
    """Random sparsity (0..126 non-zeros per kernel, > 32 exercises the spill
    path), shuffled entry order, duplicate slots, empty kernels, ragged tail,
    a non-zero ent_base — all equal to the dense pipeline bit for bit."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    ctx.set_model(stats_model(port))
    rng = np.random.default_rng(7)
    n = 3000 + 13
    counts = np.zeros((n, 126), np.uint32)
    for k in range(n):
        nnz = int(rng.integers(0, 127)) if k % 5 else int(rng.integers(0, 8))
        slots = rng.choice(126, size=nnz, replace=False)
        counts[k, slots] = rng.integers(1, 200_000, size=nnz)
    counts[10] = 0
    dcgm = rng.uniform(0, 1, size=(n, 8)).astype(np.float32)
    rp, ent = csr_from_dense(counts, rng=rng, dup=True)
    base = 1000
    ent_pad = np.concatenate([np.zeros(base, np.uint32), ent])
    rp_t = torch.from_numpy(rp + base).cuda()
    ent_t = torch.from_numpy(ent.view(np.int32)).cuda()  # points at global index `base`
    dc_t = torch.from_numpy(np.ascontiguousarray(dcgm.T)).cuda()
    b = ctx.pipeline_csr(rp_t, ent_t, dc_t, 0.5, ent_base=base, want_params=True)
    a = ctx.pipeline(torch.from_numpy(np.ascontiguousarray(counts.T).view(np.int32)).cuda(), dc_t,
                     0.5, want_params=True)
    for f in ("idx", "cost", "energy", "time", "params", "clamped"):
        np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())
    # host buffers (chunked path) give the same answers
    h = ctx.pipeline_csr(torch.from_numpy(rp).pin_memory(),
                         torch.from_numpy(ent.view(np.int32)).pin_memory(),
                         torch.from_numpy(np.ascontiguousarray(dcgm.T)).pin_memory(), 0.5,
                         want_params=True)
    for f in ("idx", "cost", "energy", "time", "params", "clamped"):
        np.testing.assert_array_equal(h[f].numpy(), a[f].cpu().numpy())
    del ent_pad


def test_pipeline_csr_sorted_random_slots(ctx, port):
    """Slot-sorted entries over all 126 categories (each engine's fast path, incl.
    the tcgen05 engine's reordered layer-1 columns), equal to the dense pipeline."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    ctx.set_model(stats_model(port))
    rng = np.random.default_rng(8)
    n = 4096 + 5
    counts = np.zeros((n, 126), np.uint32)
    for k in range(n):
        nnz = int(rng.integers(1, 25))
        slots = rng.choice(126, size=nnz, replace=False)
        counts[k, slots] = rng.integers(1, 300_000, size=nnz)
    dcgm = rng.uniform(0, 1, size=(n, 8)).astype(np.float32)
    rp, ent = csr_from_dense(counts)
    dc_t = torch.from_numpy(np.ascontiguousarray(dcgm.T)).cuda()
    b = ctx.pipeline_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(ent.view(np.int32)).cuda(),
                         dc_t, 0.5, want_params=True)
    a = ctx.pipeline(torch.from_numpy(np.ascontiguousarray(counts.T).view(np.int32)).cuda(), dc_t,
                     0.5, want_params=True)
    for f in ("idx", "cost", "energy", "time", "params", "clamped"):
        np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())


def test_pipeline_csr_long_sorted_rows(ctx, port):
    """Slot-sorted rows of 20..70 entries (the tcgen05 engine's two-pass producer for
    any row up to 64 entries, the general path beyond; tiles over the shared-memory
    stage read from global), entry arrays starting 1..3 words past a 16-byte
    boundary — equal to the dense pipeline bit for bit."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    ctx.set_model(stats_model(port))
    rng = np.random.default_rng(9)
    n = 6000 + 7
    counts = np.zeros((n, 126), np.uint32)
    for k in range(n):
        nnz = int(rng.integers(20, 71)) if k < 3000 else int(rng.integers(20, 31))
        slots = rng.choice(126, size=nnz, replace=False)
        counts[k, slots] = rng.integers(1, 120_000, size=nnz)
    dcgm = rng.uniform(0, 1, size=(n, 8)).astype(np.float32)
    rp, ent = csr_from_dense(counts)
    dc_t = torch.from_numpy(np.ascontiguousarray(dcgm.T)).cuda()
    a = ctx.pipeline(torch.from_numpy(np.ascontiguousarray(counts.T).view(np.int32)).cuda(), dc_t,
                     0.5, want_params=True)
    for shift in (0, 1, 2, 3):
        buf = torch.zeros(len(ent) + 8, dtype=torch.int32, device="cuda")
        buf[shift:shift + len(ent)] = torch.from_numpy(ent.view(np.int32)).cuda()
        b = ctx.pipeline_csr(torch.from_numpy(rp).cuda(), buf[shift:shift + len(ent)], dc_t, 0.5,
                             want_params=True)
        for f in ("idx", "cost", "energy", "time", "params", "clamped"):
            np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())


def test_pipeline_dense_via_csr(ctx, port):
    """Auto engine, dense counts on the device: compacted to CSR and run on the
    tensor-core CSR pipeline — equal to pipeline_csr on the same kernels bit for bit
    (synthetic stream with a ragged tail, random rows over all 126 slots); a count
    >= 2^25 (outside the CSR field) falls back to the dense kernels."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    ctx.set_model(stats_model(port))
    ctx.set_option("mlp_engine", 2)
    try:
        n = 20_000 + 37
        d = ctx.gen_synthetic(n, root=43, params=False)
        s = ctx.gen_synthetic_csr(n, root=43)
        a = ctx.pipeline(d["counts"], d["dcgm"], 0.8, want_params=True)
        b = ctx.pipeline_csr(s["row_ptr"], s["entries"], s["dcgm"], 0.8, want_params=True)
        for f in ("idx", "cost", "energy", "time", "params", "clamped"):
            np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())
        rng = np.random.default_rng(21)
        m = 5000 + 3
        counts = np.zeros((m, 126), np.uint32)
        for k in range(m):
            nnz = int(rng.integers(0, 60))
            counts[k, rng.choice(126, size=nnz, replace=False)] = rng.integers(1, 1 << 20, size=nnz)
        dcgm = torch.from_numpy(np.ascontiguousarray(rng.uniform(0, 1, (8, m)).astype(np.float32))).cuda()
        ct = torch.from_numpy(np.ascontiguousarray(counts.T).view(np.int32)).cuda()
        a = ctx.pipeline(ct, dcgm, 0.5, want_params=True)
        rp, ent = csr_from_dense(counts)
        b = ctx.pipeline_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(ent.view(np.int32)).cuda(),
                             dcgm, 0.5, want_params=True)
        for f in ("idx", "cost", "energy", "time", "params", "clamped"):
            np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())
        counts[7, 3] = 1 << 26  # outside the CSR count field
        ct = torch.from_numpy(np.ascontiguousarray(counts.T).view(np.int32)).cuda()
        a = ctx.pipeline(ct, dcgm, 0.5, want_params=True)
        ctx.set_option("dense_csr", 0)
        b = ctx.pipeline(ct, dcgm, 0.5, want_params=True)
        for f in ("idx", "cost", "energy", "time", "params", "clamped"):
            np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())
    finally:
        ctx.set_option("dense_csr", 1)
        ctx.set_option("mlp_engine", 2)


def test_pipeline_csr_host_large(ctx, port):
    dom = config_domain("c3")
    ctx.set_domain(dom)
    ctx.set_model(stats_model(port))
    n = (1 << 21) + 4321  # more than one host chunk
    s = ctx.gen_synthetic_csr(n, root=47)
    dev_out = ctx.pipeline_csr(s["row_ptr"], s["entries"], s["dcgm"], 0.8, want_params=True)
    host_out = ctx.pipeline_csr(s["row_ptr"].cpu().pin_memory(), s["entries"].cpu().pin_memory(),
                                s["dcgm"].cpu().pin_memory(), 0.8, want_params=True)
    for f in ("idx", "cost", "energy", "time", "params", "clamped"):
        np.testing.assert_array_equal(host_out[f].numpy(), dev_out[f].cpu().numpy())


def test_pipeline_csr_nonfinite_weight_disables_row_skipping(ctx, port):
    """The CSR path skips all-zero input rows of a tile (exact for finite W1).
    An infinite W1 entry on an absent slot makes the reference's product
    inf * 0 = NaN, so the skip must switch off: CSR == dense, NaNs included."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    m = stats_model(port)
    n = 4096 + 5
    d = ctx.gen_synthetic(n, root=53, params=False)
    counts = d["counts"].cpu().numpy().T.view(np.uint32)
    absent = int(np.flatnonzero(counts.sum(axis=0) == 0)[0])  # a slot no kernel uses
    m.weights[0] = m.weights[0].copy()
    m.weights[0][3, 8 + absent] = np.inf  # neuron 3, fused row 8 + slot
    ctx.set_model(m)
    s = ctx.gen_synthetic_csr(n, root=53)
    a = ctx.pipeline(d["counts"], d["dcgm"], 0.8, want_params=True)
    b = ctx.pipeline_csr(s["row_ptr"], s["entries"], s["dcgm"], 0.8, want_params=True)
    assert np.isnan(a["params"].cpu().numpy()).any() or (a["clamped"].cpu().numpy() != 0).any()
    for f in ("idx", "cost", "energy", "time", "params", "clamped"):
        np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())
    # finite again: skipping back on, still equal
    ctx.set_model(stats_model(port))
    a = ctx.pipeline(d["counts"], d["dcgm"], 0.8, want_params=True)
    b = ctx.pipeline_csr(s["row_ptr"], s["entries"], s["dcgm"], 0.8, want_params=True)
    for f in ("idx", "cost", "energy", "time", "params", "clamped"):
        np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())


@pytest.mark.parametrize("cfg", ["c2", "c3"])
def test_pipeline_fast_sweep_bit_identical(ctx, port, cfg):
    """The fused kernel's group-minimum sweep == the pair-by-pair scan, bit for bit."""
    dom = config_domain(cfg)
    ctx.set_domain(dom)
    ctx.set_model(stats_model(port))
    n = 50_000 + 7
    g = ctx.gen_synthetic_csr(n, root=0x5EED, first=3)
    outs = []
    try:
        for fast in (1, 0):
            ctx.set_option("fast_sweep", fast)
            for eta in (0.0, 0.8):
                o = ctx.pipeline_csr(g["row_ptr"], g["entries"], g["dcgm"], eta)
                outs.append({k: v.cpu().numpy() for k, v in o.items() if v is not None})
    finally:
        ctx.set_option("fast_sweep", 1)
    for a, b in zip(outs[:2], outs[2:]):
        for k in a:
            np.testing.assert_array_equal(a[k].view(np.uint8), b[k].view(np.uint8), err_msg=k)


# ---- north_star's index rule at scale: the benchmarked path vs the oracle --------------
def bench_model(ctx):
    """bench.py's model: init_mlp(default, 424242), target stats of 65,536 truth
    parameters of the 0xC0FFEE stream (population mean / std)."""
    m = init_mlp(seed=424242)
    p = ctx.gen_synthetic(65536, root=0xC0FFEE, counts=False, dcgm=False)["params"]
    p = p.double().cpu().numpy()
    m.target_mean, m.target_std = p.mean(1), p.std(1)
    return m


def pipeline_vs_oracle(ctx, port, m, dom, rp, ent, counts, dcgm, eta):
    """CSR pipeline on the device vs port.pipeline on the same kernels: params within
    1e-5 (+1e-6 std), the index rule at every mismatch, outputs at agreeing indices."""
    n = len(counts)
    dc_t = torch.from_numpy(np.ascontiguousarray(dcgm.T.astype(np.float32))).cuda()
    out = ctx.pipeline_csr(rp, ent, dc_t, eta, want_params=True)
    dev = dom.dev.as_array()
    st, want = port.pipeline(counts, dcgm.astype(np.float32).astype(np.float64), m,
                             dom.core_freqs_mhz, dom.mem_freqs_mhz, dev, eta, dom.dev.pmax_w)
    assert st == 0
    p = out["params"].cpu().numpy().T.astype(np.float64)
    tol = 1e-5 * np.abs(want["params"]) + 1e-6 * m.target_std[None, :]
    err = np.abs(p - want["params"])
    assert (err <= tol).all(), f"params outside tolerance at {np.argwhere(err > tol)[:5]}"
    idx = out["idx"].cpu().numpy()
    rule = check_index_rule(p, want["params"], idx, want["idx"], dom.core_freqs_mhz,
                            dom.mem_freqs_mhz, dev, eta, dom.dev.pmax_w)
    same = idx == want["idx"]
    for f in ("cost", "energy", "time"):
        assert rel_err(out[f].cpu().numpy()[same], want[f][same]).max() <= 2e-5, f
    return rule, out


def test_pipeline_csr_bench_stream_vs_oracle(ctx, port):
    """The exact benchmark workload (bench.py: root 0xD50B203, C3 128x4, eta 0.8, the
    bench model), 1,048,576 kernels through dso_pipeline_csr vs the oracle pipeline."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    m = bench_model(ctx)
    ctx.set_model(m)
    n = 1 << 20
    g = ctx.gen_synthetic_csr(n, root=0xD50B203)
    host = port.gen_stream(0xD50B203, n, want=("counts", "dcgm"))
    np.testing.assert_array_equal(g["dcgm"].cpu().numpy().T, host["dcgm"].astype(np.float32))
    rule, _ = pipeline_vs_oracle(ctx, port, m, dom, g["row_ptr"], g["entries"], host["counts"],
                                 host["dcgm"], 0.8)
    print(f"bench stream, {n} kernels: {rule}")
    assert rule["mismatches"] <= n // 1000


def realistic_counts(rng, n, lo=20, hi=30):
    """Kernels listing 20-30 of the 126 categories: a Zipf-like preference for the
    frequent opcodes / types / spaces, the rest spread over every slot; counts
    log-uniform in [1, 2e6] (totals straddle 2^24 now and then)."""
    w = 1.0 / (1.0 + np.arange(126)) ** 0.8
    w = w[rng.permutation(126)]
    w /= w.sum()
    counts = np.zeros((n, 126), np.uint32)
    nnz = rng.integers(lo, hi + 1, size=n)
    for k in range(n):
        slots = rng.choice(126, size=int(nnz[k]), replace=False, p=w)
        counts[k, slots] = np.exp(rng.uniform(0, np.log(2e6), size=len(slots))).astype(np.uint32) + 1
    return counts


def ptx_fixture_counts():
    """Per-kernel count histograms of the reference's PTX fixtures (tests/golden/ptx)."""
    import glob
    import os
    from paper_2407_13096_b200.ingest import parse_ptx
    rows = []
    for f in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "ptx", "*.ptx"))):
        for _name, c, _total in parse_ptx(open(f).read()):
            rows.append(np.asarray(c, np.uint32))
    return np.array(rows, np.uint32)


def test_pipeline_csr_realistic_mix_vs_oracle(ctx, port):
    """A realistic slot distribution (20-30 listed categories over all 126, not the
    generator's 24) plus the PTX fixtures' histograms scaled up: device vs oracle
    under the index rule, and CSR == dense bit for bit."""
    dom = config_domain("c3")
    ctx.set_domain(dom)
    m = bench_model(ctx)
    ctx.set_model(m)
    rng = np.random.default_rng(2407)
    n = 200_000
    counts = realistic_counts(rng, n)
    fx = ptx_fixture_counts()
    reps = rng.integers(1, 5000, size=(len(fx) * 64, 1)).astype(np.uint64)
    counts[: len(fx) * 64] = np.minimum(np.tile(fx, (64, 1)).astype(np.uint64) * reps,
                                        (1 << 25) - 1).astype(np.uint32)
    dcgm = rng.uniform(0, 1, size=(n, 8))
    rp, ent = csr_from_dense(counts)
    rp_t = torch.from_numpy(rp).cuda()
    ent_t = torch.from_numpy(ent.view(np.int32)).cuda()
    rule, out = pipeline_vs_oracle(ctx, port, m, dom, rp_t, ent_t, counts, dcgm, 0.8)
    print(f"realistic mix, {n} kernels: {rule}")
    assert rule["mismatches"] <= n // 1000
    dc_t = torch.from_numpy(np.ascontiguousarray(dcgm.T.astype(np.float32))).cuda()
    a = ctx.pipeline(torch.from_numpy(np.ascontiguousarray(counts.T).view(np.int32)).cuda(), dc_t,
                     0.8, want_params=True)
    for f in ("idx", "cost", "energy", "time", "params", "clamped"):
        np.testing.assert_array_equal(a[f].cpu().numpy(), out[f].cpu().numpy())


def test_dense_csr_regrow_and_many_blocks(port):
    """The one-pass dense -> CSR compaction on a fresh context: rows denser than
    the first entry-buffer guess (~32 per kernel) make it regrow and rerun, and
    a 300k-kernel stream spans ~1,200 look-back blocks; both equal pipeline_csr
    on the same kernels bit for bit."""
    from paper_2407_13096_b200.api import Context
    c = Context(0)
    try:
        c.set_domain(config_domain("c3"))
        c.set_model(stats_model(port))
        rng = np.random.default_rng(5)
        m = 3000 + 11
        counts = np.zeros((m, 126), np.uint32)
        for k in range(m):
            nnz = int(rng.integers(90, 127))
            counts[k, rng.choice(126, size=nnz, replace=False)] = rng.integers(1, 1 << 24, size=nnz)
        dcgm = torch.from_numpy(np.ascontiguousarray(rng.uniform(0, 1, (8, m)).astype(np.float32))).cuda()
        ct = torch.from_numpy(np.ascontiguousarray(counts.T).view(np.int32)).cuda()
        a = c.pipeline(ct, dcgm, 0.3, want_params=True)
        rp, ent = csr_from_dense(counts)
        b = c.pipeline_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(ent.view(np.int32)).cuda(),
                           dcgm, 0.3, want_params=True)
        for f in ("idx", "cost", "energy", "time", "params", "clamped"):
            np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())
        n = 300_000 + 5
        d = c.gen_synthetic(n, root=77, params=False)
        s = c.gen_synthetic_csr(n, root=77)
        a = c.pipeline(d["counts"], d["dcgm"], 0.8, want_params=True)
        b = c.pipeline_csr(s["row_ptr"], s["entries"], s["dcgm"], 0.8, want_params=True)
        for f in ("idx", "cost", "params"):
            np.testing.assert_array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())
    finally:
        c.close()
