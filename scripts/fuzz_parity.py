"""Randomised parity sweep of the round-2 device paths (evidence script, GPU).

Each trial draws a random domain / batch and checks, bit for bit:
  * eta sweep: pruned kernel == unpruned group-minimum kernel == pair-by-pair scan
    (random ascending domains with 2-4 memory levels and 8-256 core levels, random
    eta lists, synthetic + tie-built params);
  * dense counts -> one-pass CSR compaction -> pipeline == pipeline_csr on the same
    kernels (random sizes, random row densities 0..126);
and, within tolerance, the tensor-core weight gradient against the FMA-pipe one
(random batch sizes, including partial 16-sample stages).
Prints one line per trial and a summary; exits non-zero on any mismatch.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_13096_b200 import DvfsDomain, default_device, init_mlp  # noqa: E402
from paper_2407_13096_b200.api import Context  # noqa: E402

rng = np.random.default_rng(int(os.environ.get("FUZZ_SEED", "20261017")))
trials = int(os.environ.get("FUZZ_TRIALS", "20"))
ctx = Context(0)
fails = 0


def soa(params):
    t = torch.from_numpy(np.ascontiguousarray(params.T.astype(np.float32))).cuda()
    return t


def rand_domain():
    dev = default_device()
    nc = int(rng.integers(8, 257))
    nm = int(rng.integers(2, 5))
    core = np.unique(np.round(np.sort(rng.uniform(705.0, 1380.0, nc)), 3))  # the benchmark range
    mem = np.unique(np.round(np.sort(rng.uniform(438.0, 877.0, nm)), 3))
    return DvfsDomain(core, mem, dev)


def tie_params(n):
    p = np.column_stack([rng.uniform(40, 90, n), rng.uniform(5, 15, n), rng.uniform(0.004, 0.02, n),
                         rng.uniform(0.002, 0.0055, n), rng.uniform(0.04, 0.3, n),
                         rng.uniform(40, 400, n), rng.uniform(40, 400, n)])
    q = n // 6
    p[:q, [1, 2, 3, 6]] = 0.0
    p[q:2 * q] = np.round(p[q:2 * q])
    p[2 * q:3 * q, 0:4] = 0.0
    return p


for t in range(trials):
    # ---- eta sweep --------------------------------------------------------------
    dom = rand_domain()
    ctx.set_domain(dom)
    n = int(rng.integers(1000, 20000))
    gen = ctx.gen_synthetic(n, root=int(rng.integers(1, 1 << 30)), counts=False, dcgm=False)
    params = np.concatenate([gen["params"].cpu().numpy().T.astype(np.float64), tie_params(2000)])
    p = soa(params)
    ne = int(rng.integers(1, 120))
    etas = np.sort(rng.uniform(0, 1, ne))
    etas[rng.integers(0, ne)] = 0.0
    out = []
    for fast, prune in ((1, 1), (1, 0), (0, 0)):
        ctx.set_option("fast_sweep", fast)
        ctx.set_option("eta_prune", prune)
        i, c = ctx.eta_sweep(p, etas)
        out.append((i.cpu().numpy(), c.cpu().numpy().view(np.uint32)))
    ctx.set_option("fast_sweep", 1)
    ctx.set_option("eta_prune", 1)
    ok_eta = all(np.array_equal(out[0][0], o[0]) and np.array_equal(out[0][1], o[1]) for o in out[1:])
    # ---- dense -> CSR compaction ---------------------------------------------------
    m = int(rng.integers(1, 40000))
    dens = rng.uniform(0, 1)
    counts = np.zeros((m, 126), np.uint32)
    nnz = rng.binomial(126, dens * 0.9, size=m)
    for k in range(m):
        if nnz[k]:
            counts[k, rng.choice(126, size=int(nnz[k]), replace=False)] = rng.integers(1, 1 << 22, size=int(nnz[k]))
    dcgm = torch.from_numpy(np.ascontiguousarray(rng.uniform(0, 1, (8, m)).astype(np.float32))).cuda()
    ct = torch.from_numpy(np.ascontiguousarray(counts.T).view(np.int32)).cuda()
    mdl = init_mlp(seed=int(rng.integers(1, 1000)))
    mdl.target_mean = np.array([60, 10, 0.01, 0.004, 0.15, 200, 200.0])
    mdl.target_std = np.array([15, 3, 0.005, 0.001, 0.07, 100, 100.0])
    ctx.set_model(mdl)
    a = ctx.pipeline(ct, dcgm, 0.6, want_params=True)
    rp = np.zeros(m + 1, np.int64)
    rp[1:] = np.cumsum((counts != 0).sum(axis=1))
    ks, ss = np.nonzero(counts)
    ent = ((counts[ks, ss].astype(np.uint64) << 7) | ss.astype(np.uint64)).astype(np.uint32)
    b = ctx.pipeline_csr(torch.from_numpy(rp).cuda(), torch.from_numpy(ent.view(np.int32)).cuda(),
                         dcgm, 0.6, want_params=True)
    ok_dense = all(np.array_equal(a[f].cpu().numpy(), b[f].cpu().numpy())
                   for f in ("idx", "cost", "params"))
    # ---- tensor-core weight gradient vs FMA pipe -------------------------------------
    B = int(rng.integers(1, 9000))
    x = torch.rand((134, B), device="cuda")
    y = torch.randn((7, B), device="cuda")
    ctx.set_option("train_tc", 1)
    g1, l1 = ctx.train_grad(x, y)
    ctx.set_option("train_tc", 0)
    g0, l0 = ctx.train_grad(x, y)
    ctx.set_option("train_tc", 1)
    g1, g0 = g1.double().cpu().numpy(), g0.double().cpu().numpy()
    err = float(np.abs(g1 - g0).max() / max(np.abs(g0).max(), 1e-30))
    ok_train = err <= 2e-5 and abs(float(l1) - float(l0)) <= 1e-9 * max(1.0, abs(float(l0)))
    ok = ok_eta and ok_dense and ok_train
    fails += 0 if ok else 1
    print(f"trial {t:2d}: eta nc={dom.nc} nm={dom.nm} n={len(params)} n_eta={ne} -> {ok_eta}; "
          f"dense m={m} density={dens:.2f} -> {ok_dense}; train B={B} rel.err={err:.2e} -> {ok_train}",
          flush=True)
print(f"fuzz parity: {trials - fails}/{trials} trials passed")
sys.exit(1 if fails else 0)
