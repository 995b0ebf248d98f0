"""Small invocation of every device entry point, for compute-sanitizer runs."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2407_13096_b200 import config_domain, init_mlp  # noqa: E402
from paper_2407_13096_b200.api import Context  # noqa: E402

ctx = Context(0)
for cfg in ("c1", "c3"):
    ctx.set_domain(config_domain(cfg))
    m = init_mlp(seed=1)
    m.target_mean = np.array([60, 10, 0.01, 0.004, 0.15, 200, 200.0])
    m.target_std = np.array([15, 3, 0.005, 0.001, 0.07, 100, 100.0])
    ctx.set_model(m)
    for n in (1, 63, 64, 65, 127, 128, 129, 1000, 4099):
        g = ctx.gen_synthetic(n, root=n)
        f = ctx.featurize(g["counts"], g["dcgm"])
        for eng in (0, 1):  # both predictor engines (FMA pipe, tcgen05)
            ctx.set_option("mlp_engine", eng)
            ctx.predict_params(f, want_raw=True)
            ctx.pipeline(g["counts"], g["dcgm"], 0.8, want_params=True)
            gc = ctx.gen_synthetic_csr(n, root=n)
            ctx.pipeline_csr(gc["row_ptr"], gc["entries"], gc["dcgm"], 0.8, want_params=True)
        ctx.set_option("mlp_engine", 2)
        p, cl, raw = ctx.predict_params(f, want_raw=True)
        ctx.brute_force_config(p, 0.8)
        ctx.brute_force_config_exact(p.double().t().contiguous(), 0.8)
        ctx.eta_sweep(p, np.arange(11) / 10.0)
        ctx.pipeline(g["counts"], g["dcgm"], 0.8, want_params=True)
        y = torch.randn((7, n), device="cuda")
        gr, loss = ctx.train_grad(f, y)
        ctx.train_apply(gr, 0.01, 1.0 / n)
        ctx.dcgm_mean(torch.rand((3, 8, n), device="cuda", dtype=torch.float64))
# the tcgen05 engine's CSR producer on irregular rows: 0..70 slot-sorted entries
# (staged / global / general paths), empty rows at the end, misaligned entry arrays
rng = np.random.default_rng(3)
ctx.set_domain(config_domain("c3"))
for n in (5, 300, 1500):
    lens = rng.integers(0, 71, size=n)
    lens[-3:] = 0
    ents, rp = [], [0]
    for L in lens:
        sl = np.sort(rng.choice(126, size=int(L), replace=False))
        ents.extend(((rng.integers(1, 5000, size=int(L)) << 7) | sl).tolist())
        rp.append(len(ents))
    ent = np.array(ents, np.int64).astype(np.int32)
    for shift in (0, 1, 3):
        buf = torch.zeros(len(ent) + 4, dtype=torch.int32, device="cuda")
        buf[shift:shift + len(ent)] = torch.from_numpy(ent).cuda()
        ctx.set_option("mlp_engine", 1)
        ctx.pipeline_csr(torch.tensor(rp, dtype=torch.int64, device="cuda"), buf[shift:shift + len(ent)],
                         torch.rand((8, n), device="cuda"), 0.8, want_params=True)
ctx.set_option("mlp_engine", 2)
# per-context scratch in any call order (regression: the eta table's growth once
# freed the dcgm_mean flag), then destroy
c2 = Context(0)
c2.set_domain(config_domain("c3"))
s = torch.rand((4, 8, 257), device="cuda", dtype=torch.float64)
c2.dcgm_mean(s)
pp = c2.gen_synthetic(1000, root=5, counts=False, dcgm=False)["params"]
c2.eta_sweep(pp, np.arange(5) / 4.0)
c2.dcgm_mean(s)
c2.eta_sweep(pp, np.arange(101) / 100.0)
c2.dcgm_mean(s)
c2.close()
torch.cuda.synchronize()
print("sanitize run ok")
