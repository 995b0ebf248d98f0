import sys, torch, numpy as np
sys.path.insert(0, '.')
from paper_2407_13096_b200.api import Context
from paper_2407_13096_b200 import config_domain, init_mlp
ctx = Context(0); ctx.set_domain(config_domain("c3")); ctx.set_model(init_mlp(seed=1))
n = 1 << 22
g = ctx.gen_synthetic(n, root=3)
f = ctx.featurize(g["counts"], g["dcgm"])
for eng in (0, 1):
    ctx.set_option("mlp_engine", eng)
    for run in ("predict", "dense"):
        fn = (lambda: ctx.predict_params(f)) if run == "predict" else (lambda: ctx.pipeline(g["counts"], g["dcgm"], 0.8))
        fn(); torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): fn()
        e1.record(); torch.cuda.synchronize()
        print(f"engine {eng} {run}: {e0.elapsed_time(e1)/5:.3f} ms per 4M kernels")
