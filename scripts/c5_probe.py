"""C5 gradient timing: the batch as a slice of the 10M-sample dataset (ld = 10M) vs a
compact copy (ld = 65,536), CUDA events over back-to-back calls (experiment script)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_13096_b200 import init_mlp, linear_domain  # noqa: E402
from paper_2407_13096_b200.api import Context  # noqa: E402

ctx = Context(0)
ctx.set_domain(linear_domain(128, 4))
m = init_mlp(seed=424242)
m.target_mean = np.array([60, 10, 0.01, 0.004, 0.15, 200, 200.0])
m.target_std = np.array([15, 3, 0.005, 0.001, 0.07, 100, 100.0])
ctx.set_model(m)
N, B = 10_000_000, 65536
g = ctx.gen_synthetic(N, root=0xACCE5505)
x = ctx.featurize(g["counts"], g["dcgm"])
del g
y = torch.randn((7, N), device="cuda")
xs, ys = x[:, :B].contiguous(), y[:, :B].contiguous()
grad = torch.empty((ctx.n_model_params,), device="cuda")


def t(fn, reps=20):
    for _ in range(3):
        fn()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


for tc in (1, 0):
    ctx.set_option("train_tc", tc)
    print(f"train_tc={tc}: slice of ld=10M {t(lambda: ctx.train_grad_slice(x, y, 0, B, grad=grad)):.3f} ms, "
          f"compact ld=65536 {t(lambda: ctx.train_grad(xs, ys, grad=grad)):.3f} ms", flush=True)
