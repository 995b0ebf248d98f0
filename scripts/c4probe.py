import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
from paper_2407_13096_b200.api import Context
from paper_2407_13096_b200 import linear_domain
ctx = Context(0)
dom = linear_domain(128, 4)
ctx.set_domain(dom)
n = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 22
g = ctx.gen_synthetic(n, root=0xD50B204, counts=False, dcgm=False)
etas = np.arange(101) / 100.0
p = g["params"]
for it in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    idx, cost = ctx.eta_sweep(p, etas)
    e1.record(); torch.cuda.synchronize()
    print(it, round(e0.elapsed_time(e1), 2), flush=True)
    del idx, cost
# preallocated outputs, raw ABI call, per-step events
import ctypes as C
from paper_2407_13096_b200.api import _ptr
idx_o = torch.empty((101, n), dtype=torch.int32, device="cuda")
cost_o = torch.empty((101, n), dtype=torch.float32, device="cuda")
ea = np.ascontiguousarray(etas)
for it in range(12):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx._raise(ctx._lib.dso_eta_sweep(ctx._h, _ptr(p), n, n, ea.ctypes.data_as(C.POINTER(C.c_double)),
                                      101, dom.dev.pmax_w, _ptr(idx_o), _ptr(cost_o), n))
    e1.record(); torch.cuda.synchronize()
    print("raw", it, round(e0.elapsed_time(e1), 2), flush=True)
