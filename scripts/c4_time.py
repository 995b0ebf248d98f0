"""C4 eta-sweep timing (experiment script): 101 etas x 4M kernels, CUDA events."""
import ctypes as C
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_13096_b200 import linear_domain  # noqa: E402
from paper_2407_13096_b200.api import Context, _ptr  # noqa: E402

ctx = Context(0)
dom = linear_domain(128, 4)
ctx.set_domain(dom)
n = 1 << 22
p = ctx.gen_synthetic(n, root=0xD50B203, counts=False, dcgm=False)["params"]
idx_o = torch.empty((101, n), dtype=torch.int32, device="cuda")
cost_o = torch.empty((101, n), dtype=torch.float32, device="cuda")
ea = np.ascontiguousarray(np.arange(101) / 100.0)
for prune in (1, 0):
  ctx.set_option("eta_prune", prune)
  ts = []
  for _ in range(6):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    ctx._raise(ctx._lib.dso_eta_sweep(ctx._h, _ptr(p), n, n, ea.ctypes.data_as(C.POINTER(C.c_double)),
                                      101, dom.dev.pmax_w, _ptr(idx_o), _ptr(cost_o), n))
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
  if prune:
    ref_idx, ref_cost = idx_o.clone(), cost_o.clone()
  else:
    print("pruned == unpruned:", bool(torch.equal(ref_idx, idx_o)), bool(torch.equal(ref_cost.view(torch.int32), cost_o.view(torch.int32))))
  print("C4 eta sweep prune=%d ms:" % prune, [round(t, 2) for t in ts])
