"""Per-phase cycle breakdown of the tensor-core engine (debug library)."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("DSO_B200_LIB", os.path.join(ROOT, "paper_2407_13096_b200", "lib", "libdso_b200_phase.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2407_13096_b200 import _lib, config_domain, init_mlp  # noqa: E402
from paper_2407_13096_b200.api import Context  # noqa: E402

L = _lib.lib()
L.dso_debug_phase_cycles.argtypes = [C.c_void_p, C.c_int]
# epilogue phases are recorded by group 0 only (every other tile): scaled x2 below
names = ["p.wait_XEMPTY", "p.put+arrive", "e.wait_D1", "e.epi1", "e.wait_D2", "e.epi2", "-",
         "e.epi3", "-", "e.sweep(prev tile)", "e.clamp+slow", "-", "-", "-",
         "p.prep", "p.chunks", "p.passA", "-", "p.mask", "p.slow"]
ctx = Context(0)
ctx.set_option("mlp_engine", 1)
n = 1 << 22
for mode in os.environ.get("TC_PHASE_MODES", "pipeline_csr,predict,pipeline").split(","):
    ctx.set_domain(config_domain(os.environ.get("TC_PHASE_DOMAIN", "c3")))
    m = init_mlp(seed=424242)
    m.target_mean = np.array([60, 10, 0.01, 0.004, 0.15, 200, 200.0])
    m.target_std = np.array([15, 3, 0.005, 0.001, 0.07, 100, 100.0])
    ctx.set_model(m)
    g = ctx.gen_synthetic(n, root=3)
    gc = ctx.gen_synthetic_csr(n, root=3)
    f = ctx.featurize(g["counts"], g["dcgm"])
    buf = (C.c_ulonglong * 32)()
    run = {"pipeline_csr": lambda: ctx.pipeline_csr(gc["row_ptr"], gc["entries"], gc["dcgm"], 0.8),
           "pipeline": lambda: ctx.pipeline(g["counts"], g["dcgm"], 0.8),
           "predict": lambda: ctx.predict_params(f)}[mode]
    run()
    L.dso_debug_phase_cycles(buf, 1)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run()
    e1.record()
    torch.cuda.synchronize()
    L.dso_debug_phase_cycles(buf, 1)
    ms = e0.elapsed_time(e1)
    tiles = n // 128
    print(f"== {mode} (tc): {ms:.3f} ms for {n} kernels; per 128-kernel tile (cycles):")
    for i, nm in enumerate(names):
        if nm:
            scale = 2 if nm.startswith("e.") else 1
            print(f"  {nm:14s} {scale * buf[i] / tiles:10.0f}")
