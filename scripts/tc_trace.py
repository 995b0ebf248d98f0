"""Event timeline of CTA 0 of the tcgen05 pipeline kernel (trace build:
scripts/build_variant.sh trace -DDSO_TC_TRACE).  Prints, per tile, the cycle at which
each role reached each point, relative to tile 8's producer start."""
import ctypes as C
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
os.environ.setdefault("DSO_B200_LIB", os.path.join(ROOT, "paper_2407_13096_b200", "lib",
                                                   "libdso_b200_trace.so"))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

from paper_2407_13096_b200 import _lib, config_domain, init_mlp  # noqa: E402
from paper_2407_13096_b200.api import Context  # noqa: E402

L = _lib.lib()
L.dso_debug_trace.argtypes = [C.c_void_p]
ctx = Context(0)
ctx.set_option("mlp_engine", 1)
ctx.set_domain(config_domain("c3"))
m = init_mlp(seed=424242)
m.target_mean = np.array([60, 10, 0.01, 0.004, 0.15, 200, 200.0])
m.target_std = np.array([15, 3, 0.005, 0.001, 0.07, 100, 100.0])
ctx.set_model(m)
n = 148 * 128 * 40
g = ctx.gen_synthetic_csr(n, root=3)
for _ in range(2):
    ctx.pipeline_csr(g["row_ptr"], g["entries"], g["dcgm"], 0.8)
ctx.sync()
buf = (C.c_ulonglong * (16 * 64 + 64 * 24))()
L.dso_debug_trace(buf)
allv = np.array(buf, dtype=np.int64)
tr = allv[:1024].reshape(16, 64)
tr2 = allv[1024:].reshape(64, 6, 4)
names = ["L1 first", "L1 last", "L2 first", "L2 last", "P start", "P mask", "-", "P done",
         "E wD1 beg", "E D1 got", "E epi1 end", "E D2 got", "E D2 read", "E epi3 end", "E done"]
t0 = tr[4, 8]
print("tile " + " ".join(f"{x:>10s}" for x in names if x != "-"))
for t in range(8, 30):
    row = [tr[e, t] - t0 for e in range(15) if e != 6]
    print(f"{t:4d} " + " ".join(f"{v:10d}" for v in row))

print("\nproducer thread 0, per chunk: claim begin / claim end / written / handed over (rel. to P mask)")
for t in range(8, 14):
    base = tr[5, t]
    print(f"{t:4d} " + "  ".join("/".join(str(int(v - base)) for v in tr2[t, c]) for c in range(5) if tr2[t, c, 0]))

print("\nproducer thread 0, prep: entries loaded / decoded / exchanged / list written (rel. to P start)")
for t in range(8, 14):
    base = tr[4, t]
    print(f"{t:4d} " + " / ".join(str(int(v - base)) for v in tr2[t, 5]) + f"   mask at {int(tr[5, t] - base)}")
