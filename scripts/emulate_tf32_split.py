"""Emulated precision of split tensor-core products for the predictor (numpy, CPU).

Compares the MLP forward with each layer's products computed as
  fp32, 1xTF32, 3xTF32 (hi.hi + hi.lo + lo.hi), and bf16 splits with 3..6 products
against the oracle's double forward on the test_gpu_mlp inputs, in units of the
1e-5 * |ref| + 1e-6 * std tolerance (worst case and 99.9th percentile).  This is the
evidence for the tcgen05 engine's 3xTF32 choice.  Test/analysis
infrastructure: it uses the oracle, like tests/.
usage: python scripts/emulate_tf32_split.py
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Port
from paper_2407_13096_b200 import init_mlp
port = Port()
m = init_mlp(seed=424242)
params = port.gen_stream(0xC0FFEE, 4096, want=("params",))["params"]
mean, std, _ = port.target_stats(params)
m.target_mean, m.target_std = mean, std
n = 20000
fused = port.gen_stream(0xD50B201, n, want=("fused",))["fused"]
rng = np.random.default_rng(1)
fused[: n // 4] = rng.uniform(0, 1, size=(n // 4, 134))
x = fused.astype(np.float32)
want = port.forward_raw(m, x.astype(np.float64))

def tf32(a):  # cvt.rna.tf32.f32: round to nearest, ties away, keep 10 mantissa bits
    a = np.asarray(a, np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x1000) & 0xFFFFE000
    return u.astype(np.uint32).view(np.float32)

def mm_fp32(a, w): return (a.astype(np.float32) @ w.T.astype(np.float32)).astype(np.float32)
def mm_3x(a, w, trunc_chunks=True):
    a = a.astype(np.float32); w = w.astype(np.float32)
    ah = tf32(a); al = tf32(a - ah); wh = tf32(w); wl = tf32(w - wh)
    # products exact in double; accumulate per 8-wide k step in float32 (emulates fp32 accumulation)
    K = a.shape[1]; acc = np.zeros((a.shape[0], w.shape[0]), np.float32)
    for k0 in range(0, K, 8):
        sl = slice(k0, k0 + 8)
        for A, W in ((ah, wh), (ah, wl), (al, wh)):
            part = (A[:, sl].astype(np.float64) @ W[:, sl].T.astype(np.float64))
            acc = (acc.astype(np.float64) + part).astype(np.float32)
    return acc
def mm_1x(a, w):
    return (tf32(a).astype(np.float64) @ tf32(w).T.astype(np.float64)).astype(np.float32)

def fwd(mm):
    h = x
    L = len(m.weights)
    for l, (W, b) in enumerate(zip(m.weights, m.biases)):
        z = (mm(h, np.asarray(W)) + np.asarray(b, np.float32)).astype(np.float32)
        h = z if l == L - 1 else (1 / (1 + np.exp(-z.astype(np.float64)))).astype(np.float32)
    return h.astype(np.float64) * std + mean
tol = 1e-5 * np.abs(want) + 1e-6 * std[None, :]
def _main_table():
  for name, mm in (("fp32", mm_fp32), ("3xtf32", mm_3x), ("1xtf32", mm_1x)):
    got = fwd(mm)
    r = np.abs(got - want) / tol
    print(name, "worst x tol", r.max(), "p99.9", np.quantile(r, 0.999))
def bf16(a):
    a = np.asarray(a, np.float32); u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)
def mm_terms(split, terms):
    def mm(a, w):
        a = a.astype(np.float32); w = w.astype(np.float32)
        A = [split(a)]; A.append(split(a - A[0])); A.append(split(a - A[0] - A[1]))
        W = [split(w)]; W.append(split(w - W[0])); W.append(split(w - W[0] - W[1]))
        K = a.shape[1]; acc = np.zeros((a.shape[0], w.shape[0]), np.float32)
        for k0 in range(0, K, 8):
            sl = slice(k0, k0 + 8)
            for i, j in terms:
                part = A[i][:, sl].astype(np.float64) @ W[j][:, sl].T.astype(np.float64)
                acc = (acc.astype(np.float64) + part).astype(np.float32)
        return acc
    return mm
def _terms_table():
    for name, mm in (("tf32 A1 W2", mm_terms(tf32, [(0, 0), (0, 1)])),
                     ("tf32 A2 W1", mm_terms(tf32, [(0, 0), (1, 0)])),
                     ("bf16 3 terms", mm_terms(bf16, [(0, 0), (0, 1), (1, 0)])),
                     ("bf16 5 terms", mm_terms(bf16, [(0, 0), (0, 1), (1, 0), (0, 2), (2, 0)])),
                     ("bf16 6 terms", mm_terms(bf16, [(0, 0), (0, 1), (1, 0), (1, 1), (0, 2), (2, 0)]))):
        r = np.abs(fwd(mm) - want) / tol
        print(name, "worst x tol", r.max(), "p99.9", np.quantile(r, 0.999))


if __name__ == "__main__":
    _main_table()
    _terms_table()
