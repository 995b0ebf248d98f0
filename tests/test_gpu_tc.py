"""GPU bring-up checks for the tcgen05 building blocks (csrc/tc.cuh) via the
dso_debug_tc_gemm probe: TMEM allocation, tcgen05.st/ld, kind::tf32 MMA with A in
TMEM and B in shared memory (SWIZZLE_NONE K-major core matrices), commit.

Bars: single-pass TF32 within TF32 rounding of the FP32 product; 3xTF32 within
FP32-accumulation error (relative 2e-6 of the row's |A|.|B| scale)."""

import ctypes as C

import numpy as np
import pytest
import torch

from paper_2407_13096_b200 import _lib

pytestmark = pytest.mark.gpu


_PROBE = None


def probe_lib():
    """The test-only probe library (csrc/tcprobe.cu, not part of libdso_b200.so)."""
    global _PROBE
    if _PROBE is None:
        import os
        _PROBE = C.CDLL(os.path.join(os.path.dirname(_lib.LIB_PATH), "libdso_tcprobe.so"))
    return _PROBE


def tc_gemm(a, b, passes, reps=1):
    f = probe_lib().dso_debug_tc_gemm
    f.argtypes = [C.c_void_p] * 3 + [C.c_int32] * 4 + [C.c_void_p]
    f.restype = C.c_int32
    A = torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()
    B = torch.from_numpy(np.ascontiguousarray(b, np.float32)).cuda()
    D = torch.zeros((128, b.shape[0]), dtype=torch.float32, device="cuda")
    cyc = torch.zeros(1, dtype=torch.int64, device="cuda")
    st = f(A.data_ptr(), B.data_ptr(), D.data_ptr(), a.shape[1], b.shape[0], passes, reps,
           cyc.data_ptr())
    assert st == 0, st
    return D.cpu().numpy(), int(cyc.item())


@pytest.mark.parametrize("K,N", [(8, 16), (136, 112), (104, 64), (56, 32), (32, 16)])
@pytest.mark.parametrize("passes", [1, 3])
def test_tc_gemm(K, N, passes):
    rng = np.random.default_rng(K * 1000 + N)
    a = rng.uniform(-1, 1, (128, K)).astype(np.float32)
    b = rng.uniform(-1, 1, (N, K)).astype(np.float32)
    d, _ = tc_gemm(a, b, passes)
    want = a.astype(np.float64) @ b.T.astype(np.float64)
    scale = np.abs(a).astype(np.float64) @ np.abs(b).T.astype(np.float64)
    err = np.abs(d - want) / scale
    bound = 2e-3 if passes == 1 else 2e-6
    assert err.max() <= bound, (err.max(), np.unravel_index(err.argmax(), err.shape))


def test_tc_gemm_rate():
    rng = np.random.default_rng(5)
    a = rng.uniform(-1, 1, (128, 136)).astype(np.float32)
    b = rng.uniform(-1, 1, (112, 136)).astype(np.float32)
    _, c1 = tc_gemm(a, b, 3, reps=1)
    _, c64 = tc_gemm(a, b, 3, reps=64)
    flops = 2 * 128 * 112 * 136 * 3 * 63
    print(f"\n3xTF32 128x112x136: {c1} cycles single, {(c64 - c1) / 63:.0f} per chain, "
          f"{flops / (c64 - c1):.0f} flop/clk/SM")


# ---- the tensor-core predictor engine (mlp_engine = 1) vs the FMA-pipe engine ----

from paper_2407_13096_b200 import config_domain, init_mlp  # noqa: E402


def _model(port=None, seed=424242):
    m = init_mlp(seed=seed)
    m.target_mean = np.array([60, 10, 0.01, 0.004, 0.15, 200, 200.0])
    m.target_std = np.array([15, 3, 0.005, 0.001, 0.07, 100, 100.0])
    return m


def _both(ctx, fn):
    out = []
    for eng in (0, 1):
        ctx.set_option("mlp_engine", eng)
        try:
            r = fn()
            out.append({k: (v.cpu().numpy() if hasattr(v, "cpu") else v) for k, v in r.items()})
        finally:
            ctx.set_option("mlp_engine", 2)
    return out


def _close(a, b, std):
    """Same NaN pattern; finite values within the MLP contract (1e-5 rel + 1e-6 std)."""
    na, nb = np.isnan(a), np.isnan(b)
    assert (na == nb).all()
    fin = ~na
    tol = 1e-5 * np.abs(a[fin]) + 1e-6 * np.broadcast_to(std[:, None], a.shape)[fin]
    assert (np.abs(a[fin] - b[fin]) <= 2 * tol).all()


def test_tc_nonfinite_dcgm_pipeline_csr(ctx):
    """A non-finite DCGM value takes the FMA-pipe forward inside the tc engine: the
    same IEEE semantics as the reference (inf * w stays inf, sigmoid(inf) = 1)."""
    ctx.set_domain(config_domain("c3"))
    m = _model()
    ctx.set_model(m)
    n = 20_000
    g = ctx.gen_synthetic_csr(n, root=5)
    d = g["dcgm"].clone()
    d[0, 7] = float("inf")
    d[3, 300] = float("-inf")
    d[5, 4097] = float("nan")
    d[:, 12345] = float("inf")
    a, b = _both(ctx, lambda: ctx.pipeline_csr(g["row_ptr"], g["entries"], d, 0.8, want_params=True))
    _close(a["params"], b["params"], m.target_std)
    for k in (7, 300, 4097, 12345):
        assert a["idx"][k] == b["idx"][k] or np.isnan(a["params"][:, k]).any()


def test_tc_nonfinite_fused_predict(ctx):
    m = _model()
    ctx.set_model(m)
    rng = np.random.default_rng(3)
    x = rng.uniform(0, 1, (134, 5000)).astype(np.float32)
    x[20, 11] = np.inf
    x[133, 12] = -np.inf
    x[0, 13] = np.nan
    xt = torch.from_numpy(x).cuda()
    a, b = _both(ctx, lambda: dict(zip(("params", "clamped", "raw"),
                                       ctx.predict_params(xt, want_raw=True))))
    _close(a["raw"], b["raw"], m.target_std)
    assert np.isnan(a["raw"][:, 13]).all() and np.isnan(b["raw"][:, 13]).all()


def test_tc_nonfinite_weights_fall_back(ctx):
    """A model with a non-finite weight is routed to the FFMA engine (host flag)."""
    m = _model()
    m.weights[1][3, 7] = np.inf
    ctx.set_model(m)
    x = torch.rand(134, 3000, device="cuda")
    a, b = _both(ctx, lambda: dict(zip(("params", "clamped", "raw"),
                                       ctx.predict_params(x, want_raw=True))))
    np.testing.assert_array_equal(a["raw"], b["raw"])


def test_tc_after_device_repack(ctx):
    """After a training step the weights are repacked on the device; the tc engine
    reads its device-side finiteness flag (both engines launched, one exits)."""
    m = _model()
    ctx.set_model(m)
    x = torch.rand(134, 4096, device="cuda")
    y = torch.randn(7, 4096, device="cuda")
    grad, _ = ctx.train_grad(x, y)
    ctx.train_apply(grad, 1e-3, 1.0 / 4096)
    a, b = _both(ctx, lambda: dict(zip(("params", "clamped", "raw"),
                                       ctx.predict_params(x, want_raw=True))))
    _close(a["raw"], b["raw"], m.target_std)
    # a non-finite update: the device flag sends the launch to the FFMA engine
    grad.fill_(float("inf"))
    ctx.train_apply(grad, 1e-3, 1.0)
    a, b = _both(ctx, lambda: dict(zip(("params", "clamped", "raw"),
                                       ctx.predict_params(x, want_raw=True))))
    np.testing.assert_array_equal(a["raw"], b["raw"])


def test_tc_engine_option_errors(ctx):
    from paper_2407_13096_b200 import DsoError
    with pytest.raises(DsoError):
        ctx.set_option("mlp_engine", 3)


def test_tc_large_domain_falls_back(ctx):
    """A domain whose level tables do not fit next to the split weights (nc = 600)
    runs the FMA-pipe kernel under mlp_engine = 1: identical to engine 0."""
    from paper_2407_13096_b200 import linear_domain
    ctx.set_domain(linear_domain(600, 4))
    m = _model()
    ctx.set_model(m)
    g = ctx.gen_synthetic_csr(3000, root=9)
    a, b = _both(ctx, lambda: ctx.pipeline_csr(g["row_ptr"], g["entries"], g["dcgm"], 0.8,
                                               want_params=True))
    for f in ("idx", "cost", "energy", "time", "params", "clamped"):
        np.testing.assert_array_equal(a[f], b[f])
