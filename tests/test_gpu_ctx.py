"""Context lifetime and multi-context use of the C-ABI (GPU).

* the per-context scratch that dso_dcgm_mean, dso_eta_sweep and dso_param_fit
  keep (flag, eta table, factored designs) survives any call order on one
  context, and dso_ctx_destroy frees each exactly once (run under
  compute-sanitizer by scripts/gpu_check.sh);
* several contexts in one process (same device here; one per device when the
  box has more) each launch the large-shared-memory kernels: the dynamic
  shared-memory attribute is applied per (kernel, device), not per process.
"""

import numpy as np
import pytest
import torch

from paper_2407_13096_b200 import config_domain, init_mlp
from paper_2407_13096_b200.api import Context

pytestmark = pytest.mark.gpu


def _model(port):
    m = init_mlp(seed=424242)
    p = port.gen_stream(0xC0FFEE, 4096, want=("params",))["params"]
    m.target_mean, m.target_std = p.mean(0), p.std(0)
    return m


def test_dcgm_eta_param_fit_any_order(port):
    """dcgm_mean -> eta_sweep (growing eta table) -> dcgm_mean -> param_fit ->
    eta_sweep (larger) -> dcgm_mean -> destroy, on one fresh context."""
    rng = np.random.default_rng(11)
    s = torch.from_numpy(rng.uniform(0, 1, size=(5, 8, 300))).cuda()
    dom = config_domain("c3")
    with Context(0) as c:
        c.set_domain(dom)
        m1, _ = c.dcgm_mean(s)
        params = c.gen_synthetic(4096, root=3, counts=False, dcgm=False)["params"]
        i1, c1 = c.eta_sweep(params, np.linspace(0, 1, 7))
        m2, _ = c.dcgm_mean(s)
        grid = [[2.0 * (fc / 1000 - 0.5) ** 2 + 0.5, fc, fm]
                for fc in (705.0, 900.0, 1100.0, 1380.0) for fm in (438.0, 877.0)]
        P = torch.rand((len(grid), 64), dtype=torch.float64, device="cuda") + 100.0
        c.param_fit(grid, power=P)
        i2, c2 = c.eta_sweep(params, np.linspace(0, 1, 101))
        m3, _ = c.dcgm_mean(s)
        torch.cuda.synchronize()
        np.testing.assert_array_equal(m1.cpu().numpy(), m2.cpu().numpy())
        np.testing.assert_array_equal(m1.cpu().numpy(), m3.cpu().numpy())
        # eta rows shared by both calls are identical
        np.testing.assert_array_equal(i1[0].cpu().numpy(), i2[0].cpu().numpy())
        np.testing.assert_array_equal(i1[-1].cpu().numpy(), i2[-1].cpu().numpy())


def _pipeline_once(c, m, n=20_000):
    c.set_domain(config_domain("c3"))
    c.set_model(m)
    g = c.gen_synthetic_csr(n, root=99)
    return {k: v.cpu().numpy() for k, v in c.pipeline_csr(g["row_ptr"], g["entries"], g["dcgm"],
                                                          0.8, want_params=True).items()}


def test_two_contexts_same_device(port):
    """Two contexts on one device, interleaved: both run the fused kernels and agree."""
    m = _model(port)
    with Context(0) as a, Context(0) as b:
        ra = _pipeline_once(a, m)
        rb = _pipeline_once(b, m)
        ra2 = _pipeline_once(a, m)
    for k in ra:
        np.testing.assert_array_equal(ra[k], rb[k])
        np.testing.assert_array_equal(ra[k], ra2[k])


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs")
def test_contexts_on_two_devices(port):
    """One context per device in one process: each device gets the shared-memory
    attribute before its first launch, and the results are identical."""
    m = _model(port)
    with Context(0) as a, Context(1) as b:
        ra = _pipeline_once(a, m)
        rb = _pipeline_once(b, m)
    for k in ra:
        np.testing.assert_array_equal(ra[k], rb[k])
