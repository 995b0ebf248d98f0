"""PTX text + DCGM CSV -> host ingestion -> fused GPU pipeline (host buffers) vs the
oracle pipeline on the same parsed counts (the reference's full path from
parse_ptx to brute_force_config)."""

import os

import numpy as np
import pytest
import torch

from helpers import check_argmin
from paper_2407_13096_b200 import config_domain, init_mlp
from paper_2407_13096_b200.ingest import ingest_corpus, parse_ptx

pytestmark = pytest.mark.gpu
HERE = os.path.join(os.path.dirname(__file__), "golden", "ptx")


def test_ptx_to_decision(ctx, port):
    files = sorted(f for f in os.listdir(HERE) if f.endswith(".ptx"))
    texts = [open(os.path.join(HERE, f)).read() for f in files]
    rng = np.random.default_rng(5)
    H = "timestamp,SMACT,SMOCC,TENSO,DRAMA,FP64A,FP32A,FP16A,INTAC\n"
    # a larger synthetic corpus: every fixture, repeated with perturbed DCGM traces
    texts = texts * 40
    dc = ["".join([H] + [f"{r}," + ",".join(f"{x:.6f}" for x in rng.uniform(0, 1, 8)) + "\n"
                         for r in range(int(rng.integers(1, 5)))]) for _ in texts]
    names, rp, ent, dcgm = ingest_corpus(texts, dc, threads=4)
    dom = config_domain("c1")
    ctx.set_domain(dom)
    m = init_mlp(seed=424242)
    m.target_mean = np.array([60, 10, 0.01, 0.004, 0.15, 200, 200.0])
    m.target_std = np.array([15, 3, 0.005, 0.001, 0.07, 100, 100.0])
    ctx.set_model(m)
    out = ctx.pipeline_csr(torch.from_numpy(rp.view(np.int64)), torch.from_numpy(ent.view(np.int32)),
                           torch.from_numpy(dcgm), 0.8, want_params=True)
    counts = np.stack([parse_ptx(t)[0][1] for t in texts]).astype(np.uint32)
    st, want = port.pipeline(counts, dcgm.T.astype(np.float64), m, dom.core_freqs_mhz,
                             dom.mem_freqs_mhz, dom.dev.as_array(), 0.8, dom.dev.pmax_w)
    assert st == 0
    p = np.asarray(out["params"]).T.astype(np.float64)
    tol = 1e-5 * np.abs(want["params"]) + 1e-6 * m.target_std[None, :]
    assert (np.abs(p - want["params"]) <= tol).all()
    idx = np.asarray(out["idx"])
    r = port.brute_force(p, dom.core_freqs_mhz, dom.mem_freqs_mhz, dom.dev.as_array(), 0.8,
                         dom.dev.pmax_w)[1]
    check_argmin(p, idx, r["idx"], dom.core_freqs_mhz, dom.mem_freqs_mhz, dom.dev.as_array(),
                 0.8, dom.dev.pmax_w)
