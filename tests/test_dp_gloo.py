"""Multi-process (world_size 2, gloo, CPU) coverage of the N>1 host logic.

* kernel sharding: contiguous shards cover the batch exactly once, and the
  per-rank results gathered in rank order equal the single-process result
  (oracle sweep on CPU stands in for the GPU kernel);
* data-parallel training: the DataParallelTrainer's allreduce-then-apply step
  on two half batches equals the single-process step on the union batch;
* timing: the max-over-ranks reduction bench.py uses.
"""

import os
import socket
import types

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import oracle
        from paper_2407_13096_b200 import config_domain, init_mlp
        from paper_2407_13096_b200.train import DataParallelTrainer, shard_bounds, target_stats
        P = oracle.port()
        # ---- kernel sharding --------------------------------------------------------
        n = 10_001
        a, b = shard_bounds(n, world, rank)
        g = P.gen_stream(0xD50B203, b - a, first=a, want=("params",), threads=1)
        dom = config_domain("c3")
        st, r = P.brute_force(g["params"], dom.core_freqs_mhz, dom.mem_freqs_mhz,
                              dom.dev.as_array(), 0.8, dom.dev.pmax_w, threads=1)
        idx = torch.from_numpy(r["idx"].astype(np.int64))
        sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([len(idx)]))
        mx = int(max(s.item() for s in sizes))
        pad = torch.full((mx,), -7, dtype=torch.int64)
        pad[:len(idx)] = idx
        gathered = [torch.zeros(mx, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(gathered, pad)
        if rank == 0:
            out["shard_idx"] = np.concatenate([gg[:int(s.item())].numpy()
                                               for gg, s in zip(gathered, sizes)])
        # ---- data-parallel SGD step -------------------------------------------------
        B = 96
        gb = P.gen_stream(0xACCE5505, B, want=("params", "fused"), threads=1)
        mean, std, _ = target_stats(gb["params"])
        y = (gb["params"] - mean) / std
        a, b = shard_bounds(B, world, rank)
        m = init_mlp(seed=11)
        m.target_mean, m.target_std = mean, std
        state = {"W": [w.copy() for w in m.weights], "b": [v.copy() for v in m.biases]}

        def grad_fn(x, yy, nloc):
            mm = types.SimpleNamespace(layer_sizes=m.layer_sizes, weights=state["W"],
                                       biases=state["b"], target_mean=mean, target_std=std)
            gw, gbb = P.analytic_gradients(mm, x, yy)
            flat = np.concatenate([v.ravel() for v in gw + gbb]) * (nloc * 7)  # batch sums
            loss = P.mse_loss(mm, x, yy) * (nloc * 7)
            return torch.from_numpy(flat), torch.tensor([loss], dtype=torch.float64)

        def apply_fn(grad, lr, scale):
            g = grad.numpy() * scale
            off = 0
            for arr in state["W"] + state["b"]:
                arr -= lr * g[off:off + arr.size].reshape(arr.shape)
                off += arr.size

        tr = DataParallelTrainer(lr=0.3, grad_fn=grad_fn, apply_fn=apply_fn)
        loss = tr.step(gb["fused"][a:b], y[a:b], b - a, B)
        if rank == 0:
            out["dp_W"] = [w.copy() for w in state["W"]]
            out["dp_loss"] = float(loss.item())
        # ---- max-over-ranks timing ----------------------------------------------------
        t = torch.tensor([1.0 + rank], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        if rank == 0:
            out["tmax"] = float(t.item())
    finally:
        dist.destroy_process_group()


def test_two_rank_sharding_and_dp_step():
    world = 2
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, free_port(), out), nprocs=world, join=True)
    import sys
    sys.path.insert(0, ROOT)
    import oracle
    from paper_2407_13096_b200 import config_domain, init_mlp
    from paper_2407_13096_b200.train import target_stats
    P = oracle.port()
    n = 10_001
    g = P.gen_stream(0xD50B203, n, want=("params",))
    dom = config_domain("c3")
    st, r = P.brute_force(g["params"], dom.core_freqs_mhz, dom.mem_freqs_mhz,
                          dom.dev.as_array(), 0.8, dom.dev.pmax_w)
    np.testing.assert_array_equal(out["shard_idx"], r["idx"])
    # single-process step on the union batch
    B = 96
    gb = P.gen_stream(0xACCE5505, B, want=("params", "fused"))
    mean, std, _ = target_stats(gb["params"])
    y = (gb["params"] - mean) / std
    m = init_mlp(seed=11)
    mm = types.SimpleNamespace(layer_sizes=m.layer_sizes, weights=m.weights, biases=m.biases,
                               target_mean=mean, target_std=std)
    gw, _ = P.analytic_gradients(mm, gb["fused"], y)
    loss = P.mse_loss(mm, gb["fused"], y)
    for got, w, g in zip(out["dp_W"], m.weights, gw):
        np.testing.assert_allclose(got, w - 0.3 * g, rtol=0, atol=1e-12)
    assert out["dp_loss"] == pytest.approx(loss, rel=1e-12)
    assert out["tmax"] == 2.0
