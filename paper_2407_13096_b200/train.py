"""Predictor training: data-parallel mini-batch SGD on the device model.

Mirrors the reference's sgd_epoch / fit_model (proj/src/mlp.cpp:84-130):
targets standardized with the dataset's population mean/std (target_stats,
mlp.cpp:57-79; zero-variance dims left unscaled), per-epoch order from
shuffled_indices(Rng(seed).fork(0x5d0)) (mlp.cpp:87,123), contiguous batches
in that order (last one partial), the loss of each batch taken on the
pre-update weights (mlp.cpp:102-103), W -= lr * g (mlp.cpp:105-108), a NaN
epoch loss stops training (mlp.cpp:126).

Data parallel: every rank computes the batch-sum gradient of
its shard of each global batch on the GPU (dso_train_grad), the sums are
all-reduced over NCCL (torch.distributed), and every rank applies the same
update lr / (B_global * out) * g_sum (dso_train_apply) — so replicas stay
identical and the step equals the single-GPU step on the union batch up to
FP32 summation order.
"""

from __future__ import annotations

import ctypes as C
import math

import numpy as np

from ._lib import lib


def target_stats(targets):
    """target_stats (mlp.cpp:57-79) on a [n, out] float64 array: population
    mean / std; zero-variance dims get mean 0, std 1 and are reported."""
    t = np.asarray(targets, np.float64)
    mean = t.mean(0)
    std = np.sqrt(((t - mean) ** 2).mean(0))
    degenerate = [int(i) for i in np.flatnonzero(std == 0.0)]
    std[degenerate] = 1.0
    mean[degenerate] = 0.0
    return mean, std, degenerate


def shuffled_order(n: int, rng_state: int):
    """shuffled_indices (rng.hpp:58-64) via the library's host restatement;
    returns (order, advanced state)."""
    out = np.empty(n, np.uint64)
    st = C.c_uint64(rng_state)
    rc = lib().dso_shuffled_indices(n, C.byref(st), out.ctypes.data_as(C.POINTER(C.c_uint64)))
    if rc:
        raise RuntimeError("dso_shuffled_indices failed")
    return out.astype(np.int64), st.value


def fork(seed: int, salt: int) -> int:
    """Rng(seed).fork(salt) state (rng.hpp:50-54)."""
    mask = (1 << 64) - 1
    s = (seed ^ ((0xd1342543de82ef95 * (salt + 1)) & mask)) & mask
    s = (s + 0x9e3779b97f4a7c15) & mask  # one next_u64() advances the state
    return s


class DataParallelTrainer:
    """Synchronous data-parallel SGD of the device model in `ctx`.

    grad_fn / apply_fn default to the device kernels; tests substitute CPU
    functions to exercise the collective plumbing on gloo."""

    def __init__(self, ctx=None, lr: float = 0.1, group=None, grad_fn=None, apply_fn=None,
                 allreduce=None):
        self.ctx = ctx
        self.lr = lr
        self.group = group
        self.grad_fn = grad_fn or (lambda x, y, n: ctx.train_grad(x, y, n=n))
        self.apply_fn = apply_fn or (lambda g, lr, s: ctx.train_apply(g, lr, s))
        self._allreduce = allreduce

    def world(self) -> int:
        import torch.distributed as dist
        if dist.is_available() and dist.is_initialized():
            return dist.get_world_size(self.group)
        return 1

    def allreduce(self, t):
        if self._allreduce is not None:
            return self._allreduce(t)
        import torch.distributed as dist
        if self.world() > 1:
            dist.all_reduce(t, op=dist.ReduceOp.SUM, group=self.group)
        return t

    def step(self, x_local, y_local, n_local: int, global_batch: int, out_dim: int = 7):
        """One synchronous step; returns the batch's mse_loss (mlp.cpp:259-263) on the
        pre-update weights, as a 0-dim tensor on the device."""
        grad, loss = self.grad_fn(x_local, y_local, n_local)
        self.allreduce(grad)
        self.allreduce(loss)
        scale = 1.0 / (global_batch * out_dim)
        self.apply_fn(grad, self.lr, scale)
        return loss * scale


def shard_bounds(n: int, world: int, rank: int):
    """Contiguous shard [a, b) of n items for rank."""
    a = n * rank // world
    b = n * (rank + 1) // world
    return a, b


def epoch_batches(n: int, batch: int):
    """Contiguous batches over the shuffled order, last one partial (mlp.cpp:242-243)."""
    for start in range(0, n, batch):
        yield start, min(batch, n - start)


def is_nan_loss(v) -> bool:
    return not math.isfinite(float(v))
