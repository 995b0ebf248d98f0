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


# ---------------------------------------------------------------------------
# Training orchestration on the device model: fit_model, prediction_mape_pct,
# cross_validate, train (reference proj/src/mlp.cpp:35-130, 348-437;
# mlp.hpp:75-121).  The dataset is a pair of float64 arrays, features [n, 134]
# and raw targets [n, 7] (TrainingExample, mlp.hpp:50-53).  Every epoch's
# shuffled order is gathered on the device once; batches are then contiguous
# column slices fed to dso_train_grad / dso_train_apply, and the epoch loss is
# read back once per epoch.

K_MAPE_FLOOR = 1e-9  # kMapeDenominatorFloor, mlp.cpp:14
K_FOLDS = 3          # cross_validate, mlp.cpp:359


def canonicalize(features, targets):
    """canonicalize (mlp.cpp:35-50): lexicographic sort by features, then targets."""
    f = np.asarray(features, np.float64)
    t = np.asarray(targets, np.float64)
    keys = np.concatenate([f, t], axis=1)
    order = np.lexsort(keys.T[::-1]) if len(keys) else np.zeros(0, np.int64)
    return f[order], t[order]


def _dev_cols(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(np.asarray(a, np.float32).T)).cuda()


def fit_model(ctx, features, targets, sizes, mean, std, lr: float, batch_size: int,
              epochs: int, seed: int, comm=None, rank: int = 0, nranks: int = 1):
    """fit_model (mlp.cpp:115-130) on the GPU: init_mlp(sizes, seed) with the given
    target stats, then the library's native epoch loop (dso_fit_model: per-epoch
    order shuffled_indices(Rng(seed).fork(0x5d0)), contiguous batches, the loss of
    every batch on the pre-update weights, stop after a NaN epoch; one CUDA graph
    replay per epoch).  Returns (model, epoch_loss_trace)."""
    from .model import init_mlp
    m = init_mlp(list(sizes), seed=seed)
    m.target_mean, m.target_std = np.array(mean, np.float64), np.array(std, np.float64)
    ctx.set_model(m)
    f = np.asarray(features, np.float64)
    y = (np.asarray(targets, np.float64) - m.target_mean) / m.target_std
    X, Y = _dev_cols(f), _dev_cols(y)
    trace = ctx.fit_model(X, Y, lr, batch_size, epochs, seed, comm=comm, rank=rank,
                          nranks=nranks)
    return ctx.get_model(), trace


def prediction_mape_pct(ctx, model, features, targets) -> float:
    """prediction_mape_pct (mlp.cpp:132-146) with the device forward_raw
    (dso_predict's raw output): inf when any prediction is non-finite."""
    ctx.set_model(model)
    t = np.asarray(targets, np.float64)
    _, _, raw = ctx.predict_params(_dev_cols(features), want_raw=True)
    pred = raw.cpu().numpy().T.astype(np.float64)
    if not np.isfinite(pred).all():
        return float("inf")
    return float(100.0 * np.mean(np.abs(pred - t) / np.maximum(np.abs(t), K_MAPE_FLOOR)))


def cross_validate(ctx, features, targets, grid, seed: int, epochs: int, sizes=None):
    """cross_validate (mlp.cpp:348-411): 3 folds from shuffled_indices(Rng(seed)
    .fork(0xf01d)) over the canonical order; per cell and fold a fit_model on the
    training split with its own target_stats, run seed seed + 1000003*fold +
    29*cell; MAPE on the validation split (inf when diverged or a split is
    empty); lowest mean wins, ties to smaller lr, then smaller batch.
    Returns {"table": [(lr, batch, [fold mapes], mean)], "best": (lr, batch)}."""
    from ._lib import DsoError, ErrorKind
    f, t = canonicalize(features, targets)
    n = len(f)
    if n < 3:
        raise DsoError(ErrorKind.DatasetTooSmall,
                       f"cross-validation needs at least 3 examples, got {n}")
    if not grid:
        raise DsoError(ErrorKind.InvalidArgument, "empty hyperparameter grid")
    sizes = list(sizes) if sizes else [f.shape[1], 100, 50, 25, t.shape[1]]
    sizes[0], sizes[-1] = f.shape[1], t.shape[1]
    order, _ = shuffled_order(n, fork(seed, 0xF01D))
    fold_of = np.empty(n, np.int64)
    fold_of[order] = np.arange(n) % K_FOLDS
    table = []
    for ci, (lr, bs) in enumerate(grid):
        mapes = []
        for fold in range(K_FOLDS):
            tr, va = fold_of != fold, fold_of == fold
            if not tr.any() or not va.any():
                mapes.append(float("inf"))
                continue
            mean, std, _ = target_stats(t[tr])
            run_seed = (seed + 1000003 * fold + 29 * ci) & ((1 << 64) - 1)
            m, trace = fit_model(ctx, f[tr], t[tr], sizes, mean, std, lr, bs, epochs, run_seed)
            diverged = bool(trace) and math.isnan(trace[-1])
            mapes.append(float("inf") if diverged else
                         prediction_mape_pct(ctx, m, f[va], t[va]))
        table.append((float(lr), int(bs), mapes, sum(mapes) / K_FOLDS))
    best = table[0]
    for row in table:
        if row[3] < best[3] or (row[3] == best[3] and (
                row[0] < best[0] or (row[0] == best[0] and row[1] < best[1]))):
            best = row
    return {"table": table, "best": (best[0], best[1])}


def train(ctx, features, targets, grid, seed: int, epochs: int, sizes=None,
          learning_rate: float = 0.1, batch_size: int = 16):
    """train (mlp.cpp:413-437): checks, cross-validation over grid, then a final
    fit_model on the whole canonical dataset with the winning cell. An empty grid
    means the single cell (learning_rate, batch_size), as TrainConfig's defaults
    (mlp.hpp:75-89, mlp.cpp:424-427).
    Returns {"model", "cv", "epoch_loss", "degenerate_targets"}."""
    from ._lib import DsoError, ErrorKind
    f = np.asarray(features, np.float64)
    t = np.asarray(targets, np.float64)
    if len(f) < 3:
        raise DsoError(ErrorKind.DatasetTooSmall,
                       f"training needs at least 3 examples, got {len(f)}")
    if not (np.isfinite(f).all() and np.isfinite(t).all()):
        raise DsoError(ErrorKind.InvalidArgument, "dataset contains non-finite values")
    f, t = canonicalize(f, t)
    sizes = list(sizes) if sizes else [f.shape[1], 100, 50, 25, t.shape[1]]
    sizes[0], sizes[-1] = f.shape[1], t.shape[1]
    if not grid:
        grid = [(float(learning_rate), int(batch_size))]
    cv = cross_validate(ctx, f, t, grid, seed, epochs, sizes)
    mean, std, degenerate = target_stats(t)
    lr, bs = cv["best"]
    model, trace = fit_model(ctx, f, t, sizes, mean, std, lr, bs, epochs, seed)
    return {"model": model, "cv": cv, "epoch_loss": trace, "degenerate_targets": degenerate}
