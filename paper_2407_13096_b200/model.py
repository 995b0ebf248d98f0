"""MLP model container — host mirror of dso::MlpModel (proj/include/dso/mlp.hpp:35-48).

Weights are kept in the reference layout (W_l of shape (sizes[l+1], sizes[l]),
row-major, float64) so a model round-trips with the reference's model JSON
(json_io.cpp:145-206).  init_mlp runs the library's host C++ restatement of
mlp.cpp:184-207 (Glorot-uniform from the splitmix64 Rng).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import DsoError, ErrorKind, lib, status_kind

K_FUSED_FEATURES = 134  # mlp.hpp:15
K_PARAMS = 7            # mlp.hpp:16


def default_layer_sizes() -> list[int]:
    """mlp.cpp:177."""
    return [K_FUSED_FEATURES, 100, 50, 25, K_PARAMS]


@dataclass
class MlpModel:
    layer_sizes: list
    weights: list
    biases: list
    target_mean: np.ndarray = field(default_factory=lambda: np.zeros(K_PARAMS))
    target_std: np.ndarray = field(default_factory=lambda: np.ones(K_PARAMS))
    seed: int = 0

    def flat(self):
        W = np.concatenate([np.asarray(w, np.float64).ravel() for w in self.weights])
        b = np.concatenate([np.asarray(b, np.float64).ravel() for b in self.biases])
        return np.ascontiguousarray(W), np.ascontiguousarray(b)

    @property
    def n_params(self) -> int:
        return sum(int(np.size(w)) + int(np.size(b)) for w, b in zip(self.weights, self.biases))

    def copy(self) -> "MlpModel":
        return MlpModel(list(self.layer_sizes), [np.array(w) for w in self.weights],
                        [np.array(b) for b in self.biases], np.array(self.target_mean),
                        np.array(self.target_std), self.seed)


def split_flat(sizes, W, b):
    ws, bs, ow, ob = [], [], 0, 0
    for l in range(len(sizes) - 1):
        fi, fo = int(sizes[l]), int(sizes[l + 1])
        ws.append(np.array(W[ow:ow + fi * fo], np.float64).reshape(fo, fi))
        bs.append(np.array(b[ob:ob + fo], np.float64))
        ow += fi * fo
        ob += fo
    return ws, bs


def init_mlp(layer_sizes=None, seed: int = 0) -> MlpModel:
    """init_mlp (mlp.cpp:184-207)."""
    sizes = list(default_layer_sizes() if layer_sizes is None else layer_sizes)
    arr = (C.c_int32 * len(sizes))(*sizes)
    nw = sum(sizes[l] * sizes[l + 1] for l in range(len(sizes) - 1))
    nb = sum(sizes[1:])
    W = np.empty(max(nw, 1))
    b = np.empty(max(nb, 1))
    st = lib().dso_init_mlp(arr, len(sizes), C.c_uint64(seed),
                            W.ctypes.data_as(C.POINTER(C.c_double)),
                            b.ctypes.data_as(C.POINTER(C.c_double)))
    if st:
        msg = ("need at least input and output layers" if len(sizes) < 2
               else "layer sizes must be positive")
        raise DsoError(status_kind(st), msg)
    ws, bs = split_flat(sizes, W, b)
    out = sizes[-1]
    return MlpModel(sizes, ws, bs, np.zeros(out), np.ones(out), seed)


def validate_model(m: MlpModel) -> None:
    """validate(MlpModel), mlp.cpp:209-226."""
    s = list(m.layer_sizes)
    if len(s) < 2 or len(m.weights) != len(s) - 1 or len(m.biases) != len(m.weights):
        raise DsoError(ErrorKind.InvalidModel, "layer bookkeeping is inconsistent")
    for l, (w, b) in enumerate(zip(m.weights, m.biases)):
        if np.shape(w) != (s[l + 1], s[l]) or np.size(b) != s[l + 1]:
            raise DsoError(ErrorKind.InvalidModel, "weight shapes do not chain")
    if np.size(m.target_mean) != s[-1] or np.size(m.target_std) != s[-1]:
        raise DsoError(ErrorKind.InvalidModel, "normalization stats do not match output")
    if not np.all(np.asarray(m.target_std) > 0.0):
        raise DsoError(ErrorKind.InvalidModel, "target std must be positive")
