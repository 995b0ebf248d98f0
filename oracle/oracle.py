"""ctypes wrappers over the CPU checkers (TEST INFRASTRUCTURE ONLY).

Array conventions (row-major per kernel, float64 unless noted):
params [n,7] = [p0, kappa_pow, gamma, c, t0, alpha, beta]; counts [n,126] uint32;
dcgm [n,8]; fused [n,134]; domain = (core[nc], mem[nm], dev[5]) with
dev = [kappa_vf, pmax_w, vmin_v, vmax_v, mhz_per_unit].
A model is any object with ``layer_sizes``, ``weights`` (list of [out,in]),
``biases`` (list of [out]), ``target_mean`` and ``target_std``.
"""

from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_PORT_SO = os.path.join(_HERE, "liboracle.so")
_REF_SO = os.path.join(_HERE, "_ref", "libdso_ref.so")
_lock = threading.Lock()

_d = C.POINTER(C.c_double)
_u32 = C.POINTER(C.c_uint32)
_u64 = C.POINTER(C.c_uint64)
_i32 = C.POINTER(C.c_int32)
_i64 = C.POINTER(C.c_int64)
_u8 = C.POINTER(C.c_uint8)
_int = C.POINTER(C.c_int)


def build() -> None:
    """Compile liboracle.so (and _ref/ when /root/reference is present)."""
    subprocess.run(["make", "-s", "-C", _HERE], check=True)


def _p(a, t):
    if a is None:
        return None
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def default_threads() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


class _Model:
    def __init__(self, m):
        self.sizes = np.ascontiguousarray(m.layer_sizes, dtype=np.int32).astype(np.intc)
        self.nl = len(self.sizes)
        self.W = _f64(np.concatenate([np.asarray(w, np.float64).ravel() for w in m.weights]))
        self.b = _f64(np.concatenate([np.asarray(b, np.float64).ravel() for b in m.biases]))
        self.mean = _f64(m.target_mean)
        self.std = _f64(m.target_std)


class Port:
    """The C restatement (oracle/dso_oracle.c)."""

    def __init__(self, path: str = _PORT_SO):
        if not os.path.exists(path):
            build()
        L = self.lib = C.CDLL(path)
        L.orc_rng_next.restype = C.c_uint64
        L.orc_rng_next.argtypes = [_u64]
        L.orc_rng_uniform01.restype = C.c_double
        L.orc_rng_uniform01.argtypes = [_u64]
        L.orc_rng_below.restype = C.c_uint64
        L.orc_rng_below.argtypes = [_u64, C.c_uint64]
        L.orc_rng_fork.restype = C.c_uint64
        L.orc_rng_fork.argtypes = [_u64, C.c_uint64]
        L.orc_shuffled_indices.argtypes = [C.c_uint64, _u64, _u64]
        L.orc_power.restype = C.c_double
        L.orc_power.argtypes = [_d, C.c_double, C.c_double, C.c_double]
        L.orc_exec_time.restype = C.c_double
        L.orc_exec_time.argtypes = [_d, C.c_double, C.c_double, C.c_double]
        L.orc_required_voltage_mhz.restype = C.c_double
        L.orc_required_voltage_mhz.argtypes = [C.c_double, _d]
        L.orc_validate_params.argtypes = [_d]
        L.orc_validate_domain.argtypes = [_d, C.c_int, _d, C.c_int, _d]
        L.orc_gen_stream.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, C.c_int64, _d, _u32,
                                     _d, _d, C.c_int]
        L.orc_gen_seeded.argtypes = [_u64, C.c_int64, _d, _u32, _d, _d]
        L.orc_gen_kernel_rho.argtypes = [C.c_uint64, C.c_double, _d, _u32, _d, _d]
        L.orc_featurize.argtypes = [_u32, C.c_int64, _d]
        L.orc_dcgm_mean.argtypes = [_d, C.c_int64, _d, _i64]
        L.orc_fuse.argtypes = [_u32, _d, C.c_int64, _d]
        L.orc_mlp_weight_count.restype = C.c_int64
        L.orc_mlp_weight_count.argtypes = [_int, C.c_int]
        L.orc_mlp_bias_count.restype = C.c_int64
        L.orc_mlp_bias_count.argtypes = [_int, C.c_int]
        L.orc_init_mlp.argtypes = [_int, C.c_int, C.c_uint64, _d, _d]
        L.orc_fit_power.argtypes = [_d, _d, C.c_int, _d]
        L.orc_fit_power.restype = C.c_int
        L.orc_fit_time.argtypes = [_d, _d, C.c_int, _d, _u8]
        L.orc_fit_time.restype = C.c_int
        L.orc_forward_raw.argtypes = [_int, C.c_int, _d, _d, _d, _d, _d, C.c_int64, _d]
        L.orc_predict_params.argtypes = [_int, C.c_int, _d, _d, _d, _d, _d, C.c_int64, _d,
                                         _u8, C.c_int]
        L.orc_mse_loss.restype = C.c_double
        L.orc_mse_loss.argtypes = [_int, C.c_int, _d, _d, _d, _d, C.c_int64]
        L.orc_analytic_gradients.argtypes = [_int, C.c_int, _d, _d, _d, _d, C.c_int64, _d, _d]
        L.orc_numeric_gradients.argtypes = [_int, C.c_int, _d, _d, _d, _d, C.c_int64,
                                            C.c_double, _d, _d]
        L.orc_sgd_epoch.restype = C.c_double
        L.orc_sgd_epoch.argtypes = [_int, C.c_int, _d, _d, _d, _d, C.c_int64, _d, _d,
                                    C.c_double, C.c_int, _u64]
        L.orc_target_stats.argtypes = [_d, C.c_int64, C.c_int, _d, _d]
        L.orc_brute_force.argtypes = [_d, C.c_int64, _d, C.c_int, _d, C.c_int, _d, C.c_double,
                                      C.c_double, _i32, _d, _d, _d, _i32, C.c_int]
        L.orc_eta_sweep.argtypes = [_d, C.c_int64, _d, C.c_int, _d, C.c_int, _d, _d, C.c_int,
                                    C.c_double, _i32, _d, C.c_int]
        L.orc_pipeline.argtypes = [_u32, _d, C.c_int64, _int, C.c_int, _d, _d, _d, _d, _d,
                                   C.c_int, _d, C.c_int, _d, C.c_double, C.c_double, _d, _u8,
                                   _i32, _d, _d, _d, C.c_int]

    # --- rng -----------------------------------------------------------------
    def rng_u64(self, seed: int, n: int) -> np.ndarray:
        s = C.c_uint64(seed)
        return np.array([self.lib.orc_rng_next(C.byref(s)) for _ in range(n)], np.uint64)

    def rng_uniform01(self, seed: int, n: int) -> np.ndarray:
        s = C.c_uint64(seed)
        return np.array([self.lib.orc_rng_uniform01(C.byref(s)) for _ in range(n)])

    def rng_below(self, seed: int, m: int, n: int) -> np.ndarray:
        s = C.c_uint64(seed)
        return np.array([self.lib.orc_rng_below(C.byref(s), m) for _ in range(n)], np.uint64)

    def fork_seeds(self, seed: int, salt0: int, n: int) -> np.ndarray:
        s = C.c_uint64(seed)
        out = []
        for i in range(n):
            child = C.c_uint64(self.lib.orc_rng_fork(C.byref(s), salt0 + i))
            out.append(self.lib.orc_rng_next(C.byref(child)))
        return np.array(out, np.uint64)

    def shuffled_indices(self, seed: int, n: int) -> np.ndarray:
        s = C.c_uint64(seed)
        out = np.empty(n, np.uint64)
        self.lib.orc_shuffled_indices(n, C.byref(s), _p(out, _u64))
        return out

    # --- model maths -----------------------------------------------------------
    def power(self, p, vc, fc, fm) -> float:
        return self.lib.orc_power(_p(_f64(p), _d), vc, fc, fm)

    def exec_time(self, p, vc, fc, fm) -> float:
        return self.lib.orc_exec_time(_p(_f64(p), _d), vc, fc, fm)

    def required_voltage_mhz(self, fc, dev) -> float:
        return self.lib.orc_required_voltage_mhz(fc, _p(_f64(dev), _d))

    def validate_params(self, p) -> int:
        return self.lib.orc_validate_params(_p(_f64(p), _d))

    def validate_domain(self, core, mem, dev) -> int:
        core, mem, dev = _f64(core), _f64(mem), _f64(dev)
        return self.lib.orc_validate_domain(_p(core, _d), len(core), _p(mem, _d), len(mem),
                                            _p(dev, _d))

    # --- generator -------------------------------------------------------------
    def gen_stream(self, root: int, n: int, first: int = 0, salt_base: int = 0,
                   threads: int | None = None, want=("params", "counts", "dcgm", "fused")):
        out = {}
        params = np.empty((n, 7)) if "params" in want else None
        counts = np.empty((n, 126), np.uint32) if "counts" in want else None
        dcgm = np.empty((n, 8)) if "dcgm" in want else None
        fused = np.empty((n, 134)) if "fused" in want else None
        self.lib.orc_gen_stream(root, salt_base, first, n, _p(params, _d), _p(counts, _u32),
                                _p(dcgm, _d), _p(fused, _d), threads or default_threads())
        for k, v in (("params", params), ("counts", counts), ("dcgm", dcgm), ("fused", fused)):
            if v is not None:
                out[k] = v
        return out

    def gen_seeded(self, seeds):
        seeds = np.ascontiguousarray(seeds, np.uint64)
        n = len(seeds)
        params, counts = np.empty((n, 7)), np.empty((n, 126), np.uint32)
        dcgm, fused = np.empty((n, 8)), np.empty((n, 134))
        self.lib.orc_gen_seeded(_p(seeds, _u64), n, _p(params, _d), _p(counts, _u32),
                                _p(dcgm, _d), _p(fused, _d))
        return dict(params=params, counts=counts, dcgm=dcgm, fused=fused)

    def gen_kernel_rho(self, seed: int, rho: float):
        params, counts = np.empty(7), np.empty(126, np.uint32)
        dcgm, fused = np.empty(8), np.empty(134)
        st = self.lib.orc_gen_kernel_rho(seed, rho, _p(params, _d), _p(counts, _u32),
                                         _p(dcgm, _d), _p(fused, _d))
        return st, dict(params=params, counts=counts, dcgm=dcgm, fused=fused)

    # --- features --------------------------------------------------------------
    def featurize(self, counts) -> np.ndarray:
        counts = np.ascontiguousarray(counts, np.uint32).reshape(-1, 126)
        out = np.empty((len(counts), 126))
        self.lib.orc_featurize(_p(counts, _u32), len(counts), _p(out, _d))
        return out

    def dcgm_mean(self, samples):
        samples = _f64(samples).reshape(-1, 8)
        out = np.empty(8)
        bad = C.c_int64(0)
        st = self.lib.orc_dcgm_mean(_p(samples, _d), len(samples), _p(out, _d), C.byref(bad))
        return st, out, bad.value

    def fuse(self, counts, dcgm) -> np.ndarray:
        counts = np.ascontiguousarray(counts, np.uint32).reshape(-1, 126)
        dcgm = _f64(dcgm).reshape(-1, 8)
        out = np.empty((len(counts), 134))
        self.lib.orc_fuse(_p(counts, _u32), _p(dcgm, _d), len(counts), _p(out, _d))
        return out

    # --- MLP -------------------------------------------------------------------
    def init_mlp(self, sizes, seed: int):
        sizes_a = np.ascontiguousarray(sizes, np.intc)
        nl = len(sizes_a)
        nw = self.lib.orc_mlp_weight_count(_p(sizes_a, _int), nl)
        nb = self.lib.orc_mlp_bias_count(_p(sizes_a, _int), nl)
        W, b = np.empty(nw), np.empty(nb)
        st = self.lib.orc_init_mlp(_p(sizes_a, _int), nl, seed, _p(W, _d), _p(b, _d))
        if st:
            raise ValueError(f"init_mlp status {st}")
        ws, bs, ow, ob = [], [], 0, 0
        for l in range(nl - 1):
            fi, fo = int(sizes[l]), int(sizes[l + 1])
            ws.append(W[ow:ow + fi * fo].reshape(fo, fi).copy())
            bs.append(b[ob:ob + fo].copy())
            ow += fi * fo
            ob += fo
        return ws, bs

    def forward_raw(self, model, x) -> np.ndarray:
        m = _Model(model)
        x = _f64(x).reshape(-1, int(m.sizes[0]))
        out = np.empty((len(x), int(m.sizes[-1])))
        self.lib.orc_forward_raw(_p(m.sizes, _int), m.nl, _p(m.W, _d), _p(m.b, _d),
                                 _p(m.mean, _d), _p(m.std, _d), _p(x, _d), len(x), _p(out, _d))
        return out

    def predict_params(self, model, x, threads: int | None = None):
        m = _Model(model)
        x = _f64(x).reshape(-1, int(m.sizes[0]))
        params = np.empty((len(x), 7))
        clamped = np.empty(len(x), np.uint8)
        self.lib.orc_predict_params(_p(m.sizes, _int), m.nl, _p(m.W, _d), _p(m.b, _d),
                                    _p(m.mean, _d), _p(m.std, _d), _p(x, _d), len(x),
                                    _p(params, _d), _p(clamped, _u8),
                                    threads or default_threads())
        return params, clamped.astype(bool)

    # --- training --------------------------------------------------------------
    def mse_loss(self, model, x, y) -> float:
        m = _Model(model)
        x = _f64(x).reshape(-1, int(m.sizes[0]))
        y = _f64(y).reshape(-1, int(m.sizes[-1]))
        return self.lib.orc_mse_loss(_p(m.sizes, _int), m.nl, _p(m.W, _d), _p(m.b, _d),
                                     _p(x, _d), _p(y, _d), len(x))

    def _grads(self, fn, model, x, y, *extra):
        m = _Model(model)
        x = _f64(x).reshape(-1, int(m.sizes[0]))
        y = _f64(y).reshape(-1, int(m.sizes[-1]))
        gW, gb = np.empty_like(m.W), np.empty_like(m.b)
        fn(_p(m.sizes, _int), m.nl, _p(m.W, _d), _p(m.b, _d), _p(x, _d), _p(y, _d), len(x),
           *extra, _p(gW, _d), _p(gb, _d))
        return _split(model.layer_sizes, gW, gb)

    def analytic_gradients(self, model, x, y):
        return self._grads(self.lib.orc_analytic_gradients, model, x, y)

    def numeric_gradients(self, model, x, y, eps: float = 1e-5):
        return self._grads(self.lib.orc_numeric_gradients, model, x, y, C.c_double(eps))

    def target_stats(self, targets):
        t = _f64(targets)
        n, od = t.shape
        mean, std = np.empty(od), np.empty(od)
        deg = self.lib.orc_target_stats(_p(t, _d), n, od, _p(mean, _d), _p(std, _d))
        return mean, std, deg

    def sgd_epoch(self, model, feats, targets, mean, std, lr, batch, rng_state: int):
        """Runs one epoch in place on a copy; returns (loss, weights, biases, rng_state)."""
        m = _Model(model)
        feats = _f64(feats)
        targets = _f64(targets)
        mean, std = _f64(mean), _f64(std)
        s = C.c_uint64(rng_state)
        loss = self.lib.orc_sgd_epoch(_p(m.sizes, _int), m.nl, _p(m.W, _d), _p(m.b, _d),
                                      _p(feats, _d), _p(targets, _d), len(feats), _p(mean, _d),
                                      _p(std, _d), lr, batch, C.byref(s))
        ws, bs = _split(model.layer_sizes, m.W, m.b)
        return loss, ws, bs, s.value

    # --- param_fit (param_fit.cpp:43-247) ---------------------------------------
    def fit_power(self, cfg, power):
        """(status, [p0, kappa_pow, gamma, c, mape_pct, constraint_active])."""
        cfg = _f64(cfg).reshape(-1, 3)
        power = _f64(power)
        out = np.zeros(6)
        st = self.lib.orc_fit_power(_p(cfg, _d), _p(power, _d), len(power), _p(out, _d))
        return st, out

    def fit_time(self, cfg, time_s):
        """(status, [t0, alpha, beta, mape_pct, constraint_active, partial, iterations,
        rss], branch[S] (1 = memory))."""
        cfg = _f64(cfg).reshape(-1, 3)
        t = _f64(time_s)
        out = np.zeros(8)
        br = np.zeros(len(t), np.uint8)
        st = self.lib.orc_fit_time(_p(cfg, _d), _p(t, _d), len(t), _p(out, _d), _p(br, _u8))
        return st, out, br

    # --- sweep -----------------------------------------------------------------
    def brute_force(self, params, core, mem, dev, eta, pmax, threads: int | None = None):
        params = _f64(params).reshape(-1, 7)
        core, mem, dev = _f64(core), _f64(mem), _f64(dev)
        n = len(params)
        idx = np.empty(n, np.int32)
        cost, energy, time = np.empty(n), np.empty(n), np.empty(n)
        ks = np.empty(n, np.int32)
        st = self.lib.orc_brute_force(_p(params, _d), n, _p(core, _d), len(core), _p(mem, _d),
                                      len(mem), _p(dev, _d), eta, pmax, _p(idx, _i32),
                                      _p(cost, _d), _p(energy, _d), _p(time, _d), _p(ks, _i32),
                                      threads or default_threads())
        return st, dict(idx=idx, cost=cost, energy=energy, time=time, kstatus=ks)

    def eta_sweep(self, params, core, mem, dev, etas, pmax, threads: int | None = None):
        params = _f64(params).reshape(-1, 7)
        core, mem, dev, etas = _f64(core), _f64(mem), _f64(dev), _f64(etas)
        n = len(params)
        idx = np.empty((len(etas), n), np.int32)
        cost = np.empty((len(etas), n))
        st = self.lib.orc_eta_sweep(_p(params, _d), n, _p(core, _d), len(core), _p(mem, _d),
                                    len(mem), _p(dev, _d), _p(etas, _d), len(etas), pmax,
                                    _p(idx, _i32), _p(cost, _d), threads or default_threads())
        return st, dict(idx=idx, cost=cost)

    def pipeline(self, counts, dcgm, model, core, mem, dev, eta, pmax,
                 threads: int | None = None):
        m = _Model(model)
        counts = np.ascontiguousarray(counts, np.uint32).reshape(-1, 126)
        dcgm = _f64(dcgm).reshape(-1, 8)
        core, mem, dev = _f64(core), _f64(mem), _f64(dev)
        n = len(counts)
        params = np.empty((n, 7))
        clamped = np.empty(n, np.uint8)
        idx = np.empty(n, np.int32)
        cost, energy, time = np.empty(n), np.empty(n), np.empty(n)
        st = self.lib.orc_pipeline(_p(counts, _u32), _p(dcgm, _d), n, _p(m.sizes, _int), m.nl,
                                   _p(m.W, _d), _p(m.b, _d), _p(m.mean, _d), _p(m.std, _d),
                                   _p(core, _d), len(core), _p(mem, _d), len(mem), _p(dev, _d),
                                   eta, pmax, _p(params, _d), _p(clamped, _u8), _p(idx, _i32),
                                   _p(cost, _d), _p(energy, _d), _p(time, _d),
                                   threads or default_threads())
        return st, dict(params=params, clamped=clamped.astype(bool), idx=idx, cost=cost,
                        energy=energy, time=time)


def _split(sizes, W, b):
    ws, bs, ow, ob = [], [], 0, 0
    for l in range(len(sizes) - 1):
        fi, fo = int(sizes[l]), int(sizes[l + 1])
        ws.append(W[ow:ow + fi * fo].reshape(fo, fi).copy())
        bs.append(b[ob:ob + fo].copy())
        ow += fi * fo
        ob += fo
    return ws, bs


class Ref:
    """The reference itself: proj/src/optimizer.cpp + headers (oracle/_ref)."""

    def __init__(self, path: str = _REF_SO):
        if not os.path.exists(path):
            build()
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} not built (reference tree absent?)")
        L = self.lib = C.CDLL(path)
        L.ref_last_message.restype = C.c_char_p
        L.ref_validate_domain.argtypes = [_d, C.c_int, _d, C.c_int, _d]
        opt = [_d, C.c_int64, _d, C.c_int, _d, C.c_int, _d, C.c_double, C.c_double, _d, _d,
               _d, _d, _i64]
        L.ref_brute_force_config.argtypes = opt + [_i32, C.c_int]
        L.ref_optimal_config.argtypes = opt + [_u8, _d, _i32, C.c_int]
        L.ref_model_eval.argtypes = [C.c_int, _d, C.c_double, C.c_double, C.c_double,
                                     C.c_double, C.c_double, _d]
        L.ref_vf_eval.argtypes = [C.c_int, C.c_double, _d, _d]
        L.ref_validate_params.argtypes = [_d]
        L.ref_rng_u64.argtypes = [C.c_uint64, C.c_int64, _u64]
        L.ref_rng_uniform01.argtypes = [C.c_uint64, C.c_int64, _d]
        L.ref_rng_below.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _u64]
        L.ref_fork_seeds.argtypes = [C.c_uint64, C.c_uint64, C.c_int64, _u64]
        L.ref_shuffled_indices.argtypes = [C.c_uint64, C.c_uint64, _u64]

    def message(self) -> str:
        return self.lib.ref_last_message().decode()

    def validate_domain(self, core, mem, dev) -> int:
        core, mem, dev = _f64(core), _f64(mem), _f64(dev)
        return self.lib.ref_validate_domain(_p(core, _d), len(core), _p(mem, _d), len(mem),
                                            _p(dev, _d))

    def _opt(self, structured, params, core, mem, dev, eta, pmax, threads):
        params = _f64(params).reshape(-1, 7)
        core, mem, dev = _f64(core), _f64(mem), _f64(dev)
        n = len(params)
        best = np.empty((n, 3))
        cost, energy, time = np.empty(n), np.empty(n), np.empty(n)
        cand = np.empty(n, np.int64)
        ks = np.empty(n, np.int32)
        args = [_p(params, _d), n, _p(core, _d), len(core), _p(mem, _d), len(mem), _p(dev, _d),
                eta, pmax, _p(best, _d), _p(cost, _d), _p(energy, _d), _p(time, _d),
                _p(cand, _i64)]
        out = dict(best=best, cost=cost, energy=energy, time=time, candidates=cand, kstatus=ks)
        if structured:
            fb = np.empty(n, np.uint8)
            pre = np.empty((n, 3))
            self.lib.ref_optimal_config(*args, _p(fb, _u8), _p(pre, _d), _p(ks, _i32),
                                        threads or default_threads())
            out.update(fallback=fb.astype(bool), presnap=pre)
        else:
            self.lib.ref_brute_force_config(*args, _p(ks, _i32), threads or default_threads())
        # grid index of the chosen pair (fc_idx * nm + fm_idx)
        fi = np.searchsorted(core, best[:, 1])
        fj = np.searchsorted(mem, best[:, 2])
        out["idx"] = np.where(ks == 0, fi * len(mem) + fj, -1).astype(np.int32)
        return out

    def brute_force_config(self, params, core, mem, dev, eta, pmax, threads=None):
        return self._opt(False, params, core, mem, dev, eta, pmax, threads)

    def optimal_config(self, params, core, mem, dev, eta, pmax, threads=None):
        return self._opt(True, params, core, mem, dev, eta, pmax, threads)

    def model_eval(self, which: str, p, vc, fc, fm, eta=0.0, pmax=0.0):
        code = {"power": 0, "exec_time": 1, "energy": 2, "cost": 3}[which]
        out = C.c_double()
        st = self.lib.ref_model_eval(code, _p(_f64(p), _d), vc, fc, fm, eta, pmax,
                                     C.byref(out))
        return st, out.value

    def vf_eval(self, which: str, x, dev):
        code = {"max_core_freq": 0, "required_voltage": 1, "required_voltage_mhz": 2}[which]
        out = C.c_double()
        st = self.lib.ref_vf_eval(code, x, _p(_f64(dev), _d), C.byref(out))
        return st, out.value

    def validate_params(self, p) -> int:
        return self.lib.ref_validate_params(_p(_f64(p), _d))

    def rng_u64(self, seed, n):
        out = np.empty(n, np.uint64)
        self.lib.ref_rng_u64(seed, n, _p(out, _u64))
        return out

    def rng_uniform01(self, seed, n):
        out = np.empty(n)
        self.lib.ref_rng_uniform01(seed, n, _p(out, _d))
        return out

    def rng_below(self, seed, m, n):
        out = np.empty(n, np.uint64)
        self.lib.ref_rng_below(seed, m, n, _p(out, _u64))
        return out

    def fork_seeds(self, seed, salt0, n):
        out = np.empty(n, np.uint64)
        self.lib.ref_fork_seeds(seed, salt0, n, _p(out, _u64))
        return out

    def shuffled_indices(self, seed, n):
        out = np.empty(n, np.uint64)
        self.lib.ref_shuffled_indices(seed, n, _p(out, _u64))
        return out


_port = None
_ref = None


def port() -> Port:
    global _port
    with _lock:
        if _port is None:
            _port = Port()
        return _port


def ref() -> Ref:
    global _ref
    with _lock:
        if _ref is None:
            _ref = Ref()
        return _ref
