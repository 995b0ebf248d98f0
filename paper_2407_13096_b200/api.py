"""Batched DSO hot path on one B200 — host side of the C-ABI (include/dso_b200.h).

Each method replaces one reference function for a whole batch of GPU kernels
(citations are to /root/reference/proj):

    Context.featurize          featurize + FusedFeatures::as_vector
                               (ptx_features.cpp:311-329, mlp.cpp:158-165)
    Context.dcgm_mean          load_dcgm_samples' per-metric mean (telemetry.cpp:73-89)
    Context.predict_params     predict_params / forward_raw (mlp.cpp:232-253)
    Context.brute_force_config brute_force_config (optimizer.cpp:90-117), FP32
    Context.brute_force_config_exact  the same in FP64, bit-exact, reference AoS layout
    Context.eta_sweep          brute_force_config at many etas
    Context.pipeline           counts + DCGM -> features -> predict -> sweep -> argmin
    Context.gen_synthetic      gen_kernel for a seeded stream (sim_harness.cpp:118-144)
    Context.train_grad / train_apply   analytic_gradients + SGD update (mlp.cpp:84-112,265-289)

Device arrays are torch CUDA tensors in structure-of-arrays layout
[rows, ld] (see the header).  Errors raise DsoError with the reference's
ErrorKind.  There is no CPU fallback: a missing library or GPU raises.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from ._lib import DSO_HOST, DsoError, ErrorKind, lib, status_kind
from .domain import DvfsDomain
from .model import MlpModel, split_flat, validate_model

try:
    import torch
except ImportError:  # pragma: no cover - torch is part of the image
    torch = None

_dp = C.POINTER(C.c_double)


def _ptr(x) -> int | None:
    if x is None:
        return None
    if torch is not None and isinstance(x, torch.Tensor):
        return x.data_ptr()
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    raise TypeError(f"unsupported array type {type(x)}")


def _is_cuda(x) -> bool:
    return torch is not None and isinstance(x, torch.Tensor) and x.is_cuda


def _check(t, dtype, rows: int | None, name: str):
    if not _is_cuda(t):
        raise DsoError(ErrorKind.InvalidArgument, f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise DsoError(ErrorKind.InvalidArgument, f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise DsoError(ErrorKind.InvalidArgument, f"{name} must be contiguous")
    if rows is not None and (t.dim() != 2 or t.shape[0] != rows):
        raise DsoError(ErrorKind.InvalidArgument,
                       f"{name} must have shape [{rows}, ld], got {tuple(t.shape)}")


_TORCH_OF = {}
if torch is not None:
    _TORCH_OF = {np.int32: (torch.int32,), np.uint32: (torch.int32,), np.float32: (torch.float32,),
                 np.int64: (torch.int64,), np.float64: (torch.float64,)}


def _check_host(t, dtypes, rows: int | None, name: str, dim: int = 2):
    """Host-buffer (numpy / CPU tensor) twin of _check: the library reads these
    through raw pointers, so dtype, rank, row count and contiguity must be exact."""
    if _is_cuda(t):
        raise DsoError(ErrorKind.InvalidArgument, f"{name}: mixed host and device buffers")
    if torch is not None and isinstance(t, torch.Tensor):
        ok = t.dtype in sum((_TORCH_OF[d] for d in dtypes), ())
        contiguous = t.is_contiguous()
        shape = tuple(t.shape)
        got = t.dtype
    elif isinstance(t, np.ndarray):
        ok = t.dtype.type in dtypes
        contiguous = t.flags.c_contiguous
        shape = t.shape
        got = t.dtype
    else:
        raise DsoError(ErrorKind.InvalidArgument, f"{name}: unsupported array type {type(t)}")
    if not ok:
        raise DsoError(ErrorKind.InvalidArgument,
                       f"{name} must be {'/'.join(d.__name__ for d in dtypes)}, got {got}")
    if not contiguous:
        raise DsoError(ErrorKind.InvalidArgument, f"{name} must be contiguous")
    if len(shape) != dim or (rows is not None and shape[0] != rows):
        want = f"[{rows}, ld]" if dim == 2 else "1-D"
        raise DsoError(ErrorKind.InvalidArgument, f"{name} must have shape {want}, got {shape}")


class Context:
    """One device's state (stream, domain tables, model); dso_ctx in the C-ABI."""

    def __init__(self, device: int = 0, use_torch_stream: bool = True):
        if torch is None or not torch.cuda.is_available():
            raise DsoError(ErrorKind.IoError, "no CUDA device available")
        self._lib = lib()
        self.device = device
        h = C.c_void_p()
        st = self._lib.dso_ctx_create(device, C.byref(h))
        if st:
            raise DsoError(status_kind(st), f"dso_ctx_create(device={device}) failed")
        self._h = h
        self.domain: DvfsDomain | None = None
        self.model: MlpModel | None = None
        if use_torch_stream:
            with torch.cuda.device(device):
                self.set_stream(torch.cuda.current_stream(device))

    # -- plumbing ---------------------------------------------------------------
    def _raise(self, st: int):
        if st:
            msg = self._lib.dso_last_error(self._h).decode()
            raise DsoError(status_kind(st), msg)

    def close(self):
        if getattr(self, "_h", None):
            self._lib.dso_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    def set_stream(self, stream) -> None:
        handle = None if stream is None else getattr(stream, "cuda_stream", stream)
        self._raise(self._lib.dso_ctx_set_stream(self._h, C.c_void_p(handle)))

    def sync(self) -> None:
        self._raise(self._lib.dso_sync(self._h))

    def set_option(self, key: str, value: int) -> None:
        """dso_set_option: verification/tuning switches: "fast_sweep" (0/1, exact
        group-minimum sweep), "eta_prune" (0/1, eta sweep over the candidate
        pairs only), "dense_csr", "train_tc", "mlp_engine" (0 = FMA-pipe predictor kernel; 1 =
        tcgen05 3xTF32 kernel for predict and the fused pipelines; 2 = auto, the
        default: tensor cores for predict and the CSR pipeline, FMA pipe for dense)."""
        self._raise(self._lib.dso_set_option(self._h, key.encode(), int(value)))

    @property
    def launch_count(self) -> int:
        """Device kernels launched through this context (evidence counter)."""
        return int(self._lib.dso_launch_count(self._h))

    def counters(self, reset: bool = False) -> dict:
        """dso_get_counters: work the kernels actually issued on this context
        (tcgen05 layer-1 / layer-2 k-steps, 128-kernel tiles)."""
        buf = (C.c_uint64 * 3)()
        self._raise(self._lib.dso_get_counters(self._h, buf, 3, 1 if reset else 0))
        return {"tc_l1_ksteps": int(buf[0]), "tc_l2_ksteps": int(buf[1]), "tc_tiles": int(buf[2])}

    def _empty(self, shape, dtype):
        return torch.empty(shape, dtype=dtype, device=f"cuda:{self.device}")

    # -- state --------------------------------------------------------------------
    def set_domain(self, domain: DvfsDomain) -> None:
        """validate(DvfsDomain) (optimizer.cpp:58-88) + table upload."""
        core = np.ascontiguousarray(domain.core_freqs_mhz, np.float64)
        mem = np.ascontiguousarray(domain.mem_freqs_mhz, np.float64)
        dev = domain.dev.as_array()
        self._raise(self._lib.dso_set_domain(self._h, core.ctypes.data_as(_dp), len(core),
                                             mem.ctypes.data_as(_dp), len(mem),
                                             dev.ctypes.data_as(_dp)))
        self.domain = domain

    def set_model(self, model: MlpModel) -> None:
        """validate(MlpModel) (mlp.cpp:209-226) + packed FP32 upload."""
        validate_model(model)
        W, b = model.flat()
        sizes = (C.c_int32 * len(model.layer_sizes))(*model.layer_sizes)
        mean = np.ascontiguousarray(model.target_mean, np.float64)
        std = np.ascontiguousarray(model.target_std, np.float64)
        self._raise(self._lib.dso_set_model(self._h, sizes, len(model.layer_sizes),
                                            W.ctypes.data_as(_dp), b.ctypes.data_as(_dp),
                                            mean.ctypes.data_as(_dp), std.ctypes.data_as(_dp)))
        self.model = model

    def get_model(self) -> MlpModel:
        """The device model (e.g. after training) in the reference layout."""
        m = self.model
        W, b = m.flat()
        W2, b2 = np.empty_like(W), np.empty_like(b)
        self._raise(self._lib.dso_get_model(self._h, W2.ctypes.data_as(_dp),
                                            b2.ctypes.data_as(_dp)))
        ws, bs = split_flat(m.layer_sizes, W2, b2)
        return MlpModel(list(m.layer_sizes), ws, bs, np.array(m.target_mean),
                        np.array(m.target_std), m.seed)

    # -- synthetic inputs -----------------------------------------------------------
    def gen_synthetic(self, n: int, root: int, salt_base: int = 0, first: int = 0,
                      ld: int | None = None, params=True, counts=True, dcgm=True):
        """gen_kernel(Rng(root).fork(salt_base+first+k).next_u64()) for k < n."""
        ld = n if ld is None else ld
        out = {}
        p = self._empty((7, ld), torch.float32) if params else None
        c = self._empty((126, ld), torch.int32) if counts else None
        d = self._empty((8, ld), torch.float32) if dcgm else None
        self._raise(self._lib.dso_gen_synthetic(self._h, C.c_uint64(root), C.c_uint64(salt_base),
                                                first, n, ld, _ptr(p), _ptr(c), _ptr(d)))
        if params:
            out["params"] = p
        if counts:
            out["counts"] = c
        if dcgm:
            out["dcgm"] = d
        return out

    def gen_synthetic_csr(self, n: int, root: int, salt_base: int = 0, first: int = 0,
                          ld: int | None = None):
        """The synthetic stream with sparse counts: row_ptr [n+1] int64 (24k),
        entries [24n] int32 ((count << 7) | slot), dcgm [8, ld]."""
        ld = n if ld is None else ld
        rp = self._empty((n + 1,), torch.int64)
        ent = self._empty((max(24 * n, 1),), torch.int32)
        d = self._empty((8, ld), torch.float32)
        self._raise(self._lib.dso_gen_synthetic_csr(self._h, C.c_uint64(root),
                                                    C.c_uint64(salt_base), first, n, _ptr(rp),
                                                    _ptr(ent), _ptr(d), ld))
        return {"row_ptr": rp, "entries": ent, "dcgm": d}

    # -- feature stage ----------------------------------------------------------------
    def featurize(self, counts, dcgm, n: int | None = None, out=None):
        _check(counts, torch.int32, 126, "counts")
        _check(dcgm, torch.float32, 8, "dcgm")
        ld = counts.shape[1]
        n = ld if n is None else n
        if dcgm.shape[1] != ld:
            raise DsoError(ErrorKind.InvalidArgument, "counts and dcgm must share ld")
        fused = self._empty((134, ld), torch.float32) if out is None else out
        self._raise(self._lib.dso_featurize(self._h, _ptr(counts), _ptr(dcgm), n, ld,
                                            _ptr(fused)))
        return fused

    def featurize_u64(self, counts, dcgm, n: int | None = None, out=None):
        """featurize + as_vector on the reference's 64-bit counts: counts CUDA int64
        [126, ld] (uint64 bit patterns), dcgm float32 [8, ld] -> fused [134, ld]."""
        _check(counts, torch.int64, 126, "counts")
        _check(dcgm, torch.float32, 8, "dcgm")
        ld = counts.shape[1]
        n = ld if n is None else n
        if dcgm.shape[1] != ld:
            raise DsoError(ErrorKind.InvalidArgument, "counts and dcgm must share ld")
        fused = self._empty((134, ld), torch.float32) if out is None else out
        self._raise(self._lib.dso_featurize_u64(self._h, _ptr(counts), _ptr(dcgm), n, ld,
                                                _ptr(fused)))
        return fused

    def dcgm_mean(self, samples, n: int | None = None):
        """samples: float64 [rows, 8, ld] -> (mean float32 [8, ld], bad_row int64 [ld])."""
        if not _is_cuda(samples) or samples.dtype != torch.float64 or samples.dim() != 3 \
                or samples.shape[1] != 8:
            raise DsoError(ErrorKind.InvalidArgument, "samples must be CUDA float64 [rows,8,ld]")
        rows, _, ld = samples.shape
        n = ld if n is None else n
        out = self._empty((8, ld), torch.float32)
        bad = self._empty((ld,), torch.int64)
        st = self._lib.dso_dcgm_mean(self._h, _ptr(samples.contiguous()), rows, n, ld,
                                     _ptr(out), _ptr(bad))
        if st and status_kind(st) == ErrorKind.OutOfRange:
            rowk = bad[:n].cpu().numpy()
            nz = np.flatnonzero(rowk)
            if len(nz) == 0:
                self._raise(st)
            first = int(nz[0])
            raise DsoError(ErrorKind.OutOfRange,
                           f"kernel {first}: row {int(rowk[first])}: metric value outside [0, 1]")
        self._raise(st)
        return out, bad

    # -- predictor ------------------------------------------------------------------
    def predict_params(self, fused, n: int | None = None, want_raw: bool = False):
        """predict_params for every column: (params [7, ld], clamped [ld] bool, raw|None).
        A model with another chain (TrainConfig.layer_sizes) reads [sizes[0], ld] and
        returns raw [sizes[-1], ld] (forward_raw); params / clamped need 7 outputs."""
        sizes = self._sizes()
        _check(fused, torch.float32, sizes[0], "fused")
        ld = fused.shape[1]
        n = ld if n is None else n
        params = self._empty((7, ld), torch.float32) if sizes[-1] == 7 else None
        clamped = self._empty((ld,), torch.uint8) if sizes[-1] == 7 else None
        raw = self._empty((sizes[-1], ld), torch.float32) if want_raw else None
        self._raise(self._lib.dso_predict(self._h, _ptr(fused), n, ld, _ptr(params),
                                          _ptr(clamped), _ptr(raw)))
        return params, (clamped.bool() if clamped is not None else None), raw

    def _sizes(self):
        return list(self.model.layer_sizes) if self.model is not None else [134, 100, 50, 25, 7]

    # -- sweep ----------------------------------------------------------------------
    def brute_force_config(self, params, eta: float, pmax_w: float | None = None,
                           n: int | None = None):
        """FP32 batch of brute_force_config: dict(idx, cost, energy, time, kstatus)."""
        _check(params, torch.float32, 7, "params")
        ld = params.shape[1]
        n = ld if n is None else n
        pmax = self.domain.dev.pmax_w if pmax_w is None else pmax_w
        out = {k: self._empty((ld,), torch.float32) for k in ("cost", "energy", "time")}
        out["idx"] = self._empty((ld,), torch.int32)
        out["kstatus"] = self._empty((ld,), torch.int32)
        self._raise(self._lib.dso_sweep(self._h, _ptr(params), n, ld, eta, pmax,
                                        _ptr(out["idx"]), _ptr(out["cost"]),
                                        _ptr(out["energy"]), _ptr(out["time"]),
                                        _ptr(out["kstatus"])))
        return out

    def brute_force_config_exact(self, params_aos, eta: float, pmax_w: float | None = None):
        """FP64, bit-exact brute_force_config over KernelModelParams[n] (AoS [n, 7]).
        Accepts a CUDA float64 tensor or a host numpy array (staged by the library)."""
        pmax = self.domain.dev.pmax_w if pmax_w is None else pmax_w
        if _is_cuda(params_aos):
            if params_aos.dtype != torch.float64 or params_aos.dim() != 2 \
                    or params_aos.shape[1] != 7 or not params_aos.is_contiguous():
                raise DsoError(ErrorKind.InvalidArgument, "params must be contiguous f64 [n, 7]")
            n = params_aos.shape[0]
            out = {k: self._empty((n,), torch.float64) for k in ("cost", "energy", "time")}
            out["idx"] = self._empty((n,), torch.int32)
            out["kstatus"] = self._empty((n,), torch.int32)
            flags = 0
        else:
            params_aos = np.ascontiguousarray(params_aos, np.float64).reshape(-1, 7)
            n = len(params_aos)
            out = {k: np.empty(n) for k in ("cost", "energy", "time")}
            out["idx"] = np.empty(n, np.int32)
            out["kstatus"] = np.empty(n, np.int32)
            flags = DSO_HOST
        self._raise(self._lib.dso_sweep_f64(self._h, _ptr(params_aos), n, eta, pmax,
                                            _ptr(out["idx"]), _ptr(out["cost"]),
                                            _ptr(out["energy"]), _ptr(out["time"]),
                                            _ptr(out["kstatus"]), flags))
        return out

    def optimal_config(self, params_aos, eta: float, pmax_w: float | None = None):
        """FP64, bit-exact optimal_config (optimizer.cpp:119-205) over KernelModelParams[n]
        (AoS [n, 7]): dict(idx, cost, energy, time, candidates, fallback, presnap [n, 3],
        kstatus).  CUDA float64 tensor or host numpy array (staged by the library)."""
        pmax = self.domain.dev.pmax_w if pmax_w is None else pmax_w
        if _is_cuda(params_aos):
            if params_aos.dtype != torch.float64 or params_aos.dim() != 2 \
                    or params_aos.shape[1] != 7 or not params_aos.is_contiguous():
                raise DsoError(ErrorKind.InvalidArgument, "params must be contiguous f64 [n, 7]")
            n = params_aos.shape[0]
            out = {k: self._empty((n,), torch.float64) for k in ("cost", "energy", "time")}
            out["idx"] = self._empty((n,), torch.int32)
            out["kstatus"] = self._empty((n,), torch.int32)
            out["candidates"] = self._empty((n,), torch.int64)
            out["fallback"] = self._empty((n,), torch.uint8)
            out["presnap"] = self._empty((n, 3), torch.float64)
            flags = 0
        else:
            params_aos = np.ascontiguousarray(params_aos, np.float64).reshape(-1, 7)
            n = len(params_aos)
            out = {k: np.empty(n) for k in ("cost", "energy", "time")}
            out["idx"] = np.empty(n, np.int32)
            out["kstatus"] = np.empty(n, np.int32)
            out["candidates"] = np.empty(n, np.int64)
            out["fallback"] = np.empty(n, np.uint8)
            out["presnap"] = np.empty((n, 3))
            flags = DSO_HOST
        self._raise(self._lib.dso_optimal_config(
            self._h, _ptr(params_aos), n, eta, pmax, _ptr(out["idx"]), _ptr(out["cost"]),
            _ptr(out["energy"]), _ptr(out["time"]), _ptr(out["candidates"]),
            _ptr(out["fallback"]), _ptr(out["presnap"]), _ptr(out["kstatus"]), flags))
        return out

    def param_fit(self, cfg, power=None, time=None):
        """Batched fit_power / fit_time (param_fit.cpp:43-247) of n kernels measured on one
        grid.  cfg [S, 3] = (vc, fc_mhz, fm_mhz); power / time [S, n] float64 (CUDA tensors or
        host numpy; either may be None).  Returns dict(pfit [6, n], pstatus [n],
        tfit [8, n], tstatus [n]) — see include/dso_b200.h for the rows."""
        cfg = np.ascontiguousarray(cfg, np.float64).reshape(-1, 3)
        S = len(cfg)
        ref = power if power is not None else time
        host = not _is_cuda(ref)
        if host:
            power = None if power is None else np.ascontiguousarray(power, np.float64)
            time = None if time is None else np.ascontiguousarray(time, np.float64)
            n = ref.shape[1]
            mk = lambda shape, dt: np.empty(shape, dt)  # noqa: E731
        else:
            for t in (power, time):
                if t is not None and (t.dtype != torch.float64 or not t.is_contiguous()):
                    raise DsoError(ErrorKind.InvalidArgument, "power/time must be contiguous f64")
            n = ref.shape[1]
            mk = lambda shape, dt: self._empty(shape, {np.float64: torch.float64,  # noqa: E731
                                                        np.int32: torch.int32}[dt])
        out = {}
        if power is not None:
            out["pfit"], out["pstatus"] = mk((6, n), np.float64), mk((n,), np.int32)
        if time is not None:
            out["tfit"], out["tstatus"] = mk((8, n), np.float64), mk((n,), np.int32)
        self._raise(self._lib.dso_param_fit(
            self._h, cfg.ctypes.data, S, _ptr(power), _ptr(time), n, n, _ptr(out.get("pfit")),
            _ptr(out.get("pstatus")), _ptr(out.get("tfit")), _ptr(out.get("tstatus")),
            DSO_HOST if host else 0))
        return out

    def eta_sweep(self, params, etas, pmax_w: float | None = None, n: int | None = None):
        """brute_force_config at every eta: (idx [n_eta, ld], cost [n_eta, ld])."""
        _check(params, torch.float32, 7, "params")
        ld = params.shape[1]
        n = ld if n is None else n
        etas = np.ascontiguousarray(etas, np.float64)
        pmax = self.domain.dev.pmax_w if pmax_w is None else pmax_w
        idx = self._empty((len(etas), ld), torch.int32)
        cost = self._empty((len(etas), ld), torch.float32)
        self._raise(self._lib.dso_eta_sweep(self._h, _ptr(params), n, ld,
                                            etas.ctypes.data_as(_dp), len(etas), pmax,
                                            _ptr(idx), _ptr(cost), ld))
        return idx, cost

    # -- fused pipeline ---------------------------------------------------------------
    def pipeline(self, counts, dcgm, eta: float, pmax_w: float | None = None,
                 n: int | None = None, want_params: bool = False, out: dict | None = None):
        """counts [126, ld] int32 + dcgm [8, ld] float32 -> dict(idx, cost, energy, time
        [, params, clamped]).  CUDA tensors run on the device; CPU tensors / numpy arrays
        (pinned for full speed) are staged through the device in overlapped chunks."""
        pmax = self.domain.dev.pmax_w if pmax_w is None else pmax_w
        host = not _is_cuda(counts)
        ld = counts.shape[1]
        n = ld if n is None else n
        if out is None:
            out = self.alloc_pipeline_out(ld, host=host, want_params=want_params,
                                          like=counts)
        if not host:
            _check(counts, torch.int32, 126, "counts")
            _check(dcgm, torch.float32, 8, "dcgm")
        else:
            _check_host(counts, (np.uint32, np.int32), 126, "counts")
            _check_host(dcgm, (np.float32,), 8, "dcgm")
        if dcgm.shape[1] != ld:
            raise DsoError(ErrorKind.InvalidArgument, "counts and dcgm must share ld")
        if not 0 <= n <= ld:
            raise DsoError(ErrorKind.InvalidArgument, "batch requires 0 <= n <= ld")
        self._raise(self._lib.dso_pipeline(
            self._h, _ptr(counts), _ptr(dcgm), n, ld, eta, pmax, _ptr(out.get("params")),
            _ptr(out.get("clamped")), _ptr(out["idx"]), _ptr(out.get("cost")),
            _ptr(out.get("energy")), _ptr(out.get("time")), DSO_HOST if host else 0))
        return out

    def pipeline_csr(self, row_ptr, entries, dcgm, eta: float, pmax_w: float | None = None,
                     n: int | None = None, ent_base: int = 0, want_params: bool = False,
                     out: dict | None = None):
        """Fused pipeline on sparse counts (dso_pipeline_csr): row_ptr [n+1] int64,
        entries int32 ((count << 7) | slot), dcgm [8, ld] float32.  CUDA tensors run
        on the device; CPU (pinned) tensors / numpy go through the chunked host path."""
        pmax = self.domain.dev.pmax_w if pmax_w is None else pmax_w
        host = not _is_cuda(row_ptr)
        if host:
            _check_host(row_ptr, (np.int64,), None, "row_ptr", dim=1)
            _check_host(entries, (np.int32, np.uint32), None, "entries", dim=1)
            _check_host(dcgm, (np.float32,), 8, "dcgm")
        else:
            for t, dt, name in ((row_ptr, torch.int64, "row_ptr"), (entries, torch.int32, "entries")):
                if not _is_cuda(t) or t.dtype != dt or t.dim() != 1 or not t.is_contiguous():
                    raise DsoError(ErrorKind.InvalidArgument,
                                   f"{name} must be a contiguous 1-D CUDA {dt} tensor")
            _check(dcgm, torch.float32, 8, "dcgm")
        ld = dcgm.shape[1]
        n = ld if n is None else n
        if not 0 <= n <= ld:
            raise DsoError(ErrorKind.InvalidArgument, "batch requires 0 <= n <= ld")
        if row_ptr.shape[0] < n + 1:
            raise DsoError(ErrorKind.InvalidArgument, "row_ptr needs n + 1 entries")
        if out is None:
            out = self.alloc_pipeline_out(ld, host=host, want_params=want_params, like=dcgm)
        self._raise(self._lib.dso_pipeline_csr(
            self._h, _ptr(row_ptr), _ptr(entries), C.c_uint64(ent_base), _ptr(dcgm), n, ld, eta,
            pmax, _ptr(out.get("params")), _ptr(out.get("clamped")), _ptr(out["idx"]),
            _ptr(out.get("cost")), _ptr(out.get("energy")), _ptr(out.get("time")),
            DSO_HOST if host else 0))
        return out

    def alloc_pipeline_out(self, ld: int, host: bool = False, want_params: bool = False,
                           like=None, pin: bool = True):
        if host:
            if torch is not None and (like is None or isinstance(like, torch.Tensor)):
                mk = lambda shape, dt: torch.empty(shape, dtype=dt, pin_memory=pin)  # noqa: E731
                f32, i32, u8 = torch.float32, torch.int32, torch.uint8
            else:
                mk = lambda shape, dt: np.empty(shape, dt)  # noqa: E731
                f32, i32, u8 = np.float32, np.int32, np.uint8
        else:
            mk = self._empty
            f32, i32, u8 = torch.float32, torch.int32, torch.uint8
        out = {"idx": mk((ld,), i32), "cost": mk((ld,), f32), "energy": mk((ld,), f32),
               "time": mk((ld,), f32)}
        if want_params:
            out["params"] = mk((7, ld), f32)
            out["clamped"] = mk((ld,), u8)
        return out

    # -- training ---------------------------------------------------------------------
    @property
    def n_model_params(self) -> int:
        return int(self._lib.dso_model_param_count(self._h))

    def train_grad(self, x, y_std, n: int | None = None, grad=None):
        """Sum over the batch of per-sample gradients of 0.5*||out - y||^2 (device model).
        Returns (grad float32 [n_params], loss_sum float)."""
        sizes = self._sizes()
        _check(x, torch.float32, sizes[0], "x")
        _check(y_std, torch.float32, sizes[-1], "y_std")
        ld = x.shape[1]
        n = ld if n is None else n
        if grad is None:
            grad = self._empty((self.n_model_params,), torch.float32)
        loss = self._empty((1,), torch.float64)
        self._raise(self._lib.dso_train_grad(self._h, _ptr(x), _ptr(y_std), n, ld, _ptr(grad),
                                             _ptr(loss)))
        return grad, loss

    def train_grad_slice(self, x, y_std, start: int, count: int, grad=None):
        """train_grad on columns [start, start+count) of [134, ld] / [7, ld] tensors
        (a batch of a device-resident dataset, no copy)."""
        sizes = self._sizes()
        _check(x, torch.float32, sizes[0], "x")
        _check(y_std, torch.float32, sizes[-1], "y_std")
        ld = x.shape[1]
        if y_std.shape[1] != ld or start < 0 or start + count > ld:
            raise DsoError(ErrorKind.InvalidArgument, "slice outside the dataset")
        if grad is None:
            grad = self._empty((self.n_model_params,), torch.float32)
        loss = self._empty((1,), torch.float64)
        self._raise(self._lib.dso_train_grad(self._h, _ptr(x) + 4 * start, _ptr(y_std) + 4 * start,
                                             count, ld, _ptr(grad), _ptr(loss)))
        return grad, loss

    def train_apply(self, grad, lr: float, scale: float) -> None:
        """W -= lr * scale * grad on the device model (mlp.cpp:105-108)."""
        self._raise(self._lib.dso_train_apply(self._h, _ptr(grad), lr, scale))

    def train_step(self, x, y_std, lr: float, global_batch: int, n: int | None = None,
                   comm=None, want_loss: bool = True, start: int = 0):
        """dso_train_step: one data-parallel SGD step inside the library (gradient of
        columns [start, start + n) -> NCCL allreduce over `comm` (NcclComm or None) ->
        update).  Returns the global batch's mse_loss on the pre-update weights
        (float) or None."""
        _check(x, torch.float32, None, "x")
        _check(y_std, torch.float32, None, "y_std")
        ld = x.shape[1]
        n = ld - start if n is None else n
        if y_std.shape[1] != ld or start < 0 or n < 0 or start + n > ld:
            raise DsoError(ErrorKind.InvalidArgument, "slice outside the dataset")
        loss = C.c_double()
        self._raise(self._lib.dso_train_step(self._h, _ptr(x) + 4 * start,
                                             _ptr(y_std) + 4 * start, n, ld, float(lr),
                                             int(global_batch), None if comm is None else comm.handle,
                                             C.byref(loss) if want_loss else None))
        return loss.value if want_loss else None

    def fit_model(self, x, y_std, lr: float, batch: int, epochs: int, seed: int, comm=None,
                  rank: int = 0, nranks: int = 1):
        """dso_fit_model: fit_model's epoch loop (mlp.cpp:84-130) on the device model
        (set beforehand); x [in, n], y_std [out, n] CUDA float32.  Returns the
        epoch-loss trace (list, NaN-terminated on divergence)."""
        _check(x, torch.float32, None, "x")
        _check(y_std, torch.float32, None, "y_std")
        n = x.shape[1]
        trace = (C.c_double * max(epochs, 1))()
        ran = C.c_int32()
        self._raise(self._lib.dso_fit_model(self._h, _ptr(x), _ptr(y_std), n, n, float(lr),
                                            int(batch), int(epochs), C.c_uint64(seed),
                                            None if comm is None else comm.handle, rank, nranks,
                                            trace, C.byref(ran)))
        return [float(trace[i]) for i in range(ran.value)]


class NcclComm:
    """An NCCL communicator created by the library (dso_nccl_comm_init) for the
    ranks of a torch.distributed group: rank 0's unique id is broadcast over the
    group (any backend), then every rank joins on its device."""

    def __init__(self, device: int, group=None):
        import torch.distributed as dist
        L = lib()
        self._lib = L
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            st = L.dso_nccl_unique_id(uid)
            if st:
                raise DsoError(status_kind(st), "dso_nccl_unique_id failed (is libnccl.so.2 loadable?)")
        obj = [bytes(uid)]
        dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group else 0,
                                   group=group)
        uid = (C.c_uint8 * 128).from_buffer_copy(obj[0])
        h = C.c_void_p()
        st = L.dso_nccl_comm_init(world, uid, rank, device, C.byref(h))
        if st:
            raise DsoError(status_kind(st), "dso_nccl_comm_init failed")
        self.handle, self.rank, self.world = h, rank, world

    def close(self):
        if getattr(self, "handle", None):
            self._lib.dso_nccl_comm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
