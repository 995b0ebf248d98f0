"""ctypes binding of libdso_b200.so (include/dso_b200.h).

The product path is the CUDA library; this module only loads it and declares
the C-ABI prototypes.  If the library is missing the import fails loudly —
there is no CPU fallback.
"""

from __future__ import annotations

import ctypes as C
import enum
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DSO_B200_LIB") or os.path.join(_HERE, "lib", "libdso_b200.so")


class ErrorKind(enum.IntEnum):
    """dso::ErrorKind (reference proj/include/dso/error.hpp:10-25)."""

    MalformedPtx = 0
    EmptyTrace = 1
    OutOfRange = 2
    SchemaMismatch = 3
    NonPositivePower = 4
    EtaOutOfRange = 5
    VoltageBelowKappa = 6
    FrequencyBelowKappa = 7
    RankDeficient = 8
    Underdetermined = 9
    DatasetTooSmall = 10
    InvalidArgument = 11
    InvalidModel = 12
    IoError = 13


class DsoError(RuntimeError):
    """dso::Error (error.hpp:47-60): a kind plus a message; str() is
    "<Kind>: <message>" like the reference's what()."""

    def __init__(self, kind: ErrorKind, message: str):
        super().__init__(f"{kind.name}: {message}")
        self.kind = kind
        self.message = message


DSO_OK = 0
DSO_ERR_CUDA = 100
DSO_HOST = 1


def status_kind(status: int) -> ErrorKind:
    if status == DSO_ERR_CUDA:
        return ErrorKind.IoError
    return ErrorKind(status - 1)


_lib = None


def lib() -> C.CDLL:
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(
                f"{LIB_PATH} is not built; run __graft_entry__.build() or "
                "`make -C paper_2407_13096_b200/csrc` (there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        _declare(L)
        _lib = L
    return _lib


def _declare(L: C.CDLL) -> None:
    vp, i32, i64, u32, u64, d = (C.c_void_p, C.c_int32, C.c_int64, C.c_uint32, C.c_uint64,
                                 C.c_double)
    P = C.POINTER
    L.dso_ctx_create.argtypes = [i32, P(vp)]
    L.dso_ctx_destroy.argtypes = [vp]
    L.dso_ctx_set_stream.argtypes = [vp, vp]
    L.dso_sync.argtypes = [vp]
    L.dso_last_error.argtypes = [vp]
    L.dso_last_error.restype = C.c_char_p
    L.dso_status_name.argtypes = [i32]
    L.dso_status_name.restype = C.c_char_p
    L.dso_launch_count.argtypes = [vp]
    L.dso_launch_count.restype = i64
    L.dso_get_counters.argtypes = [vp, P(u64), i32, i32]
    L.dso_get_counters.restype = i32
    L.dso_set_option.argtypes = [vp, C.c_char_p, i64]
    L.dso_set_option.restype = i32
    L.dso_set_domain.argtypes = [vp, P(d), i32, P(d), i32, P(d)]
    L.dso_validate_domain.argtypes = [P(d), i32, P(d), i32, P(d), C.c_char_p, i32]
    L.dso_validate_domain.restype = i32
    L.dso_set_model.argtypes = [vp, P(i32), i32, P(d), P(d), P(d), P(d)]
    L.dso_get_model.argtypes = [vp, P(d), P(d)]
    L.dso_init_mlp.argtypes = [P(i32), i32, u64, P(d), P(d)]
    L.dso_shuffled_indices.argtypes = [u64, P(u64), P(u64)]
    L.dso_featurize.argtypes = [vp, vp, vp, i64, i64, vp]
    L.dso_featurize_u64.argtypes = [vp, vp, vp, i64, i64, vp]
    L.dso_featurize_u64.restype = i32
    L.dso_dcgm_mean.argtypes = [vp, vp, i64, i64, i64, vp, vp]
    L.dso_predict.argtypes = [vp, vp, i64, i64, vp, vp, vp]
    L.dso_sweep.argtypes = [vp, vp, i64, i64, d, d, vp, vp, vp, vp, vp]
    L.dso_sweep_f64.argtypes = [vp, vp, i64, d, d, vp, vp, vp, vp, vp, u32]
    L.dso_optimal_config.argtypes = [vp, vp, i64, d, d, vp, vp, vp, vp, vp, vp, vp, vp, u32]
    L.dso_optimal_config.restype = i32
    L.dso_param_fit.argtypes = [vp, vp, i32, vp, vp, i64, i64, vp, vp, vp, vp, u32]
    L.dso_param_fit.restype = i32
    L.dso_ptx_parse.argtypes = [C.c_char_p, i64, P(vp), C.c_char_p, i32]
    L.dso_ptx_parse.restype = i32
    L.dso_ptx_free.argtypes = [vp]
    L.dso_ptx_free.restype = None
    L.dso_ptx_kernel_count.argtypes = [vp]
    L.dso_ptx_kernel_count.restype = i64
    L.dso_ptx_kernel_name.argtypes = [vp, i64]
    L.dso_ptx_kernel_name.restype = C.c_char_p
    L.dso_ptx_kernel_counts.argtypes = [vp, i64, vp, vp]
    L.dso_ptx_kernel_counts.restype = i32
    L.dso_ptx_counts.argtypes = [vp, vp, i64]
    L.dso_ptx_counts.restype = i32
    L.dso_ptx_nnz.argtypes = [vp]
    L.dso_ptx_nnz.restype = i64
    L.dso_ptx_csr.argtypes = [vp, vp, vp]
    L.dso_ptx_csr.restype = i32
    L.dso_category_name.argtypes = [i32]
    L.dso_category_name.restype = C.c_char_p
    L.dso_load_dcgm_csv.argtypes = [C.c_char_p, i64, vp, C.c_char_p, i32]
    L.dso_load_dcgm_csv.restype = i32
    L.dso_eta_sweep.argtypes = [vp, vp, i64, i64, P(d), i32, d, vp, vp, i64]
    L.dso_pipeline.argtypes = [vp, vp, vp, i64, i64, d, d, vp, vp, vp, vp, vp, vp, u32]
    L.dso_pipeline_csr.argtypes = [vp, vp, vp, u64, vp, i64, i64, d, d, vp, vp, vp, vp, vp, vp, u32]
    L.dso_pipeline_csr.restype = i32
    L.dso_gen_synthetic_csr.argtypes = [vp, u64, u64, i64, i64, vp, vp, vp, i64]
    L.dso_gen_synthetic_csr.restype = i32
    L.dso_gen_synthetic.argtypes = [vp, u64, u64, i64, i64, i64, vp, vp, vp]
    L.dso_train_grad.argtypes = [vp, vp, vp, i64, i64, vp, vp]
    L.dso_train_apply.argtypes = [vp, vp, d, d]
    L.dso_train_step.argtypes = [vp, vp, vp, i64, i64, d, i64, vp, P(d)]
    L.dso_train_step.restype = i32
    L.dso_fit_model.argtypes = [vp, vp, vp, i64, i64, d, i32, i32, u64, vp, i32, i32, P(d), P(i32)]
    L.dso_fit_model.restype = i32
    L.dso_nccl_unique_id.argtypes = [vp]
    L.dso_nccl_unique_id.restype = i32
    L.dso_nccl_comm_init.argtypes = [i32, vp, i32, i32, P(vp)]
    L.dso_nccl_comm_init.restype = i32
    L.dso_nccl_comm_destroy.argtypes = [vp]
    L.dso_nccl_comm_destroy.restype = i32
    L.dso_nccl_version.argtypes = [P(i32)]
    L.dso_nccl_version.restype = i32
    L.dso_probe_fp32_peak.argtypes = [vp, i32, P(d)]
    L.dso_probe_fp32_peak.restype = i32
    L.dso_model_param_count.argtypes = [vp]
    L.dso_model_param_count.restype = i64
    for name in ("dso_ctx_create", "dso_ctx_destroy", "dso_ctx_set_stream", "dso_sync",
                 "dso_set_domain", "dso_set_model", "dso_get_model", "dso_init_mlp",
                 "dso_shuffled_indices", "dso_featurize", "dso_dcgm_mean", "dso_predict",
                 "dso_sweep", "dso_sweep_f64", "dso_eta_sweep", "dso_pipeline",
                 "dso_gen_synthetic", "dso_train_grad", "dso_train_apply"):
        getattr(L, name).restype = i32


# Every symbol include/dso_b200.h declares (checked by tests/test_abi.py).
EXPORTED = (
    "dso_ctx_create", "dso_ctx_destroy", "dso_ctx_set_stream", "dso_sync", "dso_last_error",
    "dso_status_name", "dso_launch_count", "dso_get_counters", "dso_set_option", "dso_set_domain", "dso_validate_domain", "dso_set_model", "dso_get_model",
    "dso_init_mlp", "dso_shuffled_indices", "dso_featurize", "dso_featurize_u64", "dso_dcgm_mean", "dso_predict",
    "dso_sweep", "dso_sweep_f64", "dso_optimal_config", "dso_param_fit", "dso_eta_sweep", "dso_pipeline",
    "dso_pipeline_csr",
    "dso_gen_synthetic", "dso_gen_synthetic_csr",
    "dso_train_grad", "dso_train_apply", "dso_train_step", "dso_fit_model",
    "dso_nccl_unique_id", "dso_nccl_comm_init", "dso_nccl_comm_destroy", "dso_nccl_version",
    "dso_model_param_count", "dso_probe_fp32_peak",
    "dso_ptx_parse", "dso_ptx_free", "dso_ptx_kernel_count", "dso_ptx_kernel_name",
    "dso_ptx_kernel_counts", "dso_ptx_counts", "dso_ptx_nnz", "dso_ptx_csr", "dso_category_name",
    "dso_load_dcgm_csv",
)
