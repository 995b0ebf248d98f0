"""paper_2407_13096_b200 — B200-native data-parallel core of DSO (arXiv 2407.13096).

Hot path (per GPU kernel of a batch): PTX instruction-mix features fused with
DCGM metrics -> MLP predictor of the 7 DVFS-model parameters -> P(f), T(f) over
the (core x memory) frequency grid -> eta-weighted objective -> optimal pair.
Hand-written sm_100a CUDA in csrc/, behind the C-ABI include/dso_b200.h; this
package is the Python host side (ctypes + torch device memory).
"""

from ._lib import DsoError, ErrorKind, LIB_PATH  # noqa: F401
from .domain import (DeviceConstants, DvfsDomain, config_domain, default_device,  # noqa: F401
                     default_domain, linear_domain, validate_domain)
from .model import (MlpModel, default_layer_sizes, init_mlp, split_flat,  # noqa: F401
                    validate_model)

__all__ = [
    "DsoError", "ErrorKind", "DeviceConstants", "DvfsDomain", "config_domain",
    "default_device", "default_domain", "linear_domain", "validate_domain", "MlpModel", "default_layer_sizes",
    "init_mlp", "Context",
]


def __getattr__(name):
    if name == "Context":
        from .api import Context
        return Context
    raise AttributeError(name)
