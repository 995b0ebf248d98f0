"""The C-ABI library (CPU-side checks: no device compute is called here).

* libdso_b200.so loads and exports every entry point include/dso_b200.h declares;
* the host C++ inside the library (validation, Glorot init, Fisher-Yates) agrees
  with the reference (oracle/_ref) and the golden vectors;
* without a GPU the product fails loudly — there is no CPU fallback.
"""

import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_2407_13096_b200 import (DsoError, ErrorKind, config_domain, default_domain,
                                   init_mlp, validate_domain)
from paper_2407_13096_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "dso_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(dso_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    L = _lib.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(L, s), s
    assert sorted(_lib.EXPORTED) == syms


def test_status_names_follow_error_kinds():
    L = _lib.lib()
    for kind in ErrorKind:
        assert L.dso_status_name(kind.value + 1).decode() == kind.name
    assert L.dso_status_name(_lib.DSO_ERR_CUDA).decode() == "IoError"


def test_init_mlp_matches_oracle(port, golden_json):
    g = golden_json("mlp_forward_golden.json")
    m = init_mlp(g["layer_sizes"], g["seed"])
    ws, bs = port.init_mlp(g["layer_sizes"], g["seed"])
    for a, b in zip(m.weights, ws):
        np.testing.assert_array_equal(a, b)
    for a, b in zip(m.biases, bs):
        np.testing.assert_array_equal(a, b)
    with pytest.raises(DsoError) as e:
        init_mlp([134], 1)
    assert e.value.kind == ErrorKind.InvalidModel


def test_shuffled_indices_match_reference(golden_json):
    L = _lib.lib()
    out = np.empty(20, np.uint64)
    st = C.c_uint64(99)
    assert L.dso_shuffled_indices(20, C.byref(st), out.ctypes.data_as(C.POINTER(C.c_uint64))) == 0
    assert [int(v) for v in out] == golden_json("rng_golden.json")["shuffled_seed_99_n_20"]


def test_validate_domain_matches_reference(ref):
    """test_optimizer.cpp:199-214 plus each validate(DeviceConstants) branch."""
    import copy
    good = default_domain()
    validate_domain(good)
    for name in ("c1", "c1_literal", "c2", "c3", "c4"):
        validate_domain(config_domain(name))
    cases = []
    d = copy.deepcopy(good)
    d.core_freqs_mhz = np.array([900.0, 900.0])
    cases.append(d)
    d = copy.deepcopy(good)
    d.mem_freqs_mhz = np.array([])
    cases.append(d)
    from paper_2407_13096_b200 import DeviceConstants
    for dev in (DeviceConstants(0.5, 300, 0.55, 0.6, 1000), DeviceConstants(0.6, 300, 0.55, 2.1, 1000),
                DeviceConstants(0.5, -1, 0.55, 2.1, 1000), DeviceConstants(0.5, 300, 0.0, 2.1, 1000),
                DeviceConstants(0.5, 300, 0.55, 2.1, 0.0)):
        d = copy.deepcopy(good)
        d.dev = dev
        cases.append(d)
    d = copy.deepcopy(good)
    d.core_freqs_mhz = np.array([400.0, 900.0])
    cases.append(d)
    for d in cases:
        want = ref.validate_domain(d.core_freqs_mhz, d.mem_freqs_mhz, d.dev.as_array())
        assert want != 0
        with pytest.raises(DsoError) as e:
            validate_domain(d)
        assert e.value.kind.value + 1 == want
        assert e.value.message == ref.message()


def test_no_gpu_fails_loudly():
    import torch
    if torch.cuda.is_available():
        pytest.skip("a GPU is visible")
    from paper_2407_13096_b200.api import Context
    with pytest.raises(DsoError) as e:
        Context(0)
    assert e.value.kind == ErrorKind.IoError
