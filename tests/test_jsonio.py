"""Reference JSON formats (json_io.cpp): model round trip bit-exact (acceptance
criterion 8), JSONL datasets, error kinds; the golden MLP fixture parses."""

import json
import os

import numpy as np
import pytest

from paper_2407_13096_b200 import DsoError, ErrorKind, init_mlp
from paper_2407_13096_b200.jsonio import (dataset_from_jsonl, dataset_to_jsonl, model_from_json,
                                          model_to_json)


def test_model_round_trip_bit_exact():
    m = init_mlp(seed=424242)
    m.target_mean = np.random.default_rng(1).normal(size=7)
    m.target_std = np.random.default_rng(2).uniform(0.1, 3, 7)
    m.seed = 424242
    m2 = model_from_json(model_to_json(m))
    for a, b in zip(m.weights + m.biases, m2.weights + m2.biases):
        np.testing.assert_array_equal(np.asarray(a).view(np.uint64), np.asarray(b).view(np.uint64))
    assert m2.layer_sizes == m.layer_sizes and m2.seed == m.seed
    assert json.loads(model_to_json(m))["format_version"] == 1
    assert model_to_json(m2) == model_to_json(m)


def test_model_errors():
    m = init_mlp(seed=1)
    m.weights[0][0, 0] = np.nan
    with pytest.raises(DsoError) as e:
        model_to_json(m)
    assert e.value.kind == ErrorKind.InvalidModel
    with pytest.raises(DsoError) as e:
        model_from_json('{"layer_sizes": [2, 1]}')
    assert e.value.kind == ErrorKind.SchemaMismatch
    good = json.loads(model_to_json(init_mlp(seed=1)))
    good["weights"][0] = good["weights"][0][:-1]
    with pytest.raises(DsoError) as e:
        model_from_json(json.dumps(good))
    assert e.value.kind == ErrorKind.InvalidModel


def test_dataset_jsonl():
    rng = np.random.default_rng(3)
    f, t = rng.uniform(size=(5, 134)), rng.normal(size=(5, 7))
    f2, t2 = dataset_from_jsonl(dataset_to_jsonl(f, t).replace("\n", "\r\n"))
    np.testing.assert_array_equal(f, f2)
    np.testing.assert_array_equal(t, t2)
    with pytest.raises(DsoError) as e:
        dataset_from_jsonl('{"features": [1]}\n')
    assert e.value.kind == ErrorKind.SchemaMismatch
