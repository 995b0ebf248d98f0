"""JSON I/O in the reference's formats (proj/src/json_io.cpp, proj/schemas/*.json):
the model document (model.schema.json: row-major weights per layer, format_version
1), JSON-lines training datasets (dataset_line.schema.json) and the campaign report
(campaign_report.schema.json).  Floats are written with repr (shortest round-trip),
so a model trained on the GPU round-trips bit-exactly (acceptance criterion 8)."""

from __future__ import annotations

import json
import math

import numpy as np

from ._lib import DsoError, ErrorKind
from .model import MlpModel, validate_model

FORMAT_VERSION = 1  # json_io.cpp kFormatVersion


def model_to_json(model: MlpModel) -> str:
    """to_json(MlpModel) (json_io.cpp:145-171): validate, reject non-finite values."""
    validate_model(model)
    for arr in list(model.weights) + list(model.biases):
        if not np.isfinite(np.asarray(arr)).all():
            raise DsoError(ErrorKind.InvalidModel, "non-finite weights cannot be serialized")
    doc = {"format_version": FORMAT_VERSION,
           "layer_sizes": [int(s) for s in model.layer_sizes],
           "weights": [[float(v) for v in np.asarray(w, np.float64).ravel()] for w in model.weights],
           "biases": [[float(v) for v in np.asarray(b, np.float64)] for b in model.biases],
           "target_mean": [float(v) for v in model.target_mean],
           "target_std": [float(v) for v in model.target_std],
           "seed": int(model.seed)}
    return json.dumps(doc)


def model_from_json(text: str) -> MlpModel:
    """model_from_json (json_io.cpp:173-206)."""
    try:
        j = json.loads(text)
    except json.JSONDecodeError as e:
        raise DsoError(ErrorKind.SchemaMismatch, f"model: {e}") from None
    if not all(k in j for k in ("layer_sizes", "weights", "biases", "target_mean", "target_std")):
        raise DsoError(ErrorKind.SchemaMismatch, "incomplete model document")
    sizes = [int(s) for s in j["layer_sizes"]]
    if len(sizes) < 2:
        raise DsoError(ErrorKind.InvalidModel, "need at least two layers")
    if len(j["weights"]) != len(sizes) - 1 or len(j["biases"]) != len(j["weights"]):
        raise DsoError(ErrorKind.InvalidModel, "layer count mismatch")
    ws, bs = [], []
    for l in range(len(sizes) - 1):
        flat = j["weights"][l]
        if len(flat) != sizes[l + 1] * sizes[l]:
            raise DsoError(ErrorKind.InvalidModel, "weight matrix size mismatch")
        ws.append(np.array(flat, np.float64).reshape(sizes[l + 1], sizes[l]))
        bs.append(np.array(j["biases"][l], np.float64))
    m = MlpModel(sizes, ws, bs, np.array(j["target_mean"], np.float64),
                 np.array(j["target_std"], np.float64), int(j.get("seed", 0)))
    validate_model(m)
    return m


def dataset_to_jsonl(features, targets) -> str:
    """dataset_to_jsonl (json_io.cpp:254-264)."""
    f = np.asarray(features, np.float64)
    t = np.asarray(targets, np.float64)
    return "".join(json.dumps({"features": [float(v) for v in a], "targets": [float(v) for v in b]},
                              separators=(",", ":")) + "\n" for a, b in zip(f, t))


def dataset_from_jsonl(text: str):
    """dataset_from_jsonl (json_io.cpp:266-289): (features [n, d], targets [n, k])."""
    feats, targs = [], []
    for no, line in enumerate(text.split("\n"), 1):
        line = line.rstrip("\r")
        if not line:
            continue
        try:
            j = json.loads(line)
        except json.JSONDecodeError as e:
            raise DsoError(ErrorKind.SchemaMismatch, f"dataset line {no}: {e}") from None
        if "features" not in j or "targets" not in j:
            raise DsoError(ErrorKind.SchemaMismatch, f"dataset line {no} needs features and targets")
        feats.append(j["features"])
        targs.append(j["targets"])
    return np.array(feats, np.float64), np.array(targs, np.float64)


def _cfg(vc, fc, fm):
    return {"vc": vc, "fc_mhz": fc, "fm_mhz": fm}


def campaign_report_to_json(rep, domain) -> str:
    """to_json(CampaignReport) (json_io.cpp:208-234)."""
    from .campaign import _vc
    dev = domain.dev.as_array()
    fcd, fmd = domain.core_freqs_mhz[-1], domain.mem_freqs_mhz[-1]
    rows = []
    for r in rep.rows:
        apps = [{"name": a["name"], "default": _cfg(_vc(fcd, dev), fcd, fmd),
                 "optimized": _cfg(_vc(a["fc_mhz"], dev), a["fc_mhz"], a["fm_mhz"]),
                 "energy_saving_pct": a["energy_saving_pct"], "time_loss_pct": a["time_loss_pct"]}
                for a in r["apps"]]
        rows.append({"eta": r["eta"], "mean_energy_saving_pct": r["mean_energy_saving_pct"],
                     "mean_time_loss_pct": r["mean_time_loss_pct"], "apps": apps})
    cell = rep.selected_cell or (0.0, 0)
    doc = {"format_version": FORMAT_VERSION, "seed": rep.seed, "corpus_size": rep.corpus_size,
           "test_size": rep.test_size, "noise_level": rep.noise_level,
           "oracle_predictor": rep.oracle_predictor, "time_mape_pct": rep.time_mape_pct,
           "power_mape_pct": rep.power_mape_pct,
           "selected_cell": {"learning_rate": cell[0], "batch_size": cell[1]}, "etas": rows}
    if not all(math.isfinite(x) for x in (rep.time_mape_pct, rep.power_mape_pct)):
        raise DsoError(ErrorKind.InvalidArgument, "non-finite report values")
    return json.dumps(doc)
