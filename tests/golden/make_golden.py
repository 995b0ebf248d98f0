"""Regenerate tests/golden/* from the reference (run in the build container only).

Sources (all under /root/reference/proj, read-only):
  * tests/fixtures/mlp_forward_golden.json  -> mlp_forward_golden.json (values copied)
  * src/ptx_features.cpp:18-49 category lists -> categories.json (parsed)
  * the reference brute_force_config / optimal_config / Rng, compiled from
    src/optimizer.cpp + include/dso/*.hpp into oracle/_ref/libdso_ref.so
    -> sweep_golden.npz, rng_golden.json
  * test_output.txt:15-20 recorded acceptance lines -> kat.json

The GPU box has no /root/reference; tests there read these files (and the
prebuilt oracle/_ref/*.so, which travels with the repo snapshot).

    python tests/golden/make_golden.py
"""

from __future__ import annotations

import json
import os
import re
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
REF = "/root/reference/proj"
sys.path.insert(0, ROOT)

import oracle  # noqa: E402

KREF = [10.0, 5.0, 2.0, 3.0, 1.0, 8.0, 6.0]  # test_optimizer.cpp:25 / test_dvfs_model.cpp:10


def toy_domain():
    """test_optimizer.cpp:17-23."""
    return (np.array([1.0, 2.0, 3.0, 4.0]), np.array([2.0, 6.0, 18.0, 54.0]),
            np.array([0.2, 200.0, 1.0, 30.0, 1.0]))


def default_dev():
    return np.array([0.5, 300.0, 0.55, 2.10, 1000.0])


def domains():
    dev = default_dev()
    d = {
        "toy": toy_domain(),
        "c1": (np.array([705.0 + 52.0 * k for k in range(13)] + [1380.0]),
               np.array([438.0, 658.0, 877.0]), dev),
        "c1_literal": (705.0 + 75.0 * np.arange(10), np.array([877.0]), dev),
        "c2": (705.0 + 675.0 * np.arange(64) / 63, np.array([877.0]), dev),
        "c3": (705.0 + 675.0 * np.arange(128) / 127, 438.0 + 439.0 * np.arange(4) / 3, dev),
        "grid10x10": (np.array([700.0 + 60.0 * i for i in range(1, 11)]),
                      np.array([300.0 + 60.0 * i for i in range(1, 11)]), dev),
    }
    return d


def edge_params():
    """Hand-made edge cases: invalid (negative, alpha+beta == 0), zero gamma/c
    (exact energy ties), alpha = 0 / beta = 0 (test_optimizer.cpp:176-197), NaN p0."""
    return np.array([
        KREF,
        [20.0, 5.0, 0.01, 0.002, 0.05, 200.0, 0.0],   # beta = 0
        [20.0, 5.0, 0.01, 0.002, 0.05, 0.0, 200.0],   # alpha = 0
        [50.0, 10.0, 0.0, 0.0, 0.1, 100.0, 100.0],    # gamma = c = 0
        [50.0, 0.0, 0.0, 0.0, 0.1, 100.0, 100.0],     # P constant
        [-1.0, 5.0, 0.01, 0.002, 0.05, 100.0, 100.0],  # invalid: negative
        [20.0, 5.0, 0.01, 0.002, 0.05, 0.0, 0.0],     # invalid: alpha + beta == 0
        [np.nan, 5.0, 0.01, 0.002, 0.05, 100.0, 100.0],  # NaN p0 passes validation
        [60.0, 8.0, 0.01, 0.004, 0.0, 400.0, 40.0],   # t0 = 0
    ])


def main():
    os.makedirs(HERE, exist_ok=True)
    R = oracle.ref()
    P = oracle.port()

    # -- MLP golden (copied values) ------------------------------------------------
    g = json.load(open(os.path.join(REF, "tests/fixtures/mlp_forward_golden.json")))
    json.dump({"source": "proj/tests/fixtures/mlp_forward_golden.json",
               "description": g["description"], "seed": 424242,
               "layer_sizes": [134, 100, 50, 25, 7], "outputs": g["outputs"]},
              open(os.path.join(HERE, "mlp_forward_golden.json"), "w"), indent=1)

    # -- category lists (ptx_features.cpp:18-49) ------------------------------------
    src = open(os.path.join(REF, "src/ptx_features.cpp")).read()

    def parse(name):
        m = re.search(name + r"\s*=\s*\{(.*?)\};", src, re.S)
        return re.findall(r'"([^"]*)"', m.group(1))

    cats = {"instr": parse("kInstrCategories"), "dtype": parse("kDtypeCategories"),
            "memspace": parse("kMemspaceCategories"),
            "source": "proj/src/ptx_features.cpp:18-49"}
    assert len(cats["instr"]) == 101 and len(cats["dtype"]) == 17 and len(cats["memspace"]) == 8
    json.dump(cats, open(os.path.join(HERE, "categories.json"), "w"), indent=1)

    # -- sweep golden: the reference brute_force_config --------------------------------
    out = {}
    doms = domains()
    etas = [0.0, 0.2, 0.5, 0.8, 1.0]
    for name, (core, mem, dev) in doms.items():
        if name == "toy":
            params = np.array([KREF])
        elif name == "grid10x10":
            params = edge_params()
        else:
            n = {"c1": 2000, "c1_literal": 1000, "c2": 2000, "c3": 1000}[name]
            params = P.gen_stream(0xD50B200 + len(name), n, want=("params",))["params"]
            if name == "c1":
                params = np.concatenate([params, edge_params()])
        out[f"{name}/core"], out[f"{name}/mem"], out[f"{name}/dev"] = core, mem, dev
        out[f"{name}/params"] = params
        pmaxes = [dev[1]] if name != "toy" else [200.0]
        for eta in etas:
            for pm in pmaxes:
                r = R.brute_force_config(params, core, mem, dev, eta, pm, threads=8)
                key = f"{name}/eta{eta}"
                out[key + "/idx"] = r["idx"]
                out[key + "/cost"] = r["cost"]
                out[key + "/energy"] = r["energy"]
                out[key + "/time"] = r["time"]
                out[key + "/kstatus"] = r["kstatus"]
                out[key + "/pmax"] = np.array([pm])
    # AC1 (acceptance_main.cpp:52-85): Rng(0xACCE5501) -> (seed, eta) x 200, optimal_config
    import ctypes as C
    s = C.c_uint64(0xACCE5501)
    seeds, ac1_eta = [], []
    for _ in range(200):
        seeds.append(P.lib.orc_rng_next(C.byref(s)))
        ac1_eta.append(P.lib.orc_rng_uniform01(C.byref(s)))
    k = P.gen_seeded(np.array(seeds, np.uint64))
    core, mem, dev = doms["c1"]
    idx, fb, cost = [], [], []
    for i in range(200):
        r = R.optimal_config(k["params"][i:i + 1], core, mem, dev, ac1_eta[i], 300.0, threads=1)
        b = R.brute_force_config(k["params"][i:i + 1], core, mem, dev, ac1_eta[i], 300.0,
                                 threads=1)
        idx.append(int(b["idx"][0]))
        fb.append(bool(r["fallback"][0]))
        cost.append(float(r["cost"][0]))
    out["ac1/seeds"] = np.array(seeds, np.uint64)
    out["ac1/eta"] = np.array(ac1_eta)
    out["ac1/params"] = k["params"]
    out["ac1/idx"] = np.array(idx, np.int32)
    out["ac1/fallback"] = np.array(fb)
    out["ac1/opt_cost"] = np.array(cost)
    np.savez_compressed(os.path.join(HERE, "sweep_golden.npz"), **out)

    # -- RNG golden: the reference Rng (rng.hpp) ----------------------------------------
    rng = {
        "u64_seed_42": [int(v) for v in R.rng_u64(42, 16)],
        "uniform01_seed_7": [float(v) for v in R.rng_uniform01(7, 16)],
        "below_seed_3_m_10": [int(v) for v in R.rng_below(3, 10, 32)],
        "fork_seeds_0xACCE5506_0x7e57000": [int(v) for v in
                                            R.fork_seeds(0xACCE5506, 0x7e57000, 20)],
        "shuffled_seed_99_n_20": [int(v) for v in R.shuffled_indices(99, 20)],
        "source": "proj/include/dso/rng.hpp via oracle/_ref/libdso_ref.so",
    }
    json.dump(rng, open(os.path.join(HERE, "rng_golden.json"), "w"), indent=1)

    # -- KATs recorded by the reference (test_output.txt) --------------------------------
    rec = open(os.path.join(REF, "test_output.txt")).read().splitlines()
    kat = {
        "source": "proj/test_output.txt:14-23",
        "ac1_line": next(l for l in rec if "criterion 1" in l),
        "ac2_line": next(l for l in rec if "criterion 2" in l),
        "ac4_line": next(l for l in rec if "criterion 4" in l),
        "ac6_line": next(l for l in rec if "criterion 6" in l),
        "ac6_saving_pct_1dp": 24.1,
        "ac6_loss_pct_2dp": 2.00,
        "ac2_non_fallback": 103,
        "ac4_mutation_2dp": 4.76e-02,
        "ac6_seed": 0xACCE5506,
        "ac1_seed": 0xACCE5501,
    }
    json.dump(kat, open(os.path.join(HERE, "kat.json"), "w"), indent=1)
    print("wrote", sorted(os.listdir(HERE)))


if __name__ == "__main__":
    main()
