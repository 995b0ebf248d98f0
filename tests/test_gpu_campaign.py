"""run_campaign on the device components vs the reference's acceptance criteria
(proj/tests/acceptance/acceptance_main.cpp:254-330; recorded results
proj/test_output.txt:19-20) and vs the reference's own optimal_config."""

import time

import numpy as np
import pytest

from paper_2407_13096_b200 import default_domain
from paper_2407_13096_b200.campaign import Rng, gen_truth, run_campaign

pytestmark = pytest.mark.gpu


def test_truth_matches_device_generator(ctx):
    """gen_truth (host, double) == the device generator's params (float) for the
    same seeds: both follow gen_kernel (sim_harness.cpp:118-137)."""
    root = Rng(0xACCE5506)
    seeds = [root.fork(0x7E57000 + i).next_u64() for i in range(20)]
    want = np.array([gen_truth(s) for s in seeds]).astype(np.float32)
    g = ctx.gen_synthetic(20, root=0xACCE5506, salt_base=0x7E57000)
    np.testing.assert_array_equal(g["params"].cpu().numpy().T, want)


def test_ac6_oracle_predictor(ctx, ref):
    """AC6: oracle predictor, seed 0xACCE5506: eta = 0.8 saves 24.1 % at 2.00 % loss
    (24.1042 / 2.0001, SURVEY.md Appendix B probe); monotone sweep; the chosen
    configurations equal the reference optimal_config's."""
    etas = (0.0, 0.2, 0.4, 0.6, 0.8, 1.0)
    rep = run_campaign(ctx, seed=0xACCE5506, etas=etas, oracle_predictor=True)
    row = {r["eta"]: r for r in rep.rows}
    assert row[0.8]["mean_energy_saving_pct"] == pytest.approx(24.1042, abs=5e-4)
    assert row[0.8]["mean_time_loss_pct"] == pytest.approx(2.0001, abs=5e-4)
    assert row[0.0]["mean_time_loss_pct"] <= 0.5
    for a, b in zip(rep.rows, rep.rows[1:]):
        assert b["mean_energy_saving_pct"] >= a["mean_energy_saving_pct"] - 1e-9
        assert b["mean_time_loss_pct"] >= a["mean_time_loss_pct"] - 1e-9
    import json

    from paper_2407_13096_b200.jsonio import campaign_report_to_json
    doc = json.loads(campaign_report_to_json(rep, default_domain()))
    assert doc["format_version"] == 1 and len(doc["etas"]) == len(etas)
    assert set(doc["etas"][0]["apps"][0]) == {"name", "default", "optimized", "energy_saving_pct",
                                              "time_loss_pct"}
    dom = default_domain()
    root = Rng(0xACCE5506)
    truth = np.array([gen_truth(root.fork(0x7E57000 + i).next_u64()) for i in range(20)])
    for r in rep.rows:
        want = ref.optimal_config(truth, dom.core_freqs_mhz, dom.mem_freqs_mhz,
                                  dom.dev.as_array(), r["eta"], dom.dev.pmax_w)
        got = [(a["fc_mhz"], a["fm_mhz"]) for a in r["apps"]]
        assert got == [tuple(b[1:]) for b in want["best"]]


def test_ac5_learned_pipeline(ctx):
    """AC5: 138-train / 20-test campaign with the learned predictor (param_fit ->
    train -> predict on the GPU): grid MAPEs <= 10 % (reference: 3.46 % / 1.44 %,
    34.2 s on its CPU)."""
    t0 = time.perf_counter()
    rep = run_campaign(ctx, seed=0xACCE5505, etas=(0.8,))
    secs = time.perf_counter() - t0
    print(f"AC5 on the GPU: time MAPE {rep.time_mape_pct:.2f} %, power MAPE "
          f"{rep.power_mape_pct:.2f} %, cell {rep.selected_cell}, {secs:.1f} s")
    assert rep.time_mape_pct <= 10.0 and rep.power_mape_pct <= 10.0
    assert rep.selected_cell in ((0.3, 8), (0.3, 16))
