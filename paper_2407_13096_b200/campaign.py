"""run_campaign on the device components (reference proj/src/sim_harness.cpp:229-346).

The reference's end-to-end experiment: a corpus of synthetic training kernels is
measured over the whole DVFS grid with multiplicative noise (measure_sweep,
sim_harness.cpp:145-170), each sweep is regressed to the 7 model parameters
(fit_power / fit_time, param_fit.cpp), the MLP is cross-validated and trained on
(features -> fitted parameters) (train, mlp.cpp:413-437), the test kernels'
parameters are predicted (predict_params), and optimal_config's choice per eta is
scored against each kernel's ground truth: prediction MAPE over the grid, and
energy saving / time loss versus the default (max fc, max fm) setting.

Here every data-parallel step runs on the GPU through the C-ABI: the synthetic
kernels' features (dso_gen_synthetic + dso_featurize), param_fit
(dso_param_fit), training (dso_train_grad / dso_train_apply via train.train),
prediction (dso_predict) and optimal_config (dso_optimal_config).  The host
keeps the seeded bookkeeping of the reference: the splitmix64 streams (rng.hpp),
the ground-truth parameter draws of gen_kernel (sim_harness.cpp:118-137), the
measurement noise and the scoring arithmetic, all in double in the reference's
operation order.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from ._lib import DsoError, ErrorKind
from .domain import DvfsDomain, default_domain

MASK = (1 << 64) - 1


class Rng:
    """splitmix64 (rng.hpp:11-56)."""

    def __init__(self, seed: int):
        self.state = seed & MASK

    def next_u64(self) -> int:
        self.state = (self.state + 0x9E3779B97F4A7C15) & MASK
        z = self.state
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & MASK
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & MASK
        return z ^ (z >> 31)

    def uniform01(self) -> float:
        return float(self.next_u64() >> 11) * 2.0 ** -53

    def uniform(self, lo: float, hi: float) -> float:
        return lo + (hi - lo) * self.uniform01()

    def fork(self, salt: int) -> "Rng":
        child = Rng(self.state ^ ((0xD1342543DE82EF95 * (salt + 1)) & MASK))
        child.next_u64()
        return child


# gen_kernel ranges (sim_harness.cpp:24-30): (lo, hi, jitter)
_ALPHA, _BETA = (40.0, 400.0, 0.10), (40.0, 400.0, 0.10)
_T0, _GAMMA = (0.04, 0.30, 0.05), (0.004, 0.020, 0.10)
_C, _P0, _KAPPA = (0.002, 0.0055, 0.10), (40.0, 90.0, 0.05), (5.0, 15.0, 0.05)


def _jittered(r, w, rng):  # sim_harness.cpp:34-38
    return (r[0] + (r[1] - r[0]) * w) * (1.0 + r[2] * rng.uniform(-1.0, 1.0))


def gen_truth(seed: int) -> np.ndarray:
    """The ground-truth KernelModelParams of gen_kernel(seed) (sim_harness.cpp:118-137),
    in double: [p0, kappa_pow, gamma, c, t0, alpha, beta]."""
    rho = Rng(seed).uniform01()
    rng = Rng(seed).fork(0x6E6B)
    alpha = _jittered(_ALPHA, 1.0 - rho, rng)
    beta = _jittered(_BETA, rho, rng)
    t0 = _jittered(_T0, rng.uniform01(), rng)
    gamma = _jittered(_GAMMA, 1.0 - rho, rng)
    c = _jittered(_C, rho, rng)
    p0 = _jittered(_P0, rng.uniform01(), rng)
    kappa = _jittered(_KAPPA, rng.uniform01(), rng)
    return np.array([p0, kappa, gamma, c, t0, alpha, beta])


def _vc(fc, dev):  # required_voltage_mhz (dvfs_model.hpp:117-128)
    d = fc / dev[4] - dev[0]
    return 2.0 * d * d + dev[0]


def _power(p, vc, fc, fm):  # dvfs_model.hpp:81-84
    return ((p[0] + p[1] * vc) + p[2] * fm) + ((p[3] * vc) * vc) * fc


def _time(p, fc, fm):  # dvfs_model.hpp:88-90 (std::max)
    a, b = p[5] / fm, p[6] / fc
    return p[4] + (b if a < b else a)


@dataclass
class CampaignReport:
    """CampaignReport (sim_harness.hpp:85-100)."""
    seed: int
    corpus_size: int
    test_size: int
    noise_level: float
    oracle_predictor: bool
    time_mape_pct: float = 0.0
    power_mape_pct: float = 0.0
    selected_cell: tuple | None = None
    rows: list = field(default_factory=list)  # dicts: eta, mean saving/loss, apps


def run_campaign(ctx, corpus_size: int = 138, test_size: int = 20,
                 domain: DvfsDomain | None = None, etas=(0.2, 0.4, 0.6, 0.8, 1.0),
                 noise_level: float = 0.01, seed: int = 0, oracle_predictor: bool = False,
                 train_epochs: int = 1000, train_grid=((0.3, 8), (0.3, 16))) -> CampaignReport:
    """run_campaign (sim_harness.cpp:229-346) with CampaignConfig's defaults
    (sim_harness.hpp:60-76)."""
    from .train import train as train_model
    domain = default_domain() if domain is None else domain
    ctx.set_domain(domain)  # validate(domain)
    if corpus_size < 3 and not oracle_predictor:
        raise DsoError(ErrorKind.DatasetTooSmall, "corpus too small to train on")
    if test_size < 1:
        raise DsoError(ErrorKind.InvalidArgument, "need at least one test kernel")
    if noise_level < 0.0:
        raise DsoError(ErrorKind.InvalidArgument, "noise_level must be nonnegative")
    root = Rng(seed)
    dev = domain.dev.as_array()
    core, mem = list(domain.core_freqs_mhz), list(domain.mem_freqs_mhz)
    test_seeds = [root.fork(0x7E57000 + i).next_u64() for i in range(test_size)]
    test_truth = np.array([gen_truth(s) for s in test_seeds])
    rep = CampaignReport(seed, corpus_size, test_size, noise_level, oracle_predictor)

    def features(salt_base, n):
        g = ctx.gen_synthetic(n, root=seed, salt_base=salt_base)
        return ctx.featurize(g["counts"], g["dcgm"]), g["params"]

    if oracle_predictor:
        predicted = test_truth
    else:
        # measure every training kernel over the grid and fit it (sim_harness.cpp:258-277)
        train_seeds = [root.fork(i).next_u64() for i in range(corpus_size)]
        truth = np.array([gen_truth(s) for s in train_seeds])
        cfg = np.array([[_vc(fc, dev), fc, fm] for fc in core for fm in mem])
        S = len(cfg)
        P = np.empty((S, corpus_size))
        T = np.empty((S, corpus_size))
        for i in range(corpus_size):
            mrng = root.fork(0x3EA50000 + i)
            for s, (vc, fc, fm) in enumerate(cfg):
                T[s, i] = _time(truth[i], fc, fm) * (1.0 + noise_level * mrng.uniform(-1.0, 1.0))
                P[s, i] = _power(truth[i], vc, fc, fm) * (1.0 + noise_level * mrng.uniform(-1.0, 1.0))
        fit = ctx.param_fit(cfg, P, T)
        for i in range(corpus_size):
            for key in ("pstatus", "tstatus"):
                if fit[key][i]:
                    kind = ErrorKind(int(fit[key][i]) - 1)
                    raise DsoError(kind, f"synthetic_{train_seeds[i]}: param_fit failed")
        fitted = np.column_stack([fit["pfit"][0], fit["pfit"][1], fit["pfit"][2], fit["pfit"][3],
                                  fit["tfit"][0], fit["tfit"][1], fit["tfit"][2]])
        x, _ = features(0, corpus_size)
        x_train = x[:, :corpus_size].cpu().numpy().T.astype(np.float64)
        tr = train_model(ctx, x_train, fitted, [tuple(c) for c in train_grid],
                         seed=root.fork(0x7A17).next_u64(), epochs=train_epochs)
        rep.selected_cell = tr["cv"]["best"]
        ctx.set_model(tr["model"])
        xt, _ = features(0x7E57000, test_size)
        params, _, _ = ctx.predict_params(xt)
        predicted = params[:, :test_size].cpu().numpy().T.astype(np.float64)
        # prediction quality across the grid against ground truth (sim_harness.cpp:290-311)
        tacc = pacc = 0.0
        terms = 0
        for i in range(test_size):
            for fc in core:
                for fm in mem:
                    vc = _vc(fc, dev)
                    tt, pt = _time(test_truth[i], fc, fm), _power(test_truth[i], vc, fc, fm)
                    tacc += abs(_time(predicted[i], fc, fm) - tt) / tt
                    pacc += abs(_power(predicted[i], vc, fc, fm) - pt) / pt
                    terms += 1
        rep.time_mape_pct = 100.0 * tacc / terms
        rep.power_mape_pct = 100.0 * pacc / terms

    # score optimal_config per eta against ground truth (sim_harness.cpp:313-344)
    fc_d, fm_d = core[-1], mem[-1]
    vc_d = _vc(fc_d, dev)
    nm = len(mem)
    for eta in etas:
        opt = ctx.optimal_config(np.ascontiguousarray(predicted), float(eta), dev[1])
        if (opt["kstatus"] != 0).any():
            k = int(np.flatnonzero(opt["kstatus"])[0])
            raise DsoError(ErrorKind(int(opt["kstatus"][k]) - 1), "invalid predicted parameters")
        apps = []
        sav = loss = 0.0
        for i in range(test_size):
            tr_ = test_truth[i]
            fi, fj = divmod(int(opt["idx"][i]), nm)
            fc, fm = core[fi], mem[fj]
            vc = _vc(fc, dev)
            e_def = _power(tr_, vc_d, fc_d, fm_d) * _time(tr_, fc_d, fm_d)
            t_def = _time(tr_, fc_d, fm_d)
            e_opt = _power(tr_, vc, fc, fm) * _time(tr_, fc, fm)
            t_opt = _time(tr_, fc, fm)
            s = 100.0 * (e_def - e_opt) / e_def
            lo = 100.0 * (t_opt - t_def) / t_def
            sav += s
            loss += lo
            apps.append({"name": f"synthetic_{test_seeds[i]}", "fc_mhz": fc, "fm_mhz": fm,
                         "energy_saving_pct": s, "time_loss_pct": lo})
        rep.rows.append({"eta": float(eta), "mean_energy_saving_pct": sav / test_size,
                         "mean_time_loss_pct": loss / test_size, "apps": apps})
    return rep
