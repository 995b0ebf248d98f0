"""Vectorised double-precision evaluation in the reference's operation order
(proj/include/dso/dvfs_model.hpp:81-104), used by the parity checkers to judge
near-ties: numpy float64 is IEEE and never contracts a*b+c."""

import numpy as np


def vc_of(core, dev):
    d = np.asarray(core) / dev[4] - dev[0]
    return 2.0 * d * d + dev[0]


def eval_at(params, idx, core, mem, dev, eta, pmax):
    """(cost, energy, time) of pair idx for each kernel (params [n,7] float64)."""
    params = np.asarray(params, np.float64)
    idx = np.asarray(idx)
    nm = len(mem)
    i, j = idx // nm, idx % nm
    fc = np.asarray(core)[i]
    fm = np.asarray(mem)[j]
    vc = vc_of(core, dev)[i]
    p0, kp, g, c, t0, a, b = params.T
    P = ((p0 + kp * vc) + g * fm) + ((c * vc) * vc) * fc
    ta, tb = a / fm, b / fc
    T = t0 + np.where(ta < tb, tb, ta)
    C = (eta * P + (1.0 - eta) * pmax) * T
    return C, P * T, T


def check_argmin(params, gpu_idx, want_idx, core, mem, dev, eta, pmax, tie_rel=1e-6):
    """Indices must match except on near-ties: the reference's double cost at the
    GPU's pair may exceed the optimum by at most tie_rel (relative).
    Returns (n_mismatch, worst_rel_gap)."""
    gpu_idx = np.asarray(gpu_idx).astype(np.int64)
    want_idx = np.asarray(want_idx).astype(np.int64)
    bad = np.flatnonzero(gpu_idx != want_idx)
    if len(bad) == 0:
        return 0, 0.0
    cg, _, _ = eval_at(params[bad], gpu_idx[bad], core, mem, dev, eta, pmax)
    cw, _, _ = eval_at(params[bad], want_idx[bad], core, mem, dev, eta, pmax)
    gap = (cg - cw) / np.abs(cw)
    worst = float(gap.max())
    assert worst <= tie_rel, (
        f"{len(bad)} index mismatches, worst relative cost gap {worst:.3e} > {tie_rel} "
        f"(first kernel {bad[int(np.argmax(gap))]})")
    return len(bad), worst


def rel_err(got, want, floor=0.0):
    got = np.asarray(got, np.float64)
    want = np.asarray(want, np.float64)
    return np.abs(got - want) / np.maximum(np.abs(want), floor)


def f32(x):
    return np.asarray(x, np.float64).astype(np.float32)


def check_index_rule(gpu_params, ref_params, gpu_idx, ref_idx, core, mem, dev, eta, pmax,
                     tie_rel=1e-6):
    """north_star's index contract for a predicted-parameter pipeline: the chosen
    index equals the all-double oracle's except on objective near-ties.

    The GPU predicts the parameters in FP32 (within 1e-5 relative of the oracle's),
    so its objective is the oracle's shifted by the parameter error.  At every
    index mismatch the ORACLE-side cost gap C_ref(gpu) - C_ref(ref) (reference
    double cost, oracle parameters) must be explained by that shift:

        gap <= tie_rel + d(gpu) + d(ref),   d(x) = |C_ref(x) - C_gpu(x)| / C_ref(ref)

    where C_gpu is the double cost with the GPU's parameters.  With parameters
    within 1e-5 relative, d(x) <= ~2e-5 (P, T and eta*P + K are sums of
    non-negative terms), so no mismatch can hide a gap larger than ~4e-5; the
    bound is evaluated per kernel.  Returns dict(n, mismatches, worst_gap,
    worst_gap_over_bound)."""
    gpu_idx = np.asarray(gpu_idx).astype(np.int64)
    ref_idx = np.asarray(ref_idx).astype(np.int64)
    bad = np.flatnonzero(gpu_idx != ref_idx)
    out = {"n": int(len(gpu_idx)), "mismatches": int(len(bad)), "worst_gap": 0.0,
           "worst_gap_over_bound": 0.0}
    if len(bad) == 0:
        return out
    rp = np.asarray(ref_params, np.float64)[bad]
    gp = np.asarray(gpu_params, np.float64)[bad]
    c_rg, _, _ = eval_at(rp, gpu_idx[bad], core, mem, dev, eta, pmax)
    c_rr, _, _ = eval_at(rp, ref_idx[bad], core, mem, dev, eta, pmax)
    c_gg, _, _ = eval_at(gp, gpu_idx[bad], core, mem, dev, eta, pmax)
    c_gr, _, _ = eval_at(gp, ref_idx[bad], core, mem, dev, eta, pmax)
    scale = np.abs(c_rr)
    gap = (c_rg - c_rr) / scale
    bound = tie_rel + (np.abs(c_rg - c_gg) + np.abs(c_rr - c_gr)) / scale
    ratio = gap / bound
    k = int(np.argmax(ratio))
    out.update(worst_gap=float(gap.max()), worst_gap_over_bound=float(ratio.max()))
    assert (gap <= bound).all(), (
        f"{len(bad)} index mismatches; kernel {bad[k]}: oracle-side cost gap {gap[k]:.3e} "
        f"exceeds the near-tie bound {bound[k]:.3e}")
    return out
