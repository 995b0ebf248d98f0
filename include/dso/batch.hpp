// dso/batch.hpp — drop-in batched GPU versions of the DSO hot path with the
// reference's own types and error behaviour.
//
// Include next to the reference headers (proj/include/dso/*.hpp) and link
// libdso_b200.so (include/dso_b200.h is the C-ABI underneath).  Every function
// mirrors a reference function for a whole batch:
//
//   brute_force_config_batch  <-  brute_force_config   (optimizer.hpp:48-52)
//                                 bit-exact: FP64 kernel in the reference's
//                                 operation order (dso_sweep_f64)
//   optimal_config_batch      <-  optimal_config       (optimizer.hpp:39-46)
//                                 bit-exact incl. fallback, presnap and
//                                 candidates_evaluated (dso_optimal_config)
//   fit_power_batch /         <-  fit_power / fit_time (param_fit.hpp:45-56)
//   fit_time_batch                for many kernels measured on one grid
//                                 (dso_param_fit; FP64, equal to rounding)
//   optimize_kernels          <-  featurize (ptx_features.hpp:55) +
//                                 FusedFeatures::as_vector (mlp.hpp:20-25) +
//                                 predict_params (mlp.hpp:66) +
//                                 brute_force_config, fused on the GPU
//                                 (dso_pipeline_csr; FP32, 1e-5 contract)
//   GpuContext::set_domain    <-  validate(DvfsDomain) (optimizer.cpp:58-88)
//   GpuContext::set_model     <-  validate(MlpModel)   (mlp.cpp:209-226)
//
// Failures throw dso::Error with the reference's ErrorKind (error.hpp:10-25);
// a CUDA failure is reported as ErrorKind::IoError.  Like the reference the
// functions validate before computing; per-kernel parameter validation
// (dvfs_model.hpp:50-58) throws for the first invalid kernel in index order,
// as a scalar loop over brute_force_config would.
#pragma once

#include <array>
#include <cstdint>
#include <span>
#include <string>
#include <utility>
#include <vector>

#include "dso/dvfs_model.hpp"
#include "dso/error.hpp"
#include "dso/optimizer.hpp"
#include "dso/param_fit.hpp"
#include "dso_b200.h"

namespace dso {

inline void check_status(int32_t status, const dso_ctx* ctx) {
    if (status == DSO_OK) return;
    const std::string msg = ctx ? dso_last_error(ctx) : std::string(dso_status_name(status));
    if (status == DSO_ERR_CUDA) throw Error(ErrorKind::IoError, msg);
    throw Error(static_cast<ErrorKind>(status - 1), msg);
}

// One device's state (stream, domain tables, model).  Not thread-safe: one
// host thread per context, like the reference's single-writer rule.
class GpuContext {
public:
    explicit GpuContext(int device = 0) {
        check_status(dso_ctx_create(device, &ctx_), nullptr);
    }
    ~GpuContext() { dso_ctx_destroy(ctx_); }
    GpuContext(const GpuContext&) = delete;
    GpuContext& operator=(const GpuContext&) = delete;

    dso_ctx* handle() const { return ctx_; }

    void set_domain(const DvfsDomain& d) {
        const double dev[5] = {d.dev.kappa_vf, d.dev.pmax_w, d.dev.vmin_v, d.dev.vmax_v,
                               d.dev.mhz_per_unit};
        check_status(dso_set_domain(ctx_, d.core_freqs_mhz.data(),
                                    static_cast<int32_t>(d.core_freqs_mhz.size()),
                                    d.mem_freqs_mhz.data(),
                                    static_cast<int32_t>(d.mem_freqs_mhz.size()), dev),
                     ctx_);
        nm_ = d.mem_freqs_mhz.size();
        core_ = d.core_freqs_mhz;
        mem_ = d.mem_freqs_mhz;
        dev_ = d.dev;
    }

    // MlpModel in the reference layout without Eigen: weights[l] row-major
    // (sizes[l+1] x sizes[l]) concatenated, biases concatenated (model.schema.json).
    void set_model(const std::vector<int32_t>& sizes, const std::vector<double>& weights,
                   const std::vector<double>& biases, const std::vector<double>& target_mean,
                   const std::vector<double>& target_std) {
        check_status(dso_set_model(ctx_, sizes.data(), static_cast<int32_t>(sizes.size()),
                                   weights.data(), biases.data(), target_mean.data(),
                                   target_std.data()),
                     ctx_);
    }

    // dso_set_option: "mlp_engine" (0 FMA pipe, 1 tcgen05, 2 auto = default),
    // "fast_sweep" (1 default, 0 pair-by-pair scan); InvalidArgument otherwise
    void set_option(const char* key, int64_t value) {
        check_status(dso_set_option(ctx_, key, value), ctx_);
    }

    const std::vector<double>& core() const { return core_; }
    const std::vector<double>& mem() const { return mem_; }
    const DeviceConstants& dev() const { return dev_; }
    std::size_t nm() const { return nm_; }

private:
    dso_ctx* ctx_ = nullptr;
    std::size_t nm_ = 0;
    std::vector<double> core_, mem_;
    DeviceConstants dev_{};
};

// Re-upload the context's domain when it differs from `domain`.
inline void sync_domain(GpuContext& ctx, const DvfsDomain& domain) {
    if (ctx.core() != domain.core_freqs_mhz || ctx.mem() != domain.mem_freqs_mhz ||
        ctx.dev().kappa_vf != domain.dev.kappa_vf || ctx.dev().vmin_v != domain.dev.vmin_v ||
        ctx.dev().vmax_v != domain.dev.vmax_v || ctx.dev().pmax_w != domain.dev.pmax_w ||
        ctx.dev().mhz_per_unit != domain.dev.mhz_per_unit)
        ctx.set_domain(domain);
}

// brute_force_config for every element of params, bit-identical to the
// reference (optimizer.cpp:90-117).  The context's domain must equal `domain`
// (it is re-uploaded when it differs).
inline std::vector<OptimizationResult> brute_force_config_batch(
    std::span<const KernelModelParams> params, const DvfsDomain& domain, double eta,
    double pmax_w, GpuContext& ctx) {
    sync_domain(ctx, domain);
    const int64_t n = static_cast<int64_t>(params.size());
    std::vector<int32_t> idx(n), ks(n);
    std::vector<double> cost(n), energy(n), time(n);
    static_assert(sizeof(KernelModelParams) == 7 * sizeof(double), "AoS layout");
    check_status(dso_sweep_f64(ctx.handle(), reinterpret_cast<const double*>(params.data()), n,
                               eta, pmax_w, idx.data(), cost.data(), energy.data(), time.data(),
                               ks.data(), DSO_HOST),
                 ctx.handle());
    std::vector<OptimizationResult> out(n);
    const std::size_t nm = domain.mem_freqs_mhz.size();
    const long candidates = static_cast<long>(domain.core_freqs_mhz.size() * nm);
    for (int64_t k = 0; k < n; ++k) {
        if (ks[k]) {
            // validate(params) (dvfs_model.hpp:50-58), first failure in index order
            validate(params[k]);
            throw Error(static_cast<ErrorKind>(ks[k] - 1), "invalid kernel parameters");
        }
        const std::size_t i = static_cast<std::size_t>(idx[k]) / nm;
        const std::size_t j = static_cast<std::size_t>(idx[k]) % nm;
        OptimizationResult& r = out[k];
        const double fc = domain.core_freqs_mhz[i];
        r.best = DvfsConfig{required_voltage_mhz(fc, domain.dev), fc, domain.mem_freqs_mhz[j]};
        r.cost = cost[k];
        r.energy_j = energy[k];
        r.time_s = time[k];
        r.candidates_evaluated = candidates;
        r.fallback = false;
    }
    return out;
}

// optimal_config for every element of params, bit-identical to the reference
// (optimizer.cpp:119-205): best, cost, energy_j, time_s, candidates_evaluated,
// fallback and presnap_{vc,fc_mhz,fm_mhz}.
inline std::vector<OptimizationResult> optimal_config_batch(
    std::span<const KernelModelParams> params, const DvfsDomain& domain, double eta,
    double pmax_w, GpuContext& ctx) {
    sync_domain(ctx, domain);
    const int64_t n = static_cast<int64_t>(params.size());
    std::vector<int32_t> idx(n), ks(n);
    std::vector<double> cost(n), energy(n), time(n), pre(3 * n);
    std::vector<int64_t> cand(n);
    std::vector<uint8_t> fb(n);
    check_status(dso_optimal_config(ctx.handle(), reinterpret_cast<const double*>(params.data()),
                                    n, eta, pmax_w, idx.data(), cost.data(), energy.data(),
                                    time.data(), cand.data(), fb.data(), pre.data(), ks.data(),
                                    DSO_HOST),
                 ctx.handle());
    std::vector<OptimizationResult> out(n);
    const std::size_t nm = domain.mem_freqs_mhz.size();
    for (int64_t k = 0; k < n; ++k) {
        if (ks[k]) {
            validate(params[k]);
            throw Error(static_cast<ErrorKind>(ks[k] - 1), "invalid kernel parameters");
        }
        const std::size_t i = static_cast<std::size_t>(idx[k]) / nm;
        const std::size_t j = static_cast<std::size_t>(idx[k]) % nm;
        OptimizationResult& r = out[k];
        const double fc = domain.core_freqs_mhz[i];
        r.best = DvfsConfig{required_voltage_mhz(fc, domain.dev), fc, domain.mem_freqs_mhz[j]};
        r.cost = cost[k];
        r.energy_j = energy[k];
        r.time_s = time[k];
        r.candidates_evaluated = static_cast<long>(cand[k]);
        r.fallback = fb[k] != 0;
        r.presnap_vc = pre[3 * k];
        r.presnap_fc_mhz = pre[3 * k + 1];
        r.presnap_fm_mhz = pre[3 * k + 2];
    }
    return out;
}

// fit_power / fit_time for kernels measured on one grid `cfg` (every kernel's
// sample s was taken at cfg[s], as measure_sweep produces, sim_harness.cpp:157-170):
// power[k][s] / time[k][s].  Throws like a scalar loop over the reference (the
// first failing kernel in index order); TimeFit::branch and rss_trace are not
// reproduced (branch is rebuilt from the fitted coefficients; the trace holds
// the final rss only).
inline std::vector<PowerFit> fit_power_batch(const std::vector<DvfsConfig>& cfg,
                                             const std::vector<std::vector<double>>& power,
                                             GpuContext& ctx) {
    const int S = static_cast<int>(cfg.size());
    const int64_t n = static_cast<int64_t>(power.size());
    std::vector<double> c(3 * S), P((size_t)S * n), fit(6 * (size_t)n);
    std::vector<int32_t> st(n);
    for (int s = 0; s < S; ++s) {
        c[3 * s] = cfg[s].vc;
        c[3 * s + 1] = cfg[s].fc_mhz;
        c[3 * s + 2] = cfg[s].fm_mhz;
    }
    for (int64_t k = 0; k < n; ++k) {
        if (static_cast<int>(power[k].size()) != S)
            throw Error(ErrorKind::InvalidArgument, "sample count differs from the grid");
        for (int s = 0; s < S; ++s) P[(size_t)s * n + k] = power[k][s];
    }
    check_status(dso_param_fit(ctx.handle(), c.data(), S, P.data(), nullptr, n, n, fit.data(),
                               st.data(), nullptr, nullptr, DSO_HOST),
                 ctx.handle());
    std::vector<PowerFit> out(n);
    for (int64_t k = 0; k < n; ++k) {
        if (st[k]) throw Error(static_cast<ErrorKind>(st[k] - 1), "fit_power failed");
        out[k] = PowerFit{fit[k], fit[n + k], fit[2 * n + k], fit[3 * n + k], fit[4 * n + k],
                          fit[5 * n + k] != 0.0};
    }
    return out;
}

inline std::vector<TimeFit> fit_time_batch(const std::vector<DvfsConfig>& cfg,
                                           const std::vector<std::vector<double>>& time,
                                           GpuContext& ctx) {
    const int S = static_cast<int>(cfg.size());
    const int64_t n = static_cast<int64_t>(time.size());
    std::vector<double> c(3 * S), T((size_t)S * n), fit(8 * (size_t)n);
    std::vector<int32_t> st(n);
    for (int s = 0; s < S; ++s) {
        c[3 * s] = cfg[s].vc;
        c[3 * s + 1] = cfg[s].fc_mhz;
        c[3 * s + 2] = cfg[s].fm_mhz;
    }
    for (int64_t k = 0; k < n; ++k) {
        if (static_cast<int>(time[k].size()) != S)
            throw Error(ErrorKind::InvalidArgument, "sample count differs from the grid");
        for (int s = 0; s < S; ++s) T[(size_t)s * n + k] = time[k][s];
    }
    check_status(dso_param_fit(ctx.handle(), c.data(), S, nullptr, T.data(), n, n, nullptr,
                               nullptr, fit.data(), st.data(), DSO_HOST),
                 ctx.handle());
    std::vector<TimeFit> out(n);
    for (int64_t k = 0; k < n; ++k) {
        if (st[k]) throw Error(static_cast<ErrorKind>(st[k] - 1), "fit_time failed");
        TimeFit& f = out[k];
        f.t0 = fit[k];
        f.alpha = fit[n + k];
        f.beta = fit[2 * n + k];
        f.mape_pct = fit[3 * n + k];
        f.constraint_active = fit[4 * n + k] != 0.0;
        f.partial_identifiability = fit[5 * n + k] != 0.0;
        f.iterations = static_cast<int>(fit[6 * n + k]);
        f.rss_trace = {fit[7 * n + k]};
        for (int s = 0; s < S; ++s)
            // the reference's reassignment test (param_fit.cpp:93-94,212-213): the
            // final branch is the last reassignment, alpha * (1/fm) >= beta * (1/fc)
            f.branch.push_back(f.alpha * (1.0 / cfg[s].fm_mhz) >= f.beta * (1.0 / cfg[s].fc_mhz)
                                   ? TimeBranch::Memory
                                   : TimeBranch::Core);
    }
    return out;
}

// Non-zero PTX category counts of one kernel: (count-row index, count) pairs —
// the reference's KernelInstructionCounts maps (ptx_features.hpp:31-37) keyed
// by position in the canonical category lists (instr 0..100, dtype 101..117,
// memspace 118..125).
struct SparseCounts {
    std::vector<std::pair<int, std::uint32_t>> entries;
};

// DCGM ratios in DcgmMetricVector order (telemetry.hpp:13-28).
using Dcgm8 = std::array<double, 8>;

struct KernelDecision {
    KernelModelParams params;  // predict_params output (clamped)
    bool clamped = false;
    std::size_t fc_idx = 0, fm_idx = 0;
    double cost = 0, energy_j = 0, time_s = 0;  // FP32 evaluation at the chosen pair
};

// features -> predict_params -> brute_force_config for a batch of kernels on the
// GPU (one fused kernel; host buffers are staged in overlapped chunks).
inline std::vector<KernelDecision> optimize_kernels(std::span<const SparseCounts> counts,
                                                    std::span<const Dcgm8> dcgm, double eta,
                                                    double pmax_w, GpuContext& ctx) {
    if (counts.size() != dcgm.size())
        throw Error(ErrorKind::InvalidArgument, "counts and dcgm sizes differ");
    const int64_t n = static_cast<int64_t>(counts.size());
    std::vector<uint64_t> row_ptr(n + 1, 0);
    std::vector<uint32_t> entries;
    for (int64_t k = 0; k < n; ++k) {
        for (auto [slot, c] : counts[k].entries) {
            if (slot < 0 || slot >= DSO_COUNT_ROWS || c >= (1u << 25))
                throw Error(ErrorKind::InvalidArgument, "count slot or value out of range");
            entries.push_back((c << 7) | static_cast<uint32_t>(slot));
        }
        row_ptr[k + 1] = entries.size();
    }
    std::vector<float> dc(8 * n), params(7 * n), cost(n), energy(n), time(n);
    std::vector<int32_t> idx(n);
    std::vector<uint8_t> cl(n);
    for (int64_t k = 0; k < n; ++k)
        for (int m = 0; m < 8; ++m) dc[m * n + k] = static_cast<float>(dcgm[k][m]);
    check_status(dso_pipeline_csr(ctx.handle(), row_ptr.data(), entries.data(), 0, dc.data(), n,
                                  n, eta, pmax_w, params.data(), cl.data(), idx.data(),
                                  cost.data(), energy.data(), time.data(), DSO_HOST),
                 ctx.handle());
    std::vector<KernelDecision> out(n);
    const std::size_t nm = ctx.nm();
    for (int64_t k = 0; k < n; ++k) {
        KernelDecision& d = out[k];
        d.params = KernelModelParams{params[0 * n + k], params[1 * n + k], params[2 * n + k],
                                     params[3 * n + k], params[4 * n + k], params[5 * n + k],
                                     params[6 * n + k]};
        d.clamped = cl[k] != 0;
        d.fc_idx = static_cast<std::size_t>(idx[k]) / nm;
        d.fm_idx = static_cast<std::size_t>(idx[k]) % nm;
        d.cost = cost[k];
        d.energy_j = energy[k];
        d.time_s = time[k];
    }
    return out;
}

}  // namespace dso
