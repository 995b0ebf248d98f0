// ref_shim.cpp — extern "C" shim over the UNMODIFIED reference sources.
//
// TEST INFRASTRUCTURE ONLY.  oracle/Makefile compiles this file together with
// /root/reference/proj/src/optimizer.cpp (in place, read-only) against the
// reference headers proj/include/dso/{dvfs_model,error,optimizer,rng}.hpp and
// writes oracle/_ref/libdso_ref.so.  No reference source is copied into this
// repo.  The shim only marshals plain arrays into the reference's own types and
// calls the reference functions; every number it returns is computed by
// reference code.
//
// Used by tests/ to pin the C restatement (oracle/dso_oracle.c) and the CUDA
// path, and by bench.py --impl reference as the CPU baseline for the sweep.
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "dso/dvfs_model.hpp"
#include "dso/error.hpp"
#include "dso/optimizer.hpp"
#include "dso/rng.hpp"

namespace {

int status_of(const dso::Error& e) { return static_cast<int>(e.kind()) + 1; }

thread_local std::string g_msg;

dso::KernelModelParams to_params(const double* p) {
    return dso::KernelModelParams{p[0], p[1], p[2], p[3], p[4], p[5], p[6]};
}

dso::DvfsDomain to_domain(const double* core, int nc, const double* mem, int nm,
                          const double* dev) {
    dso::DvfsDomain d;
    d.core_freqs_mhz.assign(core, core + nc);
    d.mem_freqs_mhz.assign(mem, mem + nm);
    d.dev = dso::DeviceConstants{dev[0], dev[1], dev[2], dev[3], dev[4]};
    return d;
}

template <class F>
void parallel(int64_t n, int threads, F&& f) {
    if (threads <= 1 || n < 2) {
        f(int64_t{0}, n);
        return;
    }
    threads = static_cast<int>(std::min<int64_t>(threads, n));
    std::vector<std::thread> pool;
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] { f(n * t / threads, n * (t + 1) / threads); });
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

const char* ref_last_message() { return g_msg.c_str(); }

int ref_validate_domain(const double* core, int nc, const double* mem, int nm,
                        const double* dev) {
    try {
        dso::validate(to_domain(core, nc, mem, nm, dev));
        return 0;
    } catch (const dso::Error& e) {
        g_msg = e.message();
        return status_of(e);
    }
}

// brute_force_config / optimal_config over n kernels (AoS params [n][7]).
// best: [n][3] (vc, fc, fm); status per kernel (0 ok, else ErrorKind+1).
static int run_opt(bool structured, const double* params, int64_t n, const double* core,
                   int nc, const double* mem, int nm, const double* dev, double eta,
                   double pmax, double* best, double* cost, double* energy, double* time,
                   int64_t* candidates, uint8_t* fallback, double* presnap, int32_t* kstatus,
                   int threads) {
    dso::DvfsDomain dom = to_domain(core, nc, mem, nm, dev);
    parallel(n, threads, [&](int64_t lo, int64_t hi) {
        for (int64_t k = lo; k < hi; ++k) {
            try {
                dso::OptimizationResult r =
                    structured ? dso::optimal_config(to_params(params + 7 * k), dom, eta, pmax)
                               : dso::brute_force_config(to_params(params + 7 * k), dom, eta,
                                                         pmax);
                if (best) {
                    best[3 * k] = r.best.vc;
                    best[3 * k + 1] = r.best.fc_mhz;
                    best[3 * k + 2] = r.best.fm_mhz;
                }
                if (cost) cost[k] = r.cost;
                if (energy) energy[k] = r.energy_j;
                if (time) time[k] = r.time_s;
                if (candidates) candidates[k] = r.candidates_evaluated;
                if (fallback) fallback[k] = r.fallback ? 1 : 0;
                if (presnap) {
                    presnap[3 * k] = r.presnap_vc;
                    presnap[3 * k + 1] = r.presnap_fc_mhz;
                    presnap[3 * k + 2] = r.presnap_fm_mhz;
                }
                if (kstatus) kstatus[k] = 0;
            } catch (const dso::Error& e) {
                if (kstatus) kstatus[k] = status_of(e);
            }
        }
    });
    return 0;
}

int ref_brute_force_config(const double* params, int64_t n, const double* core, int nc,
                           const double* mem, int nm, const double* dev, double eta,
                           double pmax, double* best, double* cost, double* energy,
                           double* time, int64_t* candidates, int32_t* kstatus, int threads) {
    return run_opt(false, params, n, core, nc, mem, nm, dev, eta, pmax, best, cost, energy,
                   time, candidates, nullptr, nullptr, kstatus, threads);
}

int ref_optimal_config(const double* params, int64_t n, const double* core, int nc,
                       const double* mem, int nm, const double* dev, double eta, double pmax,
                       double* best, double* cost, double* energy, double* time,
                       int64_t* candidates, uint8_t* fallback, double* presnap,
                       int32_t* kstatus, int threads) {
    return run_opt(true, params, n, core, nc, mem, nm, dev, eta, pmax, best, cost, energy,
                   time, candidates, fallback, presnap, kstatus, threads);
}

// dvfs_model.hpp inlines, evaluated by the reference header.
// which: 0 power, 1 exec_time, 2 energy, 3 cost.  Returns status.
int ref_model_eval(int which, const double* p, double vc, double fc, double fm, double eta,
                   double pmax, double* out) {
    try {
        dso::KernelModelParams kp = to_params(p);
        dso::DvfsConfig cfg{vc, fc, fm};
        switch (which) {
            case 0: *out = dso::power(kp, cfg); break;
            case 1: *out = dso::exec_time(kp, cfg); break;
            case 2: *out = dso::energy(kp, cfg); break;
            default: *out = dso::cost(kp, cfg, eta, pmax); break;
        }
        return 0;
    } catch (const dso::Error& e) {
        g_msg = e.message();
        return status_of(e);
    }
}

// which: 0 max_core_freq(v), 1 required_voltage(f), 2 required_voltage_mhz(f)
int ref_vf_eval(int which, double x, const double* dev, double* out) {
    try {
        dso::DeviceConstants d{dev[0], dev[1], dev[2], dev[3], dev[4]};
        switch (which) {
            case 0: *out = dso::max_core_freq(x, d); break;
            case 1: *out = dso::required_voltage(x, d); break;
            default: *out = dso::required_voltage_mhz(x, d); break;
        }
        return 0;
    } catch (const dso::Error& e) {
        g_msg = e.message();
        return status_of(e);
    }
}

int ref_validate_params(const double* p) {
    try {
        dso::validate(to_params(p));
        return 0;
    } catch (const dso::Error& e) {
        g_msg = e.message();
        return status_of(e);
    }
}

// Rng: n draws of next_u64 / uniform01 / below(m) from Rng(seed).
void ref_rng_u64(uint64_t seed, int64_t n, uint64_t* out) {
    dso::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}
void ref_rng_uniform01(uint64_t seed, int64_t n, double* out) {
    dso::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.uniform01();
}
void ref_rng_below(uint64_t seed, uint64_t m, int64_t n, uint64_t* out) {
    dso::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.below(m);
}
// Rng(seed).fork(salt).next_u64() for salt in [salt0, salt0+n)
void ref_fork_seeds(uint64_t seed, uint64_t salt0, int64_t n, uint64_t* out) {
    dso::Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.fork(salt0 + static_cast<uint64_t>(i)).next_u64();
}
void ref_shuffled_indices(uint64_t seed, uint64_t n, uint64_t* out) {
    dso::Rng r(seed);
    auto v = dso::shuffled_indices(n, r);
    for (uint64_t i = 0; i < n; ++i) out[i] = v[i];
}

}  // extern "C"
