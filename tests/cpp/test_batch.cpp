// C++ parity test of include/dso/batch.hpp against the unmodified reference
// brute_force_config (proj/src/optimizer.cpp, linked in), mirroring the
// reference's own tests/unit/test_optimizer.cpp cases.  Built by
// tests/cpp/Makefile in the build container (the reference tree is needed to
// compile); the binary travels to the GPU box and tests/test_gpu_cpp.py runs it.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "dso/batch.hpp"
#include "dso/rng.hpp"

using namespace dso;

static int failures = 0;
#define CHECK(cond)                                                           \
    do {                                                                      \
        if (!(cond)) {                                                        \
            std::printf("[FAIL] %s:%d  %s\n", __FILE__, __LINE__, #cond);     \
            ++failures;                                                       \
        }                                                                     \
    } while (0)

static DvfsDomain toy_domain() {  // test_optimizer.cpp:17-23
    DvfsDomain d;
    d.core_freqs_mhz = {1.0, 2.0, 3.0, 4.0};
    d.mem_freqs_mhz = {2.0, 6.0, 18.0, 54.0};
    d.dev = DeviceConstants{0.2, 200.0, 1.0, 30.0, 1.0};
    return d;
}

static DvfsDomain default_domain() {  // sim_harness.cpp:108-116
    DvfsDomain d;
    for (int k = 0; k < 13; ++k) d.core_freqs_mhz.push_back(705.0 + 52.0 * k);
    d.core_freqs_mhz.push_back(1380.0);
    d.mem_freqs_mhz = {438.0, 658.0, 877.0};
    d.dev = DeviceConstants{0.5, 300.0, 0.55, 2.10, 1000.0};
    return d;
}

static bool same(const OptimizationResult& a, const OptimizationResult& b) {
    return a.best.vc == b.best.vc && a.best.fc_mhz == b.best.fc_mhz &&
           a.best.fm_mhz == b.best.fm_mhz && a.cost == b.cost && a.energy_j == b.energy_j &&
           a.time_s == b.time_s && a.candidates_evaluated == b.candidates_evaluated &&
           a.fallback == b.fallback;
}

int main() {
    GpuContext ctx(0);
    const KernelModelParams kRef{10.0, 5.0, 2.0, 3.0, 1.0, 8.0, 6.0};
    // toy domain, kRef, every eta of the reference tests: bit-identical results
    {
        DvfsDomain d = toy_domain();
        for (double eta : {0.0, 0.5, 0.8, 1.0}) {
            std::vector<KernelModelParams> p{kRef};
            auto g = brute_force_config_batch(p, d, eta, d.dev.pmax_w, ctx);
            CHECK(same(g[0], brute_force_config(kRef, d, eta, d.dev.pmax_w)));
        }
    }
    // 10x10 grid counts every point (test_optimizer.cpp:67-83)
    {
        DvfsDomain d;
        for (int i = 1; i <= 10; ++i) d.core_freqs_mhz.push_back(700.0 + 60.0 * i);
        for (int i = 1; i <= 10; ++i) d.mem_freqs_mhz.push_back(300.0 + 60.0 * i);
        d.dev = DeviceConstants{0.5, 300.0, 0.55, 2.10, 1000.0};
        std::vector<KernelModelParams> p{kRef};
        auto g = brute_force_config_batch(p, d, 0.5, d.dev.pmax_w, ctx);
        CHECK(g[0].candidates_evaluated == 100);
    }
    // 100k random kernels at random etas on the default domain (test_optimizer.cpp:85-99 scaled)
    {
        DvfsDomain d = default_domain();
        Rng rng(404);
        for (double eta : {0.0, 0.2, 0.8, 1.0}) {
            std::vector<KernelModelParams> p;
            for (int i = 0; i < 100000; ++i)
                p.push_back(KernelModelParams{rng.uniform(40, 90), rng.uniform(5, 15),
                                              rng.uniform(0.004, 0.02), rng.uniform(0.002, 0.0055),
                                              rng.uniform(0.04, 0.3), rng.uniform(36, 440),
                                              rng.uniform(36, 440)});
            auto g = brute_force_config_batch(p, d, eta, d.dev.pmax_w, ctx);
            int bad = 0;
            for (std::size_t i = 0; i < p.size(); ++i)
                bad += !same(g[i], brute_force_config(p[i], d, eta, d.dev.pmax_w));
            CHECK(bad == 0);
        }
    }
    // optimal_config_batch == the reference's optimal_config, every field incl.
    // fallback / presnap (test_optimizer.cpp:101-197 scaled; knee below the
    // core table forces the flagged brute-force fallback)
    {
        auto same_opt = [](const OptimizationResult& a, const OptimizationResult& b) {
            auto eq = [](double x, double y) { return x == y || (x != x && y != y); };
            return a.best.vc == b.best.vc && a.best.fc_mhz == b.best.fc_mhz &&
                   a.best.fm_mhz == b.best.fm_mhz && eq(a.cost, b.cost) &&
                   eq(a.energy_j, b.energy_j) && eq(a.time_s, b.time_s) &&
                   a.candidates_evaluated == b.candidates_evaluated &&
                   a.fallback == b.fallback && eq(a.presnap_vc, b.presnap_vc) &&
                   eq(a.presnap_fc_mhz, b.presnap_fc_mhz) && eq(a.presnap_fm_mhz, b.presnap_fm_mhz);
        };
        for (int which = 0; which < 2; ++which) {
            DvfsDomain d = which ? default_domain() : toy_domain();
            Rng rng(505 + which);
            for (double eta : {0.0, 0.5, 0.8, 1.0}) {
                std::vector<KernelModelParams> p{kRef};
                for (int i = 0; i < 50000; ++i) {
                    const double s = which ? 1.0 : 0.05;
                    KernelModelParams q{rng.uniform(40, 90) * s, rng.uniform(5, 15) * s,
                                        rng.uniform(0.004, 0.02), rng.uniform(0.002, 0.0055),
                                        rng.uniform(0.04, 0.3), rng.uniform(1, 440),
                                        rng.uniform(1, 440)};
                    if (i % 7 == 0) q.alpha = 0.0;
                    if (i % 11 == 0) q.beta = 0.0;
                    if (i % 13 == 0) q.beta = q.alpha * 1e-3;  // knee below the table
                    if (!(q.alpha + q.beta > 0.0)) q.beta = 1.0;
                    p.push_back(q);
                }
                auto g = optimal_config_batch(p, d, eta, d.dev.pmax_w, ctx);
                int bad = 0, fb = 0;
                for (std::size_t i = 0; i < p.size(); ++i) {
                    const OptimizationResult r = optimal_config(p[i], d, eta, d.dev.pmax_w);
                    bad += !same_opt(g[i], r);
                    fb += r.fallback;
                }
                CHECK(bad == 0);
                CHECK(fb > 0);
            }
        }
    }
    // fit_power_batch / fit_time_batch: the reference's param_fit unit-test cases
    // (test_param_fit.cpp:48-157; the reference's param_fit needs Eigen, absent)
    {
        const KernelModelParams t{10.0, 5.0, 2.0, 3.0, 1.0, 8.0, 6.0};
        std::vector<DvfsConfig> pc;
        for (double vc : {0.8, 1.2})
            for (double fc : {600.0, 1100.0})
                for (double fm : {400.0, 800.0}) pc.push_back({vc, fc, fm});
        std::vector<std::vector<double>> pw(2);
        for (auto& c : pc) {
            pw[0].push_back(power(t, c));
            pw[1].push_back(3.7 * power(t, c));
        }
        auto pf = fit_power_batch(pc, pw, ctx);
        CHECK(std::abs(pf[0].p0 - 10.0) < 1e-8 && std::abs(pf[0].c - 3.0) < 1e-8);
        CHECK(!pf[0].constraint_active && pf[0].mape_pct < 1e-9);
        CHECK(std::abs(pf[1].gamma - 3.7 * pf[0].gamma) < 1e-9 * 3.7 * pf[0].gamma);
        std::vector<DvfsConfig> tc;
        for (double fc : {1.0, 2.0, 3.0, 4.0})
            for (double fm : {1.0, 2.0, 3.0, 4.0}) tc.push_back({1.0, fc, fm});
        std::vector<std::vector<double>> tt(1);
        for (auto& c : tc) tt[0].push_back(exec_time(t, c));
        auto tf = fit_time_batch(tc, tt, ctx);
        CHECK(std::abs(tf[0].t0 - 1.0) < 1e-6 && std::abs(tf[0].alpha - 8.0) < 1e-6 &&
              std::abs(tf[0].beta - 6.0) < 1e-5);
        CHECK(!tf[0].partial_identifiability);
        std::vector<DvfsConfig> one{{1.0, 600.0, 400.0}, {1.0, 800.0, 400.0}, {1.0, 1000.0, 400.0}};
        try {
            (void)fit_power_batch(one, {{1.0, 2.0, 3.0}}, ctx);
            CHECK(false);
        } catch (const Error& e) {
            CHECK(e.kind() == ErrorKind::RankDeficient);
        }
    }
    // error behaviour: the reference's kinds (test_optimizer.cpp:199-214)
    {
        DvfsDomain d = default_domain();
        std::vector<KernelModelParams> p{kRef};
        try {
            brute_force_config_batch(p, d, 1.5, 300.0, ctx);
            CHECK(false);
        } catch (const Error& e) {
            CHECK(e.kind() == ErrorKind::EtaOutOfRange);
        }
        d.core_freqs_mhz = {900.0, 900.0};
        try {
            brute_force_config_batch(p, d, 0.5, 300.0, ctx);
            CHECK(false);
        } catch (const Error& e) {
            CHECK(e.kind() == ErrorKind::InvalidArgument);
        }
        DvfsDomain ok = default_domain();
        std::vector<KernelModelParams> bad{kRef, KernelModelParams{-1, 1, 1, 1, 1, 1, 1}};
        try {
            brute_force_config_batch(bad, ok, 0.5, 300.0, ctx);
            CHECK(false);
        } catch (const Error& e) {
            CHECK(e.kind() == ErrorKind::InvalidArgument);
        }
    }
    // fused pipeline through the C++ layer: decisions are optimal for the
    // predicted parameters (cost within 1e-6 of the reference's optimum there)
    {
        DvfsDomain d = default_domain();
        ctx.set_domain(d);
        std::vector<int32_t> sizes{134, 100, 50, 25, 7};
        std::vector<double> W, b(182, 0.0);
        Rng rng(424242);
        for (std::size_t l = 0; l + 1 < sizes.size(); ++l) {
            const double lim = std::sqrt(6.0 / (sizes[l] + sizes[l + 1]));
            for (int r = 0; r < sizes[l + 1] * sizes[l]; ++r) W.push_back(rng.uniform(-lim, lim));
        }
        ctx.set_model(sizes, W, b, {60, 10, 0.012, 0.004, 0.17, 220, 220},
                      {15, 3, 0.005, 0.001, 0.08, 110, 110});
        std::vector<SparseCounts> counts(3000);
        std::vector<Dcgm8> dcgm(3000);
        for (std::size_t k = 0; k < counts.size(); ++k) {
            for (int s = 0; s < 126; s += 1 + static_cast<int>(rng.below(9)))
                counts[k].entries.push_back({s, static_cast<uint32_t>(rng.below(100000))});
            for (int m = 0; m < 8; ++m) dcgm[k][m] = rng.uniform01();
        }
        for (int engine : {0, 1}) {  // FMA-pipe and tcgen05 predictor engines
            ctx.set_option("mlp_engine", engine);
            auto dec = optimize_kernels(counts, dcgm, 0.8, 300.0, ctx);
            int worse = 0;
            for (std::size_t k = 0; k < dec.size(); ++k) {
                KernelModelParams p = dec[k].params;
                CHECK(p.p0 >= 0 && p.alpha + p.beta > 0);
                const OptimizationResult r = brute_force_config(p, d, 0.8, 300.0);
                const double fc = d.core_freqs_mhz[dec[k].fc_idx], fm = d.mem_freqs_mhz[dec[k].fm_idx];
                const double c = cost(p, DvfsConfig{required_voltage_mhz(fc, d.dev), fc, fm}, 0.8, 300.0);
                worse += c > r.cost * (1.0 + 1e-6);
            }
            CHECK(worse == 0);
        }
        ctx.set_option("mlp_engine", 2);
        try {
            ctx.set_option("mlp_engine", 3);
            CHECK(false);
        } catch (const Error& e) {
            CHECK(e.kind() == ErrorKind::InvalidArgument);
        }
    }
    std::printf("%s: %d failure(s)\n", failures ? "FAIL" : "PASS", failures);
    return failures ? 1 : 0;
}
