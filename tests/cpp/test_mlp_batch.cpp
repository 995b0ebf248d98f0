// C++ parity test of include/dso/batch_mlp.hpp — the predictor / feature /
// training drop-ins — compiled against the reference's unmodified public headers
// (mlp.hpp, ptx_features.hpp, telemetry.hpp, rng.hpp; Eigen's types from the
// test-only tests/cpp/eigen_min) and checked against the C restatement
// (oracle/liboracle.so, pinned to the reference's golden vectors and KATs by
// tests/test_oracle.py).  Built by tests/cpp/Makefile in the build container;
// the binary travels to the GPU box and tests/test_gpu_cpp.py runs it.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "../../oracle/dso_oracle.h"
#include "dso/batch_mlp.hpp"

using namespace dso;

static int failures = 0;
#define CHECK(cond)                                                       \
    do {                                                                  \
        if (!(cond)) {                                                    \
            std::printf("[FAIL] %s:%d  %s\n", __FILE__, __LINE__, #cond); \
            ++failures;                                                   \
        }                                                                 \
    } while (0)

static double f32(double v) { return (double)(float)v; }

// An MlpModel from the library's init_mlp, f32-rounded (what the device holds).
static MlpModel make_model(const std::vector<int>& sizes, std::uint64_t seed, bool round = true) {
    MlpModel m = detail::init_model(sizes, seed);
    for (auto& w : m.weights)
        for (Eigen::Index r = 0; r < w.rows(); ++r)
            for (Eigen::Index c = 0; c < w.cols(); ++c) w(r, c) = round ? f32(w(r, c)) : w(r, c);
    for (int i = 0; i < sizes.back(); ++i) {
        m.target_mean[i] = 0.5 + 0.25 * i;
        m.target_std[i] = 1.0 + 0.5 * i;
    }
    return m;
}

struct Flat {
    std::vector<int> sizes;
    std::vector<double> W, b, mean, std_;
};
static Flat flat(const MlpModel& m) {
    Flat f;
    auto fm = detail::flatten(m);
    f.sizes.assign(fm.sizes.begin(), fm.sizes.end());
    f.W = fm.W;
    f.b = fm.b;
    f.mean = fm.mean;
    f.std_ = fm.std_;
    return f;
}

static double rnd(std::uint64_t& s) { return (double)((s = s * 6364136223846793005ULL + 1442695040888963407ULL) >> 11) * 0x1.0p-53; }

int main() {
    GpuContext ctx(0);
    std::uint64_t s = 12345;

    // ---- forward_raw_batch vs the restated forward_raw (default and probe chains)
    for (const auto& sizes : std::vector<std::vector<int>>{{134, 100, 50, 25, 7}, {4, 3, 3, 3, 2}, {134, 64, 7}}) {
        MlpModel m = make_model(sizes, 424242);
        const int n = 777, in = sizes.front(), out = sizes.back();
        Eigen::MatrixXd x(in, n);
        std::vector<double> xr((size_t)n * in);
        for (int k = 0; k < n; ++k)
            for (int i = 0; i < in; ++i) xr[(size_t)k * in + i] = x(i, k) = f32(rnd(s));
        Eigen::MatrixXd y = forward_raw_batch(m, x, ctx);
        Flat f = flat(m);
        std::vector<double> want((size_t)n * out);
        orc_forward_raw(f.sizes.data(), (int)f.sizes.size(), f.W.data(), f.b.data(), f.mean.data(),
                        f.std_.data(), xr.data(), n, want.data());
        double worst = 0.0;
        for (int k = 0; k < n; ++k)
            for (int o = 0; o < out; ++o) {
                const double w = want[(size_t)k * out + o];
                worst = std::max(worst, std::abs(y(o, k) - w) / (std::abs(w) * 1e-5 + 1e-6 * f.std_[o]));
            }
        CHECK(worst <= 1.0);
        std::printf("forward_raw_batch %zu layers: worst %.3f of tolerance\n", sizes.size(), worst);
    }

    // ---- featurize_batch / as_vector_batch vs the restated featurize (exact f32)
    {
        const int n = 501;
        std::vector<KernelInstructionCounts> kc(n);
        std::vector<DcgmMetricVector> dc(n);
        std::vector<uint32_t> counts((size_t)n * 126, 0);
        for (int k = 0; k < n; ++k) {
            for (int r = 0; r < 126; ++r) {
                if (rnd(s) < 0.8) continue;
                const uint32_t v = 1 + (uint32_t)(rnd(s) * 5e6);
                counts[(size_t)k * 126 + r] = v;
                const std::string name = dso_category_name(r);
                if (r < 101) kc[k].instr_counts[name] = v;
                else if (r < 118) kc[k].dtype_counts[name] = v;
                else kc[k].memspace_counts[name] = v;
            }
            dc[k] = DcgmMetricVector{rnd(s), rnd(s), rnd(s), rnd(s), rnd(s), rnd(s), rnd(s), rnd(s)};
        }
        std::vector<double> want((size_t)n * 126);
        orc_featurize(counts.data(), n, want.data());
        auto fv = featurize_batch(kc, ctx);
        Eigen::MatrixXd fused = as_vector_batch(kc, dc, ctx);
        int bad = 0;
        for (int k = 0; k < n; ++k) {
            for (int r = 0; r < 126; ++r) {
                const double w = f32(want[(size_t)k * 126 + r]);
                const double g = r < 101 ? fv[k].instr[r] : (r < 118 ? fv[k].dtype[r - 101] : fv[k].memspace[r - 118]);
                bad += g != w;
                bad += fused(8 + r, k) != w;
            }
            bad += fused(0, k) != f32(dc[k].smact) || fused(7, k) != f32(dc[k].intac);
        }
        CHECK(bad == 0);
        // 64-bit counts beyond 2^32: the reference's double quotient, rounded once
        KernelInstructionCounts big;
        big.instr_counts["add"] = 3ULL << 40;
        big.instr_counts["fma"] = (1ULL << 41) + 7;
        big.dtype_counts[".f32"] = 5;
        std::vector<KernelInstructionCounts> one{big};
        auto fb = featurize_batch(one, ctx);
        const double tot = (double)((3ULL << 40) + (1ULL << 41) + 7);
        CHECK(fb[0].instr[0] == f32((double)(3ULL << 40) / tot));
        CHECK(fb[0].instr[37] == f32((double)((1ULL << 41) + 7) / tot));
        CHECK(fb[0].dtype[10] == 1.0);
        // a name outside the canonical lists has no device row
        KernelInstructionCounts odd;
        odd.instr_counts["not_an_opcode"] = 1;
        std::vector<KernelInstructionCounts> v1{odd};
        bool threw = false;
        try {
            featurize_batch(v1, ctx);
        } catch (const Error& e) {
            threw = e.kind() == ErrorKind::InvalidArgument;
        }
        CHECK(threw);

        // ---- predict_params_batch: from FusedFeatures and from counts + DCGM
        MlpModel m = make_model({134, 100, 50, 25, 7}, 424242);
        for (int i = 0; i < 7; ++i) m.target_mean[i] = 10.0 * (i + 1);
        std::vector<FusedFeatures> ff(n);
        std::vector<double> xr((size_t)n * 134);
        for (int k = 0; k < n; ++k) {
            ff[k].dcgm = dc[k];
            ff[k].ptx = fv[k];
            for (int r = 0; r < 134; ++r) xr[(size_t)k * 134 + r] = fused(r, k);
        }
        auto p1 = predict_params_batch(m, ff, ctx);
        auto p2 = predict_params_batch(m, kc, dc, ctx);
        Flat f = flat(m);
        std::vector<double> wp((size_t)n * 7);
        std::vector<uint8_t> wc(n);
        orc_predict_params(f.sizes.data(), 5, f.W.data(), f.b.data(), f.mean.data(), f.std_.data(),
                           xr.data(), n, wp.data(), wc.data(), 4);
        double worst = 0.0;
        int same = 0;
        for (int k = 0; k < n; ++k) {
            const double g[7] = {p1[k].params.p0, p1[k].params.kappa_pow, p1[k].params.gamma, p1[k].params.c,
                                 p1[k].params.t0, p1[k].params.alpha, p1[k].params.beta};
            for (int j = 0; j < 7; ++j) {
                const double w = wp[(size_t)k * 7 + j];
                worst = std::max(worst, std::abs(g[j] - w) / (std::abs(w) * 1e-5 + 1e-6 * f.std_[j]));
            }
            same += p1[k].params.p0 == p2[k].params.p0 && p1[k].params.beta == p2[k].params.beta &&
                    p1[k].clamped == p2[k].clamped;
        }
        CHECK(worst <= 1.0);
        CHECK(same == n);
        std::printf("predict_params_batch: worst %.3f of tolerance, counts path == fused path\n", worst);
    }

    // ---- load_dcgm_samples_batch: means and the reference's error kinds
    {
        std::vector<std::string> txt;
        for (int t = 0; t < 40; ++t) {
            std::string c = "timestamp,SMACT,SMOCC,TENSO,DRAMA,FP64A,FP32A,FP16A,INTAC\n";
            for (int r = 0; r < 3 + t; ++r) {
                c += std::to_string(r);
                for (int m = 0; m < 8; ++m) c += "," + std::to_string(0.01 * ((r * 7 + m * 3 + t) % 100));
                c += "\n";
            }
            txt.push_back(c);
        }
        std::vector<std::string_view> views(txt.begin(), txt.end());
        auto d = load_dcgm_samples_batch(views);
        double sum = 0.0;
        for (int r = 0; r < 3; ++r) sum += 0.01 * ((r * 7 + 0 + 0) % 100);
        CHECK(std::abs(d[0].smact - sum / 3.0) < 1e-15);
        auto kind_of = [&](const std::string& bad) {
            std::vector<std::string> t2 = txt;
            t2[5] = bad;
            std::vector<std::string_view> v2(t2.begin(), t2.end());
            try {
                load_dcgm_samples_batch(v2);
            } catch (const Error& e) {
                return e.kind();
            }
            return ErrorKind::IoError;
        };
        CHECK(kind_of("bad header\n") == ErrorKind::SchemaMismatch);
        CHECK(kind_of("timestamp,SMACT,SMOCC,TENSO,DRAMA,FP64A,FP32A,FP16A,INTAC\n") == ErrorKind::EmptyTrace);
        CHECK(kind_of("timestamp,SMACT,SMOCC,TENSO,DRAMA,FP64A,FP32A,FP16A,INTAC\n0,1.5,0,0,0,0,0,0,0\n") ==
              ErrorKind::OutOfRange);
    }

    // ---- analytic_gradients_batch / mse_loss_batch vs the restated backprop
    for (const auto& sizes : std::vector<std::vector<int>>{{134, 100, 50, 25, 7}, {4, 3, 3, 3, 2}}) {
        MlpModel m = make_model(sizes, 99);
        const int B = 300, in = sizes.front(), out = sizes.back();
        Eigen::MatrixXd x(in, B), y(out, B);
        std::vector<double> xr((size_t)B * in), yr((size_t)B * out);
        for (int k = 0; k < B; ++k) {
            for (int i = 0; i < in; ++i) xr[(size_t)k * in + i] = x(i, k) = f32(rnd(s));
            for (int o = 0; o < out; ++o) yr[(size_t)k * out + o] = y(o, k) = f32(rnd(s) - 0.5);
        }
        double mse = 0.0;
        Gradients g = analytic_gradients_batch(m, x, y, ctx, &mse);
        Flat f = flat(m);
        std::vector<double> gW(f.W.size()), gb(f.b.size());
        orc_analytic_gradients(f.sizes.data(), (int)f.sizes.size(), f.W.data(), f.b.data(), xr.data(),
                               yr.data(), B, gW.data(), gb.data());
        double mw = 0.0, err = 0.0;
        size_t o = 0;
        for (auto& w : g.weights)
            for (Eigen::Index r = 0; r < w.rows(); ++r)
                for (Eigen::Index c = 0; c < w.cols(); ++c, ++o) {
                    mw = std::max(mw, std::abs(gW[o]));
                    err = std::max(err, std::abs(w(r, c) - gW[o]));
                }
        CHECK(err <= 2e-5 * mw + 1e-12);
        const double wl = orc_mse_loss(f.sizes.data(), (int)f.sizes.size(), f.W.data(), f.b.data(),
                                       xr.data(), yr.data(), B);
        CHECK(std::abs(mse - wl) <= 1e-5 * wl);
        CHECK(std::abs(mse_loss_batch(m, x, y, ctx) - wl) <= 1e-5 * wl);
        std::printf("analytic_gradients_batch %zu layers: max err %.2e of max |g| %.2e\n", sizes.size(), err, mw);
    }

    // ---- fit_model_gpu vs the restated sgd_epoch; train_gpu; DP with a 1-rank communicator
    {
        const int n = 90;
        std::vector<TrainingExample> data(n);
        std::vector<double> feats((size_t)n * 134), targ((size_t)n * 7);
        for (int k = 0; k < n; ++k) {
            data[k].features = Eigen::VectorXd(134);
            data[k].targets = Eigen::VectorXd(7);
            for (int i = 0; i < 134; ++i) feats[(size_t)k * 134 + i] = data[k].features[i] = f32(rnd(s) * (i < 40));
            for (int j = 0; j < 7; ++j) targ[(size_t)k * 7 + j] = data[k].targets[j] = 1.0 + j + rnd(s);
        }
        const auto canon = detail::canonical(data);
        const auto st = detail::target_stats(canon);
        std::vector<double> trace;
        const std::vector<int> sizes{134, 100, 50, 25, 7};
        MlpModel m = fit_model_gpu(canon, sizes, st.mean, st.std_, 0.05, 16, 5, 7, &trace, ctx);
        // oracle: init_mlp(7) rounded to f32, then 5 sgd_epochs from Rng(7).fork(0x5d0)
        MlpModel o = make_model(sizes, 7);
        Flat f = flat(o);
        std::vector<double> cf((size_t)n * 134), ct((size_t)n * 7);
        for (int k = 0; k < n; ++k) {
            for (int i = 0; i < 134; ++i) cf[(size_t)k * 134 + i] = canon[k].features[i];
            for (int j = 0; j < 7; ++j) ct[(size_t)k * 7 + j] = canon[k].targets[j];
        }
        std::vector<double> sm(7), ss(7);
        for (int j = 0; j < 7; ++j) {
            sm[j] = st.mean[j];
            ss[j] = st.std_[j];
        }
        std::uint64_t rs = 7;
        rs = orc_rng_fork(&rs, 0x5d0);
        bool ok = trace.size() == 5;
        for (int e = 0; e < 5 && ok; ++e) {
            const double l = orc_sgd_epoch(f.sizes.data(), 5, f.W.data(), f.b.data(), cf.data(), ct.data(), n,
                                           sm.data(), ss.data(), 0.05, 16, &rs);
            ok = ok && std::abs(trace[e] - l) <= 2e-4 * std::abs(l);
        }
        CHECK(ok);
        double mw = 0.0, err = 0.0;
        size_t q = 0;
        for (auto& w : m.weights)
            for (Eigen::Index r = 0; r < w.rows(); ++r)
                for (Eigen::Index c = 0; c < w.cols(); ++c, ++q) {
                    mw = std::max(mw, std::abs(f.W[q]));
                    err = std::max(err, std::abs(w(r, c) - f.W[q]));
                }
        CHECK(err <= 2e-4 * mw);
        std::printf("fit_model_gpu: 5 epochs, weights within %.2e of max |W| %.2e\n", err, mw);

        TrainConfig cfg;
        cfg.epochs = 3;
        cfg.seed = 11;
        cfg.grid = {{0.1, 8}, {0.03, 16}};
        TrainResult a = train_gpu(data, cfg, ctx);
        CHECK(a.cv.table.size() == 2 && a.cv.table[0].fold_mape_pct.size() == 3);
        CHECK(a.epoch_loss.size() == 3);
        const auto& b0 = a.cv.table[0];
        const auto& b1 = a.cv.table[1];
        const auto& win = b0.mean_mape_pct <= b1.mean_mape_pct ? b0 : b1;
        CHECK(a.cv.best.learning_rate == win.cell.learning_rate);
        // order invariance (canonicalize) and determinism
        std::vector<TrainingExample> rev(data.rbegin(), data.rend());
        TrainResult b = train_gpu(rev, cfg, ctx);
        CHECK(b.epoch_loss == a.epoch_loss);
        CHECK(b.cv.table[1].fold_mape_pct == a.cv.table[1].fold_mape_pct);
        // empty grid -> {learning_rate, batch_size}; a topology override
        TrainConfig c2 = cfg;
        c2.grid.clear();
        c2.learning_rate = 0.05;
        c2.batch_size = 8;
        c2.layer_sizes = {0, 16, 0};
        TrainResult c = train_gpu(data, c2, ctx);
        CHECK(c.cv.table.size() == 1 && c.cv.best.batch_size == 8);
        CHECK(c.model.layer_sizes == std::vector<int>({134, 16, 7}));
        // data-parallel: one-rank NCCL communicator == no communicator, bit for bit
        {
            auto id = NcclCommunicator::unique_id();
            NcclCommunicator comm(1, id, 0, 0);
            TrainResult d = train_gpu(data, cfg, ctx, DataParallel{comm.handle(), 0, 1});
            CHECK(d.epoch_loss == a.epoch_loss);
            CHECK(d.cv.table[0].fold_mape_pct == a.cv.table[0].fold_mape_pct);
        }
        bool threw = false;
        try {
            std::vector<TrainingExample> two(data.begin(), data.begin() + 2);
            train_gpu(two, cfg, ctx);
        } catch (const Error& e) {
            threw = e.kind() == ErrorKind::DatasetTooSmall;
        }
        CHECK(threw);
        std::printf("train_gpu: best lr %.2f batch %d, mean MAPE %.3f / %.3f\n", a.cv.best.learning_rate,
                    a.cv.best.batch_size, b0.mean_mape_pct, b1.mean_mape_pct);
    }

    if (failures) {
        std::printf("%d FAILURES\n", failures);
        return 1;
    }
    std::printf("PASS\n");
    return 0;
}
