// dso/batch_mlp.hpp — drop-in batched GPU versions of the predictor / feature /
// training half of the DSO hot path, with the reference's own types
// (proj/include/dso/mlp.hpp, ptx_features.hpp, telemetry.hpp: MlpModel,
// FusedFeatures, KernelInstructionCounts, DcgmMetricVector, ParamPrediction,
// Gradients, TrainingExample, TrainConfig, CvResult, TrainResult) and dso::Error
// behaviour.  Include next to the reference headers (they need Eigen) and link
// libdso_b200.so and the CUDA runtime.  Every function mirrors a reference
// function for a whole batch:
//
//   forward_raw_batch        <-  forward_raw            (mlp.hpp:56; mlp.cpp:232-235)
//   predict_params_batch     <-  predict_params         (mlp.hpp:66; mlp.cpp:237-253)
//   featurize_batch          <-  featurize              (ptx_features.hpp:55; ptx_features.cpp:311-329)
//   as_vector_batch          <-  featurize + FusedFeatures::as_vector (mlp.cpp:158-165)
//   load_dcgm_samples_batch  <-  load_dcgm_samples      (telemetry.hpp:40; telemetry.cpp:63-101)
//   analytic_gradients_batch <-  analytic_gradients     (mlp.hpp:131-132; mlp.cpp:265-289)
//   mse_loss_batch           <-  mse_loss               (mlp.hpp:139-140; mlp.cpp:259-263)
//   fit_model_gpu            <-  fit_model              (mlp.cpp:115-130; the epochs on the device)
//   cross_validate_gpu       <-  cross_validate         (mlp.hpp:106-107; mlp.cpp:348-411)
//   train_gpu                <-  train                  (mlp.hpp:116; mlp.cpp:413-437)
//
// Data-parallel training: pass a DataParallel {nccl_comm, rank, nranks} (an
// ncclComm_t, e.g. from NcclCommunicator below) to fit_model_gpu / train_gpu on
// every rank with the same dataset and config; each rank computes its share of
// every batch and the library all-reduces the gradients over NCCL (dso_fit_model),
// so the replicas stay identical.
//
// Numerics: FP32 on the device (the 1e-5 contract); the host side only moves
// data and restates the reference's orchestration (canonical order, target
// statistics, fold split, MAPE bookkeeping, grid choice).
#pragma once

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <span>
#include <string>
#include <string_view>
#include <thread>
#include <vector>

#include "dso/batch.hpp"
#include "dso/mlp.hpp"
#include "dso/ptx_features.hpp"
#include "dso/rng.hpp"
#include "dso/telemetry.hpp"
#include "dso_b200.h"

namespace dso {

namespace detail {

inline void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw Error(ErrorKind::IoError, std::string(what) + ": " + cudaGetErrorString(e));
}

// Device buffer (RAII); one host thread per context, like GpuContext.
template <class T>
class DevBuf {
public:
    explicit DevBuf(std::size_t n) : n_(n) {
        cuda_ok(cudaMalloc(&p_, sizeof(T) * (n ? n : 1)), "cudaMalloc");
    }
    ~DevBuf() { cudaFree(p_); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    T* get() const { return p_; }
    void upload(const T* h) { cuda_ok(cudaMemcpy(p_, h, sizeof(T) * n_, cudaMemcpyHostToDevice), "H2D"); }
    void download(T* h) const {
        cuda_ok(cudaMemcpy(h, p_, sizeof(T) * n_, cudaMemcpyDeviceToHost), "D2H");
    }

private:
    T* p_ = nullptr;
    std::size_t n_;
};

// MlpModel -> the library's reference layout (row-major W_l concatenated, biases).
struct FlatModel {
    std::vector<int32_t> sizes;
    std::vector<double> W, b, mean, std_;
};

inline FlatModel flatten(const MlpModel& m) {
    FlatModel f;
    f.sizes.assign(m.layer_sizes.begin(), m.layer_sizes.end());
    // validate(MlpModel) (mlp.cpp:209-226), same kinds and messages
    if (m.layer_sizes.size() < 2 || m.weights.size() != m.layer_sizes.size() - 1 ||
        m.biases.size() != m.weights.size())
        throw Error(ErrorKind::InvalidModel, "layer bookkeeping is inconsistent");
    for (std::size_t l = 0; l < m.weights.size(); ++l) {
        const auto& w = m.weights[l];
        if (w.rows() != m.layer_sizes[l + 1] || w.cols() != m.layer_sizes[l] ||
            m.biases[l].size() != m.layer_sizes[l + 1])
            throw Error(ErrorKind::InvalidModel, "weight shapes do not chain");
        for (Eigen::Index r = 0; r < w.rows(); ++r)
            for (Eigen::Index c = 0; c < w.cols(); ++c) f.W.push_back(w(r, c));
    }
    for (const auto& b : m.biases)
        for (Eigen::Index i = 0; i < b.size(); ++i) f.b.push_back(b[i]);
    const auto out = m.layer_sizes.back();
    if (m.target_mean.size() != out || m.target_std.size() != out)
        throw Error(ErrorKind::InvalidModel, "normalization stats do not match output");
    for (Eigen::Index i = 0; i < out; ++i) {
        if (!(m.target_std[i] > 0.0)) throw Error(ErrorKind::InvalidModel, "target std must be positive");
        f.mean.push_back(m.target_mean[i]);
        f.std_.push_back(m.target_std[i]);
    }
    return f;
}

inline void upload_model(GpuContext& ctx, const MlpModel& m) {
    const FlatModel f = flatten(m);
    check_status(dso_set_model(ctx.handle(), f.sizes.data(), static_cast<int32_t>(f.sizes.size()),
                               f.W.data(), f.b.data(), f.mean.data(), f.std_.data()),
                 ctx.handle());
}

// Read the device model back into an MlpModel of the same shape.
inline void download_model(GpuContext& ctx, MlpModel& m) {
    std::size_t nw = 0, nb = 0;
    for (std::size_t l = 0; l + 1 < m.layer_sizes.size(); ++l) {
        nw += static_cast<std::size_t>(m.layer_sizes[l]) * m.layer_sizes[l + 1];
        nb += m.layer_sizes[l + 1];
    }
    std::vector<double> W(nw), b(nb);
    check_status(dso_get_model(ctx.handle(), W.data(), b.data()), ctx.handle());
    std::size_t ow = 0, ob = 0;
    for (std::size_t l = 0; l + 1 < m.layer_sizes.size(); ++l) {
        auto& w = m.weights[l];
        for (Eigen::Index r = 0; r < w.rows(); ++r)
            for (Eigen::Index c = 0; c < w.cols(); ++c) w(r, c) = W[ow++];
        for (Eigen::Index i = 0; i < m.biases[l].size(); ++i) m.biases[l][i] = b[ob++];
    }
}

// Columns of x [rows x n] as a float [rows][n] device image.
inline std::vector<float> soa(const Eigen::MatrixXd& x) {
    std::vector<float> h(static_cast<std::size_t>(x.rows() * x.cols()));
    for (Eigen::Index r = 0; r < x.rows(); ++r)
        for (Eigen::Index c = 0; c < x.cols(); ++c)
            h[static_cast<std::size_t>(r * x.cols() + c)] = static_cast<float>(x(r, c));
    return h;
}

// KernelInstructionCounts -> the library's uint64 count rows [126][n]: canonical
// category name -> slot (instr 0..100, dtype 101..117, memspace 118..125).
inline std::vector<uint64_t> count_rows(std::span<const KernelInstructionCounts> counts) {
    const std::size_t n = counts.size();
    std::vector<uint64_t> rows(static_cast<std::size_t>(DSO_COUNT_ROWS) * n, 0);
    // the library's canonical tables (dso_category_name), the same lists as
    // instruction_categories() / data_type_categories() / memory_space_categories()
    const int base[3] = {0, DSO_INSTR_SLOTS, DSO_INSTR_SLOTS + DSO_DTYPE_SLOTS};
    const int len[3] = {DSO_INSTR_SLOTS, DSO_DTYPE_SLOTS, DSO_MEMSPACE_SLOTS};
    std::map<std::string, int> slot[3];
    for (int c = 0; c < 3; ++c)
        for (int i = 0; i < len[c]; ++i) slot[c][dso_category_name(base[c] + i)] = i;
    for (std::size_t k = 0; k < n; ++k) {
        const std::map<std::string, std::uint64_t>* maps[3] = {
            &counts[k].instr_counts, &counts[k].dtype_counts, &counts[k].memspace_counts};
        for (int c = 0; c < 3; ++c)
            for (const auto& [name, v] : *maps[c]) {
                auto it = slot[c].find(name);
                // the reference adds an unlisted key to the category total but gives it no
                // slot; the device stage has no row for it
                if (it == slot[c].end())
                    throw Error(ErrorKind::InvalidArgument,
                                "non-canonical category name '" + name + "'");
                rows[static_cast<std::size_t>(base[c] + it->second) * n + k] = v;
            }
    }
    return rows;
}

}  // namespace detail

// forward_raw for every column of x ([sizes[0] x n]) -> [sizes.back() x n].
inline Eigen::MatrixXd forward_raw_batch(const MlpModel& model, const Eigen::MatrixXd& x,
                                         GpuContext& ctx) {
    detail::upload_model(ctx, model);
    const int64_t n = x.cols();
    const int out = model.layer_sizes.back();
    if (x.rows() != model.layer_sizes.front())
        throw Error(ErrorKind::InvalidArgument, "input rows differ from the model's input width");
    Eigen::MatrixXd y(out, n);
    if (n == 0) return y;
    detail::DevBuf<float> dx(static_cast<std::size_t>(x.rows() * n)), draw(static_cast<std::size_t>(out * n));
    std::vector<float> hx = detail::soa(x), hr(static_cast<std::size_t>(out * n));
    dx.upload(hx.data());
    const bool seven = out == DSO_PARAM_ROWS;
    detail::DevBuf<float> dp(seven ? 7 * n : 1);
    detail::DevBuf<uint8_t> dc(seven ? n : 1);
    check_status(dso_predict(ctx.handle(), dx.get(), n, n, seven ? dp.get() : nullptr,
                             seven ? dc.get() : nullptr, draw.get()),
                 ctx.handle());
    check_status(dso_sync(ctx.handle()), ctx.handle());
    draw.download(hr.data());
    for (int o = 0; o < out; ++o)
        for (int64_t k = 0; k < n; ++k) y(o, k) = hr[static_cast<std::size_t>(o * n + k)];
    return y;
}

namespace detail {
inline std::vector<ParamPrediction> predict_from_device(GpuContext& ctx, const float* dx, int64_t n) {
    std::vector<ParamPrediction> out(static_cast<std::size_t>(n));
    if (n == 0) return out;
    DevBuf<float> dp(static_cast<std::size_t>(7 * n));
    DevBuf<uint8_t> dc(static_cast<std::size_t>(n));
    check_status(dso_predict(ctx.handle(), dx, n, n, dp.get(), dc.get(), nullptr), ctx.handle());
    check_status(dso_sync(ctx.handle()), ctx.handle());
    std::vector<float> hp(static_cast<std::size_t>(7 * n));
    std::vector<uint8_t> hc(static_cast<std::size_t>(n));
    dp.download(hp.data());
    dc.download(hc.data());
    for (int64_t k = 0; k < n; ++k) {
        auto p = [&](int j) { return static_cast<double>(hp[static_cast<std::size_t>(j * n + k)]); };
        out[k].params = KernelModelParams{p(0), p(1), p(2), p(3), p(4), p(5), p(6)};
        out[k].clamped = hc[k] != 0;
    }
    return out;
}
}  // namespace detail

// predict_params for every kernel's FusedFeatures (as_vector layout: DCGM 8 |
// instr 101 | dtype 17 | memspace 8).  The model must map 134 -> 7.
inline std::vector<ParamPrediction> predict_params_batch(const MlpModel& model,
                                                         std::span<const FusedFeatures> features,
                                                         GpuContext& ctx) {
    detail::upload_model(ctx, model);
    if (model.layer_sizes.front() != kFusedFeatureCount || model.layer_sizes.back() != kParamCount)
        throw Error(ErrorKind::InvalidModel, "predict_params needs a 134 -> 7 model");
    const int64_t n = static_cast<int64_t>(features.size());
    std::vector<float> h(static_cast<std::size_t>(kFusedFeatureCount * n));
    for (int64_t k = 0; k < n; ++k) {
        const FusedFeatures& f = features[k];
        const double d8[8] = {f.dcgm.smact, f.dcgm.smocc, f.dcgm.tenso, f.dcgm.drama,
                              f.dcgm.fp64a, f.dcgm.fp32a, f.dcgm.fp16a, f.dcgm.intac};
        auto put = [&](int row, double v) { h[static_cast<std::size_t>(row * n + k)] = static_cast<float>(v); };
        for (int j = 0; j < 8; ++j) put(j, d8[j]);
        for (int i = 0; i < 101; ++i) put(8 + i, f.ptx.instr[i]);
        for (int i = 0; i < 17; ++i) put(109 + i, f.ptx.dtype[i]);
        for (int i = 0; i < 8; ++i) put(126 + i, f.ptx.memspace[i]);
    }
    detail::DevBuf<float> dx(h.size());
    dx.upload(h.data());
    return detail::predict_from_device(ctx, dx.get(), n);
}

// featurize + as_vector for every kernel on the device (64-bit counts, exact
// totals): [134 x n], column k = FusedFeatures{dcgm[k], featurize(counts[k])}.as_vector().
inline Eigen::MatrixXd as_vector_batch(std::span<const KernelInstructionCounts> counts,
                                       std::span<const DcgmMetricVector> dcgm, GpuContext& ctx) {
    if (counts.size() != dcgm.size())
        throw Error(ErrorKind::InvalidArgument, "counts and dcgm sizes differ");
    const int64_t n = static_cast<int64_t>(counts.size());
    Eigen::MatrixXd out(kFusedFeatureCount, n);
    if (n == 0) return out;
    const std::vector<uint64_t> rows = detail::count_rows(counts);
    std::vector<float> dc(static_cast<std::size_t>(8 * n));
    for (int64_t k = 0; k < n; ++k) {
        const DcgmMetricVector& d = dcgm[k];
        const double v[8] = {d.smact, d.smocc, d.tenso, d.drama, d.fp64a, d.fp32a, d.fp16a, d.intac};
        for (int j = 0; j < 8; ++j) dc[static_cast<std::size_t>(j * n + k)] = static_cast<float>(v[j]);
    }
    detail::DevBuf<uint64_t> drows(rows.size());
    detail::DevBuf<float> ddc(dc.size()), dfused(static_cast<std::size_t>(kFusedFeatureCount * n));
    drows.upload(rows.data());
    ddc.upload(dc.data());
    check_status(dso_featurize_u64(ctx.handle(), drows.get(), ddc.get(), n, n, dfused.get()),
                 ctx.handle());
    check_status(dso_sync(ctx.handle()), ctx.handle());
    std::vector<float> h(static_cast<std::size_t>(kFusedFeatureCount * n));
    dfused.download(h.data());
    for (int r = 0; r < kFusedFeatureCount; ++r)
        for (int64_t k = 0; k < n; ++k) out(r, k) = h[static_cast<std::size_t>(r * n + k)];
    return out;
}

// featurize for every kernel: PtxFeatureVector{instr 101, dtype 17, memspace 8}.
inline std::vector<PtxFeatureVector> featurize_batch(std::span<const KernelInstructionCounts> counts,
                                                     GpuContext& ctx) {
    std::vector<DcgmMetricVector> zero(counts.size());
    const Eigen::MatrixXd f = as_vector_batch(counts, zero, ctx);
    std::vector<PtxFeatureVector> out(counts.size());
    for (std::size_t k = 0; k < counts.size(); ++k) {
        PtxFeatureVector& v = out[k];
        v.instr = Eigen::VectorXd(101);
        v.dtype = Eigen::VectorXd(17);
        v.memspace = Eigen::VectorXd(8);
        const auto c = static_cast<Eigen::Index>(k);
        for (int i = 0; i < 101; ++i) v.instr[i] = f(8 + i, c);
        for (int i = 0; i < 17; ++i) v.dtype[i] = f(109 + i, c);
        for (int i = 0; i < 8; ++i) v.memspace[i] = f(126 + i, c);
    }
    return out;
}

// features -> predict_params for kernels given as raw counts + DCGM (device
// featurize fused with the predictor input; no host-side normalisation).
inline std::vector<ParamPrediction> predict_params_batch(const MlpModel& model,
                                                         std::span<const KernelInstructionCounts> counts,
                                                         std::span<const DcgmMetricVector> dcgm,
                                                         GpuContext& ctx) {
    detail::upload_model(ctx, model);
    if (model.layer_sizes.front() != kFusedFeatureCount || model.layer_sizes.back() != kParamCount)
        throw Error(ErrorKind::InvalidModel, "predict_params needs a 134 -> 7 model");
    if (counts.size() != dcgm.size())
        throw Error(ErrorKind::InvalidArgument, "counts and dcgm sizes differ");
    const int64_t n = static_cast<int64_t>(counts.size());
    if (n == 0) return {};
    const std::vector<uint64_t> rows = detail::count_rows(counts);
    std::vector<float> dc(static_cast<std::size_t>(8 * n));
    for (int64_t k = 0; k < n; ++k) {
        const DcgmMetricVector& d = dcgm[k];
        const double v[8] = {d.smact, d.smocc, d.tenso, d.drama, d.fp64a, d.fp32a, d.fp16a, d.intac};
        for (int j = 0; j < 8; ++j) dc[static_cast<std::size_t>(j * n + k)] = static_cast<float>(v[j]);
    }
    detail::DevBuf<uint64_t> drows(rows.size());
    detail::DevBuf<float> ddc(dc.size()), dfused(static_cast<std::size_t>(kFusedFeatureCount * n));
    drows.upload(rows.data());
    ddc.upload(dc.data());
    check_status(dso_featurize_u64(ctx.handle(), drows.get(), ddc.get(), n, n, dfused.get()),
                 ctx.handle());
    return detail::predict_from_device(ctx, dfused.get(), n);
}

// load_dcgm_samples for many traces (host parse + per-metric mean, validated as
// the reference does; parsed on all host threads); throws for the first failing
// trace in index order, with the reference's kind and message.
inline std::vector<DcgmMetricVector> load_dcgm_samples_batch(std::span<const std::string_view> csv) {
    const std::size_t n = csv.size();
    std::vector<DcgmMetricVector> out(n);
    std::vector<int32_t> st(n, 0);
    std::vector<std::string> msg(n);
    const unsigned T = std::max(1u, std::min<unsigned>(std::thread::hardware_concurrency(), 64u));
    std::vector<std::thread> pool;
    for (unsigned t = 0; t < T; ++t)
        pool.emplace_back([&, t] {
            char m[512];
            for (std::size_t k = t; k < n; k += T) {
                double v[8];
                st[k] = dso_load_dcgm_csv(csv[k].data(), static_cast<int64_t>(csv[k].size()), v, m,
                                          sizeof(m));
                if (st[k]) {
                    msg[k] = m;
                    continue;
                }
                out[k] = DcgmMetricVector{v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7]};
            }
        });
    for (auto& th : pool) th.join();
    for (std::size_t k = 0; k < n; ++k)
        if (st[k]) throw Error(static_cast<ErrorKind>(st[k] - 1), msg[k]);
    return out;
}

// analytic_gradients / mse_loss on one batch (columns of x / y_std), on the device.
inline Gradients analytic_gradients_batch(const MlpModel& model, const Eigen::MatrixXd& x,
                                          const Eigen::MatrixXd& y_std, GpuContext& ctx,
                                          double* mse = nullptr) {
    detail::upload_model(ctx, model);
    const int64_t n = x.cols();
    const int out = model.layer_sizes.back();
    if (x.rows() != model.layer_sizes.front() || y_std.rows() != out || y_std.cols() != n)
        throw Error(ErrorKind::InvalidArgument, "batch shapes do not match the model");
    const int64_t np = dso_model_param_count(ctx.handle());
    detail::DevBuf<float> dx(static_cast<std::size_t>(x.rows() * n)), dy(static_cast<std::size_t>(out * n)),
        dg(static_cast<std::size_t>(np));
    detail::DevBuf<double> dl(1);
    std::vector<float> hx = detail::soa(x), hy = detail::soa(y_std);
    dx.upload(hx.data());
    dy.upload(hy.data());
    check_status(dso_train_grad(ctx.handle(), dx.get(), dy.get(), n, n, dg.get(), dl.get()),
                 ctx.handle());
    check_status(dso_sync(ctx.handle()), ctx.handle());
    std::vector<float> g(static_cast<std::size_t>(np));
    dg.download(g.data());
    double loss_sum = 0.0;
    dl.download(&loss_sum);
    const double s = 1.0 / (static_cast<double>(n) * out);  // mse_loss's 1/(B*out)
    if (mse) *mse = loss_sum * s;
    Gradients gr;
    std::size_t o = 0;
    for (std::size_t l = 0; l + 1 < model.layer_sizes.size(); ++l) {
        Eigen::MatrixXd w(model.layer_sizes[l + 1], model.layer_sizes[l]);
        for (Eigen::Index r = 0; r < w.rows(); ++r)
            for (Eigen::Index c = 0; c < w.cols(); ++c) w(r, c) = g[o++] * s;
        gr.weights.push_back(std::move(w));
    }
    for (std::size_t l = 0; l + 1 < model.layer_sizes.size(); ++l) {
        Eigen::VectorXd b(model.layer_sizes[l + 1]);
        for (Eigen::Index i = 0; i < b.size(); ++i) b[i] = g[o++] * s;
        gr.biases.push_back(std::move(b));
    }
    return gr;
}

inline double mse_loss_batch(const MlpModel& model, const Eigen::MatrixXd& x,
                             const Eigen::MatrixXd& y_std, GpuContext& ctx) {
    double l = 0.0;
    analytic_gradients_batch(model, x, y_std, ctx, &l);
    return l;
}

// ---- training --------------------------------------------------------------
// An ncclComm_t made by the library from a unique id the host broadcasts.
class NcclCommunicator {
public:
    static std::vector<uint8_t> unique_id() {
        std::vector<uint8_t> id(DSO_NCCL_ID_BYTES);
        check_status(dso_nccl_unique_id(id.data()), nullptr);
        return id;
    }
    NcclCommunicator(int nranks, const std::vector<uint8_t>& id, int rank, int device)
        : rank_(rank), nranks_(nranks) {
        check_status(dso_nccl_comm_init(nranks, id.data(), rank, device, &comm_), nullptr);
    }
    ~NcclCommunicator() { dso_nccl_comm_destroy(comm_); }
    NcclCommunicator(const NcclCommunicator&) = delete;
    NcclCommunicator& operator=(const NcclCommunicator&) = delete;
    void* handle() const { return comm_; }
    int rank() const { return rank_; }
    int nranks() const { return nranks_; }

private:
    void* comm_ = nullptr;
    int rank_, nranks_;
};

struct DataParallel {
    void* nccl_comm = nullptr;  // ncclComm_t
    int rank = 0, nranks = 1;
};

namespace detail {

constexpr double kMapeFloor = 1e-9;  // kMapeDenominatorFloor, mlp.cpp:14

// canonicalize (mlp.cpp:35-50)
inline std::vector<TrainingExample> canonical(std::vector<TrainingExample> d) {
    auto lex_less = [](const TrainingExample& a, const TrainingExample& b) {
        if (a.features.size() != b.features.size()) return a.features.size() < b.features.size();
        for (Eigen::Index i = 0; i < a.features.size(); ++i)
            if (a.features[i] != b.features[i]) return a.features[i] < b.features[i];
        if (a.targets.size() != b.targets.size()) return a.targets.size() < b.targets.size();
        for (Eigen::Index i = 0; i < a.targets.size(); ++i)
            if (a.targets[i] != b.targets[i]) return a.targets[i] < b.targets[i];
        return false;
    };
    std::sort(d.begin(), d.end(), lex_less);
    return d;
}

struct Stats {
    std::vector<double> mean, std_;
    std::vector<int> degenerate;
};

// target_stats (mlp.cpp:57-79): population mean / std, zero-variance dims unscaled
inline Stats target_stats(const std::vector<TrainingExample>& d) {
    const auto dim = d.front().targets.size();
    Stats s;
    s.mean.assign(dim, 0.0);
    for (const auto& ex : d)
        for (Eigen::Index i = 0; i < dim; ++i) s.mean[i] += ex.targets[i];
    for (auto& m : s.mean) m /= static_cast<double>(d.size());
    std::vector<double> var(dim, 0.0);
    for (const auto& ex : d)
        for (Eigen::Index i = 0; i < dim; ++i) {
            const double e = ex.targets[i] - s.mean[i];
            var[i] += e * e;
        }
    s.std_.resize(dim);
    for (Eigen::Index i = 0; i < dim; ++i) {
        s.std_[i] = std::sqrt(var[i] / static_cast<double>(d.size()));
        if (s.std_[i] == 0.0) {
            s.std_[i] = 1.0;
            s.mean[i] = 0.0;
            s.degenerate.push_back(static_cast<int>(i));
        }
    }
    return s;
}

// layer_sizes_for (mlp.cpp:148-153)
inline std::vector<int> sizes_for(const std::vector<TrainingExample>& d, const TrainConfig& cfg) {
    std::vector<int> s = cfg.layer_sizes.empty()
                             ? std::vector<int>{kFusedFeatureCount, 100, 50, 25, kParamCount}
                             : cfg.layer_sizes;
    s.front() = static_cast<int>(d.front().features.size());
    s.back() = static_cast<int>(d.front().targets.size());
    return s;
}

// init_mlp (mlp.cpp:184-207) through the library's host restatement
inline MlpModel init_model(const std::vector<int>& sizes, std::uint64_t seed) {
    if (sizes.size() < 2) throw Error(ErrorKind::InvalidModel, "need at least input and output layers");
    for (int s : sizes)
        if (s <= 0) throw Error(ErrorKind::InvalidModel, "layer sizes must be positive");
    std::size_t nw = 0, nb = 0;
    for (std::size_t l = 0; l + 1 < sizes.size(); ++l) {
        nw += static_cast<std::size_t>(sizes[l]) * sizes[l + 1];
        nb += sizes[l + 1];
    }
    std::vector<int32_t> s32(sizes.begin(), sizes.end());
    std::vector<double> W(nw), b(nb);
    check_status(dso_init_mlp(s32.data(), static_cast<int32_t>(s32.size()), seed, W.data(), b.data()),
                 nullptr);
    MlpModel m;
    m.layer_sizes = sizes;
    m.seed = seed;
    std::size_t ow = 0, ob = 0;
    for (std::size_t l = 0; l + 1 < sizes.size(); ++l) {
        Eigen::MatrixXd w(sizes[l + 1], sizes[l]);
        for (Eigen::Index r = 0; r < w.rows(); ++r)
            for (Eigen::Index c = 0; c < w.cols(); ++c) w(r, c) = W[ow++];
        Eigen::VectorXd bb(sizes[l + 1]);
        for (Eigen::Index i = 0; i < bb.size(); ++i) bb[i] = b[ob++];
        m.weights.push_back(std::move(w));
        m.biases.push_back(std::move(bb));
    }
    m.target_mean = Eigen::VectorXd(sizes.back());
    m.target_std = Eigen::VectorXd(sizes.back());
    for (int i = 0; i < sizes.back(); ++i) {
        m.target_mean[i] = 0.0;
        m.target_std[i] = 1.0;
    }
    return m;
}

// prediction_mape_pct (mlp.cpp:132-146) with the device forward
inline double mape_pct(const MlpModel& m, const std::vector<TrainingExample>& ex, GpuContext& ctx) {
    const auto in = ex.front().features.size(), out = ex.front().targets.size();
    Eigen::MatrixXd x(in, static_cast<Eigen::Index>(ex.size()));
    for (std::size_t k = 0; k < ex.size(); ++k)
        for (Eigen::Index i = 0; i < in; ++i) x(i, static_cast<Eigen::Index>(k)) = ex[k].features[i];
    const Eigen::MatrixXd pred = forward_raw_batch(m, x, ctx);
    double acc = 0.0;
    std::size_t terms = 0;
    for (std::size_t k = 0; k < ex.size(); ++k)
        for (Eigen::Index i = 0; i < out; ++i) {
            const double p = pred(i, static_cast<Eigen::Index>(k));
            if (!std::isfinite(p)) return std::numeric_limits<double>::infinity();
            acc += std::abs(p - ex[k].targets[i]) / std::max(std::abs(ex[k].targets[i]), kMapeFloor);
            ++terms;
        }
    return 100.0 * acc / static_cast<double>(terms);
}

}  // namespace detail

// fit_model (mlp.cpp:115-130) with the epochs on the device (dso_fit_model): a
// fresh init_mlp(sizes, seed) with the given statistics, sgd_epoch order and
// update rule; loss_trace receives the epoch losses (NaN-terminated on
// divergence).  `data` in the caller's (canonical) order.
inline MlpModel fit_model_gpu(const std::vector<TrainingExample>& data, const std::vector<int>& sizes,
                              const std::vector<double>& mean, const std::vector<double>& std_,
                              double lr, int batch_size, int epochs, std::uint64_t seed,
                              std::vector<double>* loss_trace, GpuContext& ctx,
                              const DataParallel& dp = {}) {
    MlpModel m = detail::init_model(sizes, seed);
    for (int i = 0; i < sizes.back(); ++i) {
        m.target_mean[i] = mean[i];
        m.target_std[i] = std_[i];
    }
    detail::upload_model(ctx, m);
    const int64_t n = static_cast<int64_t>(data.size());
    const int in = sizes.front(), out = sizes.back();
    std::vector<float> hx(static_cast<std::size_t>(in * n)), hy(static_cast<std::size_t>(out * n));
    for (int64_t k = 0; k < n; ++k) {
        for (int i = 0; i < in; ++i) hx[static_cast<std::size_t>(i * n + k)] = static_cast<float>(data[k].features[i]);
        for (int i = 0; i < out; ++i)
            hy[static_cast<std::size_t>(i * n + k)] =
                static_cast<float>((data[k].targets[i] - mean[i]) / std_[i]);
    }
    detail::DevBuf<float> dx(hx.size()), dy(hy.size());
    dx.upload(hx.data());
    dy.upload(hy.data());
    std::vector<double> trace(static_cast<std::size_t>(std::max(epochs, 1)));
    int32_t ran = 0;
    check_status(dso_fit_model(ctx.handle(), dx.get(), dy.get(), n, n, lr, batch_size, epochs, seed,
                               dp.nccl_comm, dp.rank, dp.nranks, trace.data(), &ran),
                 ctx.handle());
    if (loss_trace) loss_trace->assign(trace.begin(), trace.begin() + ran);
    detail::download_model(ctx, m);
    return m;
}

// cross_validate (mlp.cpp:348-411) with every fit and every validation forward on the device.
inline CvResult cross_validate_gpu(const std::vector<TrainingExample>& dataset,
                                   const std::vector<GridCell>& grid, const TrainConfig& cfg,
                                   GpuContext& ctx, const DataParallel& dp = {}) {
    if (dataset.size() < 3)
        throw Error(ErrorKind::DatasetTooSmall,
                    "cross-validation needs at least 3 examples, got " + std::to_string(dataset.size()));
    if (grid.empty()) throw Error(ErrorKind::InvalidArgument, "empty hyperparameter grid");
    const auto data = detail::canonical(dataset);
    const std::vector<int> sizes = detail::sizes_for(data, cfg);
    constexpr int kFolds = 3;
    Rng fold_rng = Rng(cfg.seed).fork(0xf01dULL);
    const auto order = shuffled_indices(data.size(), fold_rng);
    std::vector<int> fold_of(data.size());
    for (std::size_t i = 0; i < data.size(); ++i) fold_of[order[i]] = static_cast<int>(i % kFolds);
    CvResult result;
    for (std::size_t ci = 0; ci < grid.size(); ++ci) {
        CvCellResult row;
        row.cell = grid[ci];
        double acc = 0.0;
        for (int fold = 0; fold < kFolds; ++fold) {
            std::vector<TrainingExample> tr, va;
            for (std::size_t i = 0; i < data.size(); ++i) (fold_of[i] == fold ? va : tr).push_back(data[i]);
            double mape;
            if (tr.empty() || va.empty()) {
                mape = std::numeric_limits<double>::infinity();
            } else {
                const detail::Stats st = detail::target_stats(tr);
                std::vector<double> trace;
                const std::uint64_t run_seed = cfg.seed + 1000003ULL * static_cast<std::uint64_t>(fold) +
                                               29ULL * static_cast<std::uint64_t>(ci);
                MlpModel m = fit_model_gpu(tr, sizes, st.mean, st.std_, row.cell.learning_rate,
                                           row.cell.batch_size, cfg.epochs, run_seed, &trace, ctx, dp);
                const bool diverged = !trace.empty() && std::isnan(trace.back());
                mape = diverged ? std::numeric_limits<double>::infinity() : detail::mape_pct(m, va, ctx);
            }
            row.fold_mape_pct.push_back(mape);
            acc += mape;
        }
        row.mean_mape_pct = acc / kFolds;
        result.table.push_back(std::move(row));
    }
    const CvCellResult* best = &result.table.front();
    for (const auto& row : result.table)
        if (row.mean_mape_pct < best->mean_mape_pct ||
            (row.mean_mape_pct == best->mean_mape_pct &&
             (row.cell.learning_rate < best->cell.learning_rate ||
              (row.cell.learning_rate == best->cell.learning_rate &&
               row.cell.batch_size < best->cell.batch_size))))
            best = &row;
    result.best = best->cell;
    return result;
}

// train (mlp.cpp:413-437): checks, cross-validation over cfg.grid (or the single
// cell {learning_rate, batch_size}), then the final fit on the whole canonical set.
inline TrainResult train_gpu(const std::vector<TrainingExample>& dataset, const TrainConfig& cfg,
                             GpuContext& ctx, const DataParallel& dp = {}) {
    if (dataset.size() < 3)
        throw Error(ErrorKind::DatasetTooSmall,
                    "training needs at least 3 examples, got " + std::to_string(dataset.size()));
    for (const auto& ex : dataset)
        if (!ex.features.allFinite() || !ex.targets.allFinite())
            throw Error(ErrorKind::InvalidArgument, "dataset contains non-finite values");
    const auto data = detail::canonical(dataset);
    const std::vector<int> sizes = detail::sizes_for(data, cfg);
    const std::vector<GridCell> grid =
        cfg.grid.empty() ? std::vector<GridCell>{{cfg.learning_rate, cfg.batch_size}} : cfg.grid;
    TrainResult result;
    result.cv = cross_validate_gpu(data, grid, cfg, ctx, dp);
    const detail::Stats st = detail::target_stats(data);
    result.degenerate_targets = st.degenerate;
    result.model = fit_model_gpu(data, sizes, st.mean, st.std_, result.cv.best.learning_rate,
                                 result.cv.best.batch_size, cfg.epochs, cfg.seed, &result.epoch_loss,
                                 ctx, dp);
    return result;
}

}  // namespace dso
