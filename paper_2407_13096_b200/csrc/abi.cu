// abi.cu — the extern "C" boundary (include/dso_b200.h) and its host logic.
//
// Host-side restatements that the boundary needs (validation with the
// reference's error kinds, per-domain tables, Glorot init, Fisher-Yates) live
// here in C++; they are host code of the product, not a CPU compute path —
// every batched computation runs in the CUDA kernels.
#include <math.h>
#include <string.h>

#include <algorithm>
#include <cmath>
#include <new>
#include <string>
#include <vector>

#include "common.cuh"

using namespace dso_b200;

namespace {

int32_t fail(dso_ctx* ctx, int32_t st, const std::string& msg) {
    if (ctx) ctx->c.last_error = msg;
    return st;
}

int32_t cuda_fail(dso_ctx* ctx, cudaError_t e, const char* where) {
    return fail(ctx, kCuda, std::string(where) + ": " + cudaGetErrorString(e));
}

#define DSO_CUDA(ctx, expr)                                      \
    do {                                                         \
        cudaError_t _e = (expr);                                 \
        if (_e != cudaSuccess) return cuda_fail(ctx, _e, #expr); \
    } while (0)

bool is_device_ptr(const void* p) {
    if (!p) return true;
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ---- Rng (reference proj/include/dso/rng.hpp:11-64) --------------------------
struct HostRng {
    uint64_t s;
    uint64_t next() {
        uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    double uniform01() { return (double)(next() >> 11) * 0x1.0p-53; }
    double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
    uint64_t below(uint64_t n) {
        uint64_t x = next();
        __uint128_t m = (__uint128_t)x * n;
        uint64_t l = (uint64_t)m;
        if (l < n) {
            uint64_t t = (0ULL - n) % n;
            while (l < t) {
                x = next();
                m = (__uint128_t)x * n;
                l = (uint64_t)m;
            }
        }
        return (uint64_t)(m >> 64);
    }
};

// validate(DeviceConstants) dvfs_model.hpp:60-70 and validate(DvfsDomain)
// optimizer.cpp:58-88, same order, same kinds, same messages.
int32_t validate_domain(dso_ctx* ctx, const double* core, int nc, const double* mem, int nm,
                        const double* dev) {
    const double kvf = dev[0], pmax = dev[1], vmin = dev[2], vmax = dev[3], mpu = dev[4];
    if (!(vmin > 0.0) || !(vmin <= vmax))
        return fail(ctx, kInvalidArgument, "voltage bounds require 0 < vmin <= vmax");
    if (!(pmax > 0.0)) return fail(ctx, kInvalidArgument, "pmax must be positive");
    if (!(kvf < vmin))
        return fail(ctx, kInvalidArgument,
                    "kappa_vf must lie below vmin so the frequency bound stays real");
    if (!(mpu > 0.0)) return fail(ctx, kInvalidArgument, "mhz_per_unit must be positive");
    const double* tabs[2] = {core, mem};
    const int lens[2] = {nc, nm};
    const char* names[2] = {"core", "memory"};
    for (int t = 0; t < 2; ++t) {
        if (lens[t] <= 0 || !tabs[t])
            return fail(ctx, kInvalidArgument,
                        std::string(names[t]) + " frequency table is empty");
        double prev = 0.0;
        for (int i = 0; i < lens[t]; ++i) {
            if (!(tabs[t][i] > prev))
                return fail(ctx, kInvalidArgument,
                            std::string(names[t]) +
                                " frequencies must be positive and strictly increasing");
            prev = tabs[t][i];
        }
    }
    for (int i = 0; i < nc; ++i) {
        const double norm = core[i] / mpu;
        if (norm < kvf)
            return fail(ctx, kFrequencyBelowKappa,
                        "core frequency " + std::to_string(core[i]) +
                            " MHz normalizes below kappa_vf");
        const double d = norm - kvf;
        const double vc = 2.0 * d * d + kvf;
        if (vc < vmin || vc > vmax)
            return fail(ctx, kOutOfRange,
                        "core frequency " + std::to_string(core[i]) + " MHz induces voltage " +
                            std::to_string(vc) + " V outside [vmin, vmax]");
    }
    return kOk;
}

template <class T>
cudaError_t ensure(T*& p, size_t count) {
    if (p) {
        cudaFree(p);
        p = nullptr;
    }
    return cudaMalloc(&p, sizeof(T) * (count ? count : 1));
}

int32_t check_ctx(dso_ctx* ctx, bool need_domain, bool need_model) {
    if (!ctx) return kInvalidArgument;
    if (need_domain && !ctx->c.has_domain)
        return fail(ctx, kInvalidArgument, "no domain set (dso_set_domain)");
    if (need_model && !ctx->c.has_model)
        return fail(ctx, kInvalidModel, "no model set (dso_set_model)");
    cudaError_t e = cudaSetDevice(ctx->c.device);
    if (e != cudaSuccess) return cuda_fail(ctx, e, "cudaSetDevice");
    return kOk;
}

int32_t check_eta(dso_ctx* ctx, double eta) {
    // cost() throws EtaOutOfRange (dvfs_model.hpp:101-102)
    if (!(eta >= 0.0 && eta <= 1.0)) return fail(ctx, kEtaOutOfRange, "eta must lie in [0, 1]");
    return kOk;
}

int32_t check_batch(dso_ctx* ctx, int64_t n, int64_t ld) {
    if (n < 0 || ld < n) return fail(ctx, kInvalidArgument, "batch requires 0 <= n <= ld");
    return kOk;
}

}  // namespace

extern "C" {

int32_t dso_ctx_create(int32_t device, dso_ctx** out) {
    if (!out) return kInvalidArgument;
    *out = nullptr;
    cudaError_t e = cudaSetDevice(device);
    if (e != cudaSuccess) return kCuda;
    dso_ctx* ctx = new (std::nothrow) dso_ctx();
    if (!ctx) return kIoError;
    ctx->c.device = device;
    e = cudaStreamCreateWithFlags(&ctx->c.own_stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) {
        delete ctx;
        return kCuda;
    }
    ctx->c.stream = ctx->c.own_stream;
    for (auto& s : ctx->c.aux) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    for (auto& ev : ctx->c.ev) cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
    e = cudaMalloc(&ctx->c.counters_dev, sizeof(unsigned long long) * DSO_N_COUNTERS);
    if (e == cudaSuccess)
        e = cudaMemset(ctx->c.counters_dev, 0, sizeof(unsigned long long) * DSO_N_COUNTERS);
    if (e != cudaSuccess) {
        cudaStreamDestroy(ctx->c.own_stream);
        delete ctx;
        return kCuda;
    }
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    ctx->c.num_sms = sms > 0 ? sms : 148;
    *out = ctx;
    return kOk;
}

int32_t dso_ctx_destroy(dso_ctx* ctx) {
    if (!ctx) return kOk;
    Ctx& c = ctx->c;
    cudaSetDevice(c.device);
    cudaStreamSynchronize(c.stream);
    cudaFree(c.dom.core4);
    cudaFree(c.dom.mem2);
    cudaFree(c.dom.core_d);
    cudaFree(c.dom.mem_d);
    cudaFree(c.dom.g1_d);
    cudaFree(c.dom.sd_g1);
    cudaFree(c.eta_dev);
    cudaFree(c.flag_dev);
    fit_plan_free(c);
    cudaFree(c.model.wt);
    cudaFree(c.model.wtc);
    cudaFree(c.model.w_master);
    cudaFree(c.model.w_train);
    cudaFree(c.scratch);
    cudaFree(c.train_scratch);
    cudaFree(c.counters_dev);
    cudaFree(c.dp_grad);
    cudaFree(c.dp_dbl);
    cudaFree(c.gen_scratch);
    cudaFree(c.dcsr_scratch);
    cudaFree(c.model.gstats);
    for (auto& s : c.aux)
        if (s) cudaStreamDestroy(s);
    for (auto& ev : c.ev)
        if (ev) cudaEventDestroy(ev);
    if (c.own_stream) cudaStreamDestroy(c.own_stream);
    delete ctx;
    return kOk;
}

int32_t dso_ctx_set_stream(dso_ctx* ctx, void* stream) {
    if (!ctx) return kInvalidArgument;
    ctx->c.stream = (cudaStream_t)stream;  // NULL = legacy default stream
    return kOk;
}

int32_t dso_sync(dso_ctx* ctx) {
    if (!ctx) return kInvalidArgument;
    DSO_CUDA(ctx, cudaSetDevice(ctx->c.device));
    DSO_CUDA(ctx, cudaStreamSynchronize(ctx->c.stream));
    return kOk;
}

const char* dso_last_error(const dso_ctx* ctx) {
    return ctx ? ctx->c.last_error.c_str() : "null context";
}

const char* dso_status_name(int32_t st) {
    // dso::error_kind_name (error.hpp:27-44), shifted by one
    static const char* names[] = {"Ok",
                                  "MalformedPtx",
                                  "EmptyTrace",
                                  "OutOfRange",
                                  "SchemaMismatch",
                                  "NonPositivePower",
                                  "EtaOutOfRange",
                                  "VoltageBelowKappa",
                                  "FrequencyBelowKappa",
                                  "RankDeficient",
                                  "Underdetermined",
                                  "DatasetTooSmall",
                                  "InvalidArgument",
                                  "InvalidModel",
                                  "IoError"};
    if (st >= 0 && st <= 14) return names[st];
    if (st == kCuda) return "IoError";
    return "Unknown";
}

int64_t dso_launch_count(const dso_ctx* ctx) { return ctx ? ctx->c.launches : 0; }

int32_t dso_get_counters(dso_ctx* ctx, uint64_t* out, int32_t n, int32_t reset) {
    if (!ctx || n < 0 || (n > 0 && !out)) return kInvalidArgument;
    if (n > DSO_N_COUNTERS) return fail(ctx, kInvalidArgument, "more counters requested than exist");
    Ctx& c = ctx->c;
    DSO_CUDA(ctx, cudaSetDevice(c.device));
    DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
    unsigned long long h[DSO_N_COUNTERS] = {};
    DSO_CUDA(ctx, cudaMemcpy(h, c.counters_dev, sizeof(h), cudaMemcpyDeviceToHost));
    for (int i = 0; i < n; ++i) out[i] = h[i];
    if (reset) DSO_CUDA(ctx, cudaMemset(c.counters_dev, 0, sizeof(h)));
    return kOk;
}

int32_t dso_set_option(dso_ctx* ctx, const char* key, int64_t value) {
    if (!ctx || !key) return kInvalidArgument;
    if (std::string(key) == "mlp_engine") {
        if (value < 0 || value > 2) return fail(ctx, kInvalidArgument, "mlp_engine is 0, 1 or 2");
        ctx->c.mlp_engine = (int)value;
        return 0;
    }
    if (std::string(key) == "fast_sweep") {
        ctx->c.fast_sweep = value != 0;
        return kOk;
    }
    if (std::string(key) == "eta_prune") {
        ctx->c.eta_prune = value != 0;
        return kOk;
    }
    if (std::string(key) == "dense_csr") {
        ctx->c.dense_csr = value != 0;
        return kOk;
    }
    if (std::string(key) == "train_tc") {
        ctx->c.train_tc = value != 0;
        return kOk;
    }
    return fail(ctx, kInvalidArgument, std::string("unknown option: ") + key);
}

int32_t dso_set_domain(dso_ctx* ctx, const double* core, int32_t nc, const double* mem,
                       int32_t nm, const double* dev) {
    if (!ctx || !dev) return kInvalidArgument;
    int32_t st = validate_domain(ctx, core, nc, mem, nm, dev);
    if (st) return st;
    if (nc > kMaxCore || nm > kMaxMem)
        return fail(ctx, kInvalidArgument,
                    "domain larger than the device tables (1024 core x 64 memory levels)");
    Ctx& c = ctx->c;
    DSO_CUDA(ctx, cudaSetDevice(c.device));
    std::vector<float4> core4(nc);
    std::vector<float2> mem2(nm);
    std::vector<double2> core_d(nc);
    std::vector<double> g1(nc);
    std::vector<int> sd(nc);
    for (int i = 0; i < nc; ++i) {
        // required_voltage_mhz (dvfs_model.hpp:117-128), in double
        const double norm = core[i] / dev[4];
        const double d = norm - dev[0];
        const double vc = 2.0 * d * d + dev[0];
        core4[i] = make_float4((float)vc, (float)(vc * vc * core[i]), (float)(1.0 / core[i]),
                               (float)core[i]);
        core_d[i] = make_double2(vc, core[i]);
        // to_mhz(max_core_freq(vc)) (dvfs_model.hpp:107-113, optimizer.cpp:141-142)
        g1[i] = (std::sqrt((vc - dev[0]) / 2.0) + dev[0]) * dev[4];
        c.dom_core[i] = core[i];
    }
    for (int i = 0; i < nc; ++i) {  // snap_down(cores, g1) (optimizer.cpp:43-48)
        sd[i] = -1;
        for (int j = 0; j < nc; ++j)
            if (core[j] <= g1[i] * (1.0 + 1e-12)) sd[i] = j;
    }
    for (int j = 0; j < nm; ++j) {
        mem2[j] = make_float2((float)mem[j], (float)(1.0 / mem[j]));
        c.dom_mem[j] = mem[j];
    }
    for (int i = 0; i < 5; ++i) c.dom_dev[i] = dev[i];
    DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
    DSO_CUDA(ctx, ensure(c.dom.core4, nc));
    DSO_CUDA(ctx, ensure(c.dom.mem2, nm));
    DSO_CUDA(ctx, ensure(c.dom.core_d, nc));
    DSO_CUDA(ctx, ensure(c.dom.mem_d, nm));
    DSO_CUDA(ctx, cudaMemcpy(c.dom.core4, core4.data(), sizeof(float4) * nc,
                             cudaMemcpyHostToDevice));
    DSO_CUDA(ctx, cudaMemcpy(c.dom.mem2, mem2.data(), sizeof(float2) * nm,
                             cudaMemcpyHostToDevice));
    DSO_CUDA(ctx, cudaMemcpy(c.dom.core_d, core_d.data(), sizeof(double2) * nc,
                             cudaMemcpyHostToDevice));
    DSO_CUDA(ctx, cudaMemcpy(c.dom.mem_d, mem, sizeof(double) * nm, cudaMemcpyHostToDevice));
    DSO_CUDA(ctx, ensure(c.dom.g1_d, nc));
    DSO_CUDA(ctx, ensure(c.dom.sd_g1, nc));
    DSO_CUDA(ctx, cudaMemcpy(c.dom.g1_d, g1.data(), sizeof(double) * nc, cudaMemcpyHostToDevice));
    DSO_CUDA(ctx, cudaMemcpy(c.dom.sd_g1, sd.data(), sizeof(int) * nc, cudaMemcpyHostToDevice));
    c.dom.nc = nc;
    c.dom.nm = nm;
    // bounds that keep every f32 cost finite for params <= 1e12 and |K| <= 1e21
    // (P <= 1e12 (1 + vc + fm + vc^2 fc) <= 1e21, T <= 1e12 (1 + 1/fm + 1/fc) <= 1e15)
    bool fast = true;
    for (int i = 0; i < nc; ++i)
        fast = fast && core4[i].x >= 0.f && core4[i].x <= 1e3f && core4[i].y >= 0.f &&
               core4[i].y <= 1e8f && core4[i].z >= 0.f && core4[i].z <= 1e3f;
    for (int j = 0; j < nm; ++j)
        fast = fast && mem2[j].x >= 0.f && mem2[j].x <= 1e6f && mem2[j].y >= 0.f &&
               mem2[j].y <= 1e3f;
    c.dom.fast_ok = fast;
    bool sorted = true;
    for (int i = 1; i < nc; ++i)
        sorted = sorted && core4[i].x >= core4[i - 1].x && core4[i].y >= core4[i - 1].y &&
                 core4[i].z <= core4[i - 1].z;
    for (int j = 1; j < nm; ++j)
        sorted = sorted && mem2[j].x >= mem2[j - 1].x && mem2[j].y <= mem2[j - 1].y;
    c.dom.sorted_ok = sorted;
    c.has_domain = true;
    return kOk;
}

int32_t dso_validate_domain(const double* core, int32_t nc, const double* mem, int32_t nm,
                            const double* dev, char* msg, int32_t msg_len) {
    if (!dev) return kInvalidArgument;
    dso_ctx tmp;
    const int32_t st = validate_domain(&tmp, core, nc, mem, nm, dev);
    if (msg && msg_len > 0) {
        const std::string& m = tmp.c.last_error;
        const size_t len = std::min<size_t>(m.size(), (size_t)msg_len - 1);
        memcpy(msg, m.data(), len);
        msg[len] = 0;
    }
    return st;
}

int32_t dso_set_model(dso_ctx* ctx, const int32_t* sizes, int32_t n_sizes, const double* W,
                      const double* b, const double* mean, const double* std_) {
    if (!ctx) return kInvalidArgument;
    // validate(MlpModel) mlp.cpp:209-226 (shapes come from sizes here)
    if (!sizes || n_sizes < 2) return fail(ctx, kInvalidModel, "layer bookkeeping is inconsistent");
    for (int i = 0; i < n_sizes; ++i)
        if (sizes[i] <= 0) return fail(ctx, kInvalidModel, "layer sizes must be positive");
    if (!W || !b || !mean || !std_)
        return fail(ctx, kInvalidModel, "weight shapes do not chain");
    const int out = sizes[n_sizes - 1];
    for (int i = 0; i < out; ++i)
        if (!(std_[i] > 0.0)) return fail(ctx, kInvalidModel, "target std must be positive");
    static const int kDefault[5] = {134, 100, 50, 25, 7};
    bool is_default = n_sizes == 5;
    for (int i = 0; is_default && i < 5; ++i) is_default = sizes[i] == kDefault[i];
    // any other chain: the generic engine (mlp_gen.cu), within its limits
    int sum_w = 0, max_w = 0;
    for (int i = 0; i < n_sizes; ++i) {
        sum_w += sizes[i];
        max_w = std::max(max_w, sizes[i]);
    }
    if (!is_default && (n_sizes - 1 > kGenMaxLayers || max_w > kGenMaxWidth || sum_w > kGenMaxSumWidths))
        return fail(ctx, kInvalidModel,
                    "the device engine for non-default chains supports <= 8 layers, widths <= 256 "
                    "and a sum of widths <= 700");
    Ctx& c = ctx->c;
    DSO_CUDA(ctx, cudaSetDevice(c.device));
    ModelDev& md = c.model;
    for (int i = 0; i < n_sizes; ++i) md.sizes[i] = sizes[i];
    md.n_layers = n_sizes;
    md.generic = !is_default;
    for (int i = 0; i < 8; ++i) {
        md.mean[i] = i < out ? (float)mean[i] : 0.f;
        md.std_[i] = i < out ? (float)std_[i] : 1.f;
    }
    md.n_weights = 0;
    md.n_biases = 0;
    for (int l = 0; l + 1 < n_sizes; ++l) {
        md.n_weights += (int64_t)sizes[l] * sizes[l + 1];
        md.n_biases += sizes[l + 1];
    }
    std::vector<float> master(md.n_weights + md.n_biases);
    for (int64_t i = 0; i < md.n_weights; ++i) master[i] = (float)W[i];
    for (int64_t i = 0; i < md.n_biases; ++i) master[md.n_weights + i] = (float)b[i];
    DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
    if (md.w_master_cap < (int64_t)master.size()) {
        cudaFree(md.w_master);
        md.w_master = nullptr;
        md.w_master_cap = 0;
        DSO_CUDA(ctx, cudaMalloc(&md.w_master, sizeof(float) * master.size()));
        md.w_master_cap = (int64_t)master.size();
    }
    md.train_dirty = true;
    DSO_CUDA(ctx, cudaMemcpy(md.w_master, master.data(), sizeof(float) * master.size(),
                             cudaMemcpyHostToDevice));
    if (md.generic) {
        std::vector<float> st(2 * out);
        for (int i = 0; i < out; ++i) {
            st[i] = (float)mean[i];
            st[out + i] = (float)std_[i];
        }
        cudaFree(md.gstats);
        md.gstats = nullptr;
        DSO_CUDA(ctx, cudaMalloc(&md.gstats, sizeof(float) * st.size()));
        DSO_CUDA(ctx, cudaMemcpy(md.gstats, st.data(), sizeof(float) * st.size(),
                                 cudaMemcpyHostToDevice));
    } else {
        DSO_CUDA(ctx, model_upload(c, W, b));
    }
    DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
    c.has_model = true;
    return kOk;
}

int64_t dso_model_param_count(const dso_ctx* ctx) {
    return ctx && ctx->c.has_model ? ctx->c.model.n_weights + ctx->c.model.n_biases : 0;
}

int32_t dso_get_model(dso_ctx* ctx, double* W, double* b) {
    int32_t st = check_ctx(ctx, false, true);
    if (st) return st;
    ModelDev& md = ctx->c.model;
    std::vector<float> master(md.n_weights + md.n_biases);
    DSO_CUDA(ctx, cudaStreamSynchronize(ctx->c.stream));
    DSO_CUDA(ctx, cudaMemcpy(master.data(), md.w_master, sizeof(float) * master.size(),
                             cudaMemcpyDeviceToHost));
    if (W)
        for (int64_t i = 0; i < md.n_weights; ++i) W[i] = master[i];
    if (b)
        for (int64_t i = 0; i < md.n_biases; ++i) b[i] = master[md.n_weights + i];
    return kOk;
}

int32_t dso_init_mlp(const int32_t* sizes, int32_t n, uint64_t seed, double* W, double* b) {
    // init_mlp, mlp.cpp:184-207
    if (!sizes || n < 2) return kInvalidModel;
    for (int i = 0; i < n; ++i)
        if (sizes[i] <= 0) return kInvalidModel;
    HostRng rng{seed};
    for (int l = 0; l + 1 < n; ++l) {
        const int fan_in = sizes[l], fan_out = sizes[l + 1];
        const double limit = sqrt(6.0 / (fan_in + fan_out));
        for (int r = 0; r < fan_out; ++r)
            for (int cc = 0; cc < fan_in; ++cc) *W++ = rng.uniform(-limit, limit);
        for (int r = 0; r < fan_out; ++r) *b++ = 0.0;
    }
    return kOk;
}

int32_t dso_shuffled_indices(uint64_t n, uint64_t* state, uint64_t* out) {
    // shuffled_indices, rng.hpp:58-64
    if (!state || (!out && n)) return kInvalidArgument;
    HostRng rng{*state};
    for (uint64_t i = 0; i < n; ++i) out[i] = i;
    for (uint64_t i = n; i > 1; --i) {
        const uint64_t j = rng.below(i);
        std::swap(out[i - 1], out[j]);
    }
    *state = rng.s;
    return kOk;
}

int32_t dso_featurize(dso_ctx* ctx, const uint32_t* counts, const float* dcgm, int64_t n,
                      int64_t ld, float* fused) {
    int32_t st = check_ctx(ctx, false, false);
    if (st) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    DSO_CUDA(ctx, launch_featurize(ctx->c, counts, dcgm, n, ld, fused));
    return kOk;
}

int32_t dso_featurize_u64(dso_ctx* ctx, const uint64_t* counts, const float* dcgm, int64_t n,
                          int64_t ld, float* fused) {
    int32_t st = check_ctx(ctx, false, false);
    if (st) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    DSO_CUDA(ctx, launch_featurize_u64(ctx->c, counts, dcgm, n, ld, fused));
    return kOk;
}

int32_t dso_dcgm_mean(dso_ctx* ctx, const double* samples, int64_t rows, int64_t n,
                      int64_t ld, float* out, int64_t* bad_row) {
    int32_t st = check_ctx(ctx, false, false);
    if (st) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    if (rows < 1) return fail(ctx, kEmptyTrace, "no data rows");
    if (!ctx->c.flag_dev) DSO_CUDA(ctx, cudaMalloc(&ctx->c.flag_dev, sizeof(int)));
    int* flag = ctx->c.flag_dev;
    DSO_CUDA(ctx, cudaMemsetAsync(flag, 0, sizeof(int), ctx->c.stream));
    DSO_CUDA(ctx, launch_dcgm_mean(ctx->c, samples, rows, n, ld, out, bad_row, flag));
    int h = 0;
    DSO_CUDA(ctx, cudaMemcpyAsync(&h, flag, sizeof(int), cudaMemcpyDeviceToHost, ctx->c.stream));
    DSO_CUDA(ctx, cudaStreamSynchronize(ctx->c.stream));
    if (h) return fail(ctx, kOutOfRange, "metric value outside [0, 1] (see bad_row)");
    return kOk;
}

int32_t dso_predict(dso_ctx* ctx, const float* fused, int64_t n, int64_t ld, float* params,
                    uint8_t* clamped, float* raw) {
    int32_t st = check_ctx(ctx, false, true);
    if (st) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    DSO_CUDA(ctx, launch_predict(ctx->c, fused, n, ld, params, clamped, raw));
    return kOk;
}

int32_t dso_sweep(dso_ctx* ctx, const float* params, int64_t n, int64_t ld, double eta,
                  double pmax, int32_t* idx, float* cost, float* energy, float* time,
                  int32_t* kstatus) {
    int32_t st = check_ctx(ctx, true, false);
    if (st) return st;
    if ((st = check_eta(ctx, eta))) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    const float K = (float)((1.0 - eta) * pmax);
    DSO_CUDA(ctx, launch_sweep_f32(ctx->c, params, n, ld, (float)eta, K, idx, cost, energy, time,
                                   kstatus));
    return kOk;
}

int32_t dso_sweep_f64(dso_ctx* ctx, const double* params, int64_t n, double eta, double pmax,
                      int32_t* idx, double* cost, double* energy, double* time,
                      int32_t* kstatus, uint32_t flags) {
    int32_t st = check_ctx(ctx, true, false);
    if (st) return st;
    if ((st = check_eta(ctx, eta))) return st;
    if (n < 0) return fail(ctx, kInvalidArgument, "n < 0");
    const double K = (1.0 - eta) * pmax;  // dvfs_model.hpp:103, (1 - eta) * pmax
    Ctx& c = ctx->c;
    if (!(flags & DSO_HOST)) {
        DSO_CUDA(ctx, launch_sweep_f64(c, params, n, eta, K, idx, cost, energy, time, kstatus));
        return kOk;
    }
    // host buffers: stage through the device in chunks on the context stream
    const int64_t chunk = std::min<int64_t>(n, 1 << 22);
    const size_t per = 7 * sizeof(double) + sizeof(int32_t) * 2 + 3 * sizeof(double);
    const size_t need = (size_t)chunk * per;
    if (c.scratch_bytes < need) {
        cudaFree(c.scratch);
        c.scratch = nullptr;
        c.scratch_bytes = 0;
        DSO_CUDA(ctx, cudaMalloc(&c.scratch, need));
        c.scratch_bytes = need;
    }
    char* base = (char*)c.scratch;
    double* dp = (double*)base;
    double* dc = dp + 7 * chunk;
    double* de = dc + chunk;
    double* dt = de + chunk;
    int32_t* di = (int32_t*)(dt + chunk);
    int32_t* dk = di + chunk;
    for (int64_t off = 0; off < n; off += chunk) {
        const int64_t m = std::min(chunk, n - off);
        DSO_CUDA(ctx, cudaMemcpyAsync(dp, params + 7 * off, sizeof(double) * 7 * m,
                                      cudaMemcpyHostToDevice, c.stream));
        DSO_CUDA(ctx, launch_sweep_f64(c, dp, m, eta, K, di, dc, de, dt, dk));
        if (idx) DSO_CUDA(ctx, cudaMemcpyAsync(idx + off, di, 4 * m, cudaMemcpyDeviceToHost, c.stream));
        if (cost) DSO_CUDA(ctx, cudaMemcpyAsync(cost + off, dc, 8 * m, cudaMemcpyDeviceToHost, c.stream));
        if (energy)
            DSO_CUDA(ctx, cudaMemcpyAsync(energy + off, de, 8 * m, cudaMemcpyDeviceToHost, c.stream));
        if (time) DSO_CUDA(ctx, cudaMemcpyAsync(time + off, dt, 8 * m, cudaMemcpyDeviceToHost, c.stream));
        if (kstatus)
            DSO_CUDA(ctx, cudaMemcpyAsync(kstatus + off, dk, 4 * m, cudaMemcpyDeviceToHost, c.stream));
    }
    DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
    return kOk;
}

int32_t dso_optimal_config(dso_ctx* ctx, const double* params, int64_t n, double eta,
                           double pmax, int32_t* idx, double* cost, double* energy,
                           double* time, int64_t* candidates, uint8_t* fallback,
                           double* presnap, int32_t* kstatus, uint32_t flags) {
    int32_t st = check_ctx(ctx, true, false);
    if (st) return st;
    if ((st = check_eta(ctx, eta))) return st;  // optimizer.cpp:123-124
    if (n < 0) return fail(ctx, kInvalidArgument, "n < 0");
    if (!idx) return fail(ctx, kInvalidArgument, "idx output is required");
    const double K = (1.0 - eta) * pmax;
    Ctx& c = ctx->c;
    if (!(flags & DSO_HOST)) {
        DSO_CUDA(ctx, launch_optimal_config(c, params, n, eta, K, idx, cost, energy, time,
                                            candidates, fallback, presnap, kstatus));
        return kOk;
    }
    // host buffers: stage through the device in chunks on the context stream
    const int64_t chunk = std::min<int64_t>(std::max<int64_t>(n, 1), 1 << 21);
    const size_t per = 7 * 8 + 3 * 8 + 8 + 3 * 8 + 4 + 4 + 1;
    const size_t need = (size_t)chunk * per + 64;
    if (c.scratch_bytes < need) {
        DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
        cudaFree(c.scratch);
        c.scratch = nullptr;
        c.scratch_bytes = 0;
        DSO_CUDA(ctx, cudaMalloc(&c.scratch, need));
        c.scratch_bytes = need;
    }
    double* dp = (double*)c.scratch;
    double* dc = dp + 7 * chunk;
    double* de = dc + chunk;
    double* dt = de + chunk;
    double* dps = dt + chunk;
    int64_t* dn = (int64_t*)(dps + 3 * chunk);
    int32_t* di = (int32_t*)(dn + chunk);
    int32_t* dk = di + chunk;
    uint8_t* df = (uint8_t*)(dk + chunk);
    for (int64_t off = 0; off < n; off += chunk) {
        const int64_t m = std::min(chunk, n - off);
        DSO_CUDA(ctx, cudaMemcpyAsync(dp, params + 7 * off, sizeof(double) * 7 * m,
                                      cudaMemcpyHostToDevice, c.stream));
        DSO_CUDA(ctx, launch_optimal_config(c, dp, m, eta, K, di, dc, de, dt, dn, df, dps, dk));
        auto back = [&](void* h, const void* d, size_t bytes) {
            return h ? cudaMemcpyAsync(h, d, bytes, cudaMemcpyDeviceToHost, c.stream)
                     : cudaSuccess;
        };
        DSO_CUDA(ctx, back(idx + off, di, 4 * m));
        DSO_CUDA(ctx, back(cost ? cost + off : nullptr, dc, 8 * m));
        DSO_CUDA(ctx, back(energy ? energy + off : nullptr, de, 8 * m));
        DSO_CUDA(ctx, back(time ? time + off : nullptr, dt, 8 * m));
        DSO_CUDA(ctx, back(candidates ? candidates + off : nullptr, dn, 8 * m));
        DSO_CUDA(ctx, back(fallback ? fallback + off : nullptr, df, m));
        DSO_CUDA(ctx, back(presnap ? presnap + 3 * off : nullptr, dps, 24 * m));
        DSO_CUDA(ctx, back(kstatus ? kstatus + off : nullptr, dk, 4 * m));
    }
    DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
    return kOk;
}

int32_t dso_param_fit(dso_ctx* ctx, const double* cfg, int32_t S, const double* power,
                      const double* time, int64_t n, int64_t ld, double* pfit,
                      int32_t* pstatus, double* tfit, int32_t* tstatus, uint32_t flags) {
    int32_t st = check_ctx(ctx, false, false);
    if (st) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    if (S < 0 || (S > 0 && !cfg)) return fail(ctx, kInvalidArgument, "bad sample grid");
    if (!power && !time) return fail(ctx, kInvalidArgument, "power and time are both NULL");
    Ctx& c = ctx->c;
    DSO_CUDA(ctx, fit_prepare(c, cfg, S));
    if (!(flags & DSO_HOST)) {
        DSO_CUDA(ctx, launch_param_fit(c, power, time, n, ld, pfit, pstatus, tfit, tstatus));
        return kOk;
    }
    // host buffers: chunks of kernels staged through the device
    const int64_t chunk = std::max<int64_t>(1, std::min<int64_t>(n, (int64_t)(1 << 28) / (16 * (S + 8))));
    const size_t per = (size_t)8 * (2 * (size_t)S + 6 + 8) + 8;
    const size_t need = (size_t)chunk * per + 256;
    if (c.scratch_bytes < need) {
        DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
        cudaFree(c.scratch);
        c.scratch = nullptr;
        c.scratch_bytes = 0;
        DSO_CUDA(ctx, cudaMalloc(&c.scratch, need));
        c.scratch_bytes = need;
    }
    double* dp = (double*)c.scratch;
    double* dt = dp + (size_t)S * chunk;
    double* dpf = dt + (size_t)S * chunk;
    double* dtf = dpf + 6 * (size_t)chunk;
    int32_t* dps = (int32_t*)(dtf + 8 * (size_t)chunk);
    int32_t* dts = dps + chunk;
    for (int64_t off = 0; off < n; off += chunk) {
        const int64_t m = std::min(chunk, n - off);
        if (power)
            DSO_CUDA(ctx, cudaMemcpy2DAsync(dp, m * 8, power + off, ld * 8, m * 8, S,
                                            cudaMemcpyHostToDevice, c.stream));
        if (time)
            DSO_CUDA(ctx, cudaMemcpy2DAsync(dt, m * 8, time + off, ld * 8, m * 8, S,
                                            cudaMemcpyHostToDevice, c.stream));
        DSO_CUDA(ctx, launch_param_fit(c, power ? dp : nullptr, time ? dt : nullptr, m, m, dpf,
                                       dps, dtf, dts));
        if (power && pfit)
            DSO_CUDA(ctx, cudaMemcpy2DAsync(pfit + off, ld * 8, dpf, m * 8, m * 8, 6,
                                            cudaMemcpyDeviceToHost, c.stream));
        if (power && pstatus)
            DSO_CUDA(ctx, cudaMemcpyAsync(pstatus + off, dps, 4 * m, cudaMemcpyDeviceToHost, c.stream));
        if (time && tfit)
            DSO_CUDA(ctx, cudaMemcpy2DAsync(tfit + off, ld * 8, dtf, m * 8, m * 8, 8,
                                            cudaMemcpyDeviceToHost, c.stream));
        if (time && tstatus)
            DSO_CUDA(ctx, cudaMemcpyAsync(tstatus + off, dts, 4 * m, cudaMemcpyDeviceToHost, c.stream));
    }
    DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
    return kOk;
}

int32_t dso_eta_sweep(dso_ctx* ctx, const float* params, int64_t n, int64_t ld,
                      const double* etas, int32_t n_eta, double pmax, int32_t* idx,
                      float* cost, int64_t ld_out) {
    int32_t st = check_ctx(ctx, true, false);
    if (st) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    if (ld_out < n) return fail(ctx, kInvalidArgument, "ld_out < n");
    if (n_eta <= 0 || !etas) return fail(ctx, kInvalidArgument, "empty eta list");
    std::vector<float2> ek(n_eta);
    for (int e = 0; e < n_eta; ++e) {
        if ((st = check_eta(ctx, etas[e]))) return st;
        ek[e] = make_float2((float)etas[e], (float)((1.0 - etas[e]) * pmax));
    }
    Ctx& c = ctx->c;
    // per-context eta table (grown on demand); a pageable H2D copy returns once
    // the host data is staged, so ek may go out of scope afterwards
    if (c.eta_cap < n_eta) {
        DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
        cudaFree(c.eta_dev);
        c.eta_dev = nullptr;
        c.eta_cap = 0;
        DSO_CUDA(ctx, cudaMalloc(&c.eta_dev, sizeof(float2) * n_eta));
        c.eta_cap = n_eta;
    }
    DSO_CUDA(ctx, cudaMemcpyAsync(c.eta_dev, ek.data(), sizeof(float2) * n_eta,
                                  cudaMemcpyHostToDevice, c.stream));
    bool fast = true, k_nonneg = true;
    for (int e = 0; e < n_eta; ++e) {
        fast = fast && fast_sweep_ok(c, ek[e].y);
        k_nonneg = k_nonneg && ek[e].x >= 0.f && ek[e].y >= 0.f;
    }
    DSO_CUDA(ctx, launch_eta_sweep(c, params, n, ld, c.eta_dev, n_eta, idx, cost, ld_out, fast,
                                   fast && k_nonneg && c.eta_prune && c.dom.sorted_ok));
    return kOk;
}

int32_t dso_gen_synthetic(dso_ctx* ctx, uint64_t root, uint64_t salt_base, int64_t first,
                          int64_t n, int64_t ld, float* params, uint32_t* counts, float* dcgm) {
    int32_t st = check_ctx(ctx, false, false);
    if (st) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    DSO_CUDA(ctx, launch_gen(ctx->c, root, salt_base, first, n, ld, params, counts, dcgm));
    return kOk;
}

int32_t dso_pipeline(dso_ctx* ctx, const uint32_t* counts, const float* dcgm, int64_t n,
                     int64_t ld, double eta, double pmax, float* params, uint8_t* clamped,
                     int32_t* idx, float* cost, float* energy, float* time, uint32_t flags) {
    int32_t st = check_ctx(ctx, true, true);
    if (st) return st;
    if ((st = check_eta(ctx, eta))) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    if (!idx) return fail(ctx, kInvalidArgument, "idx output is required");
    Ctx& c = ctx->c;
    const float K = (float)((1.0 - eta) * pmax);
    if (!(flags & DSO_HOST)) {
        // auto engine: the dense counts go through the CSR form to the tensor-core pipeline
        if (c.dense_csr && c.mlp_engine == 2 && tc_csr_eligible(c)) {
            bool done = false;
            DSO_CUDA(ctx, launch_pipeline_dense_via_csr(c, counts, dcgm, n, ld, (float)eta, K,
                                                        params, clamped, idx, cost, energy, time,
                                                        &done));
            if (done) return kOk;
        }
        DSO_CUDA(ctx, launch_pipeline(c, counts, dcgm, n, ld, (float)eta, K, params, clamped,
                                      idx, cost, energy, time, ld));
        return kOk;
    }
    // ---- host buffers: chunked, double-buffered H2D / compute / D2H --------------
    // Per chunk of CH kernels: counts [126][CH] u32 + dcgm [8][CH] f32 in, results
    // out.  Copies of chunk i+1 overlap the kernel of chunk i (aux[0] = H2D,
    // c.stream = compute, aux[1] = D2H), ordered with events.
    const int64_t CH = std::min<int64_t>(n, (int64_t)1 << 20);
    const size_t in_b = (size_t)CH * (126 * 4 + 8 * 4);
    const size_t out_b = (size_t)CH * (4 + 4 + 4 + 4 + 7 * 4 + 1);
    const size_t need = 2 * (in_b + out_b) + 256;
    if (c.scratch_bytes < need) {
        DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
        cudaFree(c.scratch);
        c.scratch = nullptr;
        c.scratch_bytes = 0;
        DSO_CUDA(ctx, cudaMalloc(&c.scratch, need));
        c.scratch_bytes = need;
    }
    struct Buf {
        uint32_t* cnt;
        float* dc;
        int32_t* idx;
        float *cost, *energy, *time, *params;
        uint8_t* cl;
    } buf[2];
    char* p = (char*)c.scratch;
    for (int s = 0; s < 2; ++s) {
        buf[s].cnt = (uint32_t*)p;
        p += (size_t)CH * 126 * 4;
        buf[s].dc = (float*)p;
        p += (size_t)CH * 8 * 4;
        buf[s].idx = (int32_t*)p;
        p += (size_t)CH * 4;
        buf[s].cost = (float*)p;
        p += (size_t)CH * 4;
        buf[s].energy = (float*)p;
        p += (size_t)CH * 4;
        buf[s].time = (float*)p;
        p += (size_t)CH * 4;
        buf[s].params = (float*)p;
        p += (size_t)CH * 7 * 4;
        buf[s].cl = (uint8_t*)p;
        p += ((size_t)CH + 15) / 16 * 16;
    }
    cudaStream_t h2d = c.aux[0], d2h = c.aux[1];
    cudaEvent_t in_ready[2] = {c.ev[0], c.ev[1]};
    cudaEvent_t done[2] = {c.ev[2], c.ev[3]};
    cudaEvent_t drained[2] = {c.ev[4], c.ev[5]};
    DSO_CUDA(ctx, cudaEventRecord(drained[0], c.stream));
    DSO_CUDA(ctx, cudaEventRecord(drained[1], c.stream));
    int64_t chunk_i = 0;
    for (int64_t off = 0; off < n; off += CH, ++chunk_i) {
        const int s = (int)(chunk_i & 1);
        const int64_t m = std::min(CH, n - off);
        Buf& B = buf[s];
        // inputs: wait until the previous user of this buffer has been drained
        DSO_CUDA(ctx, cudaStreamWaitEvent(h2d, drained[s], 0));
        DSO_CUDA(ctx, cudaMemcpy2DAsync(B.cnt, (size_t)CH * 4, counts + off, (size_t)ld * 4,
                                        (size_t)m * 4, 126, cudaMemcpyHostToDevice, h2d));
        DSO_CUDA(ctx, cudaMemcpy2DAsync(B.dc, (size_t)CH * 4, dcgm + off, (size_t)ld * 4,
                                        (size_t)m * 4, 8, cudaMemcpyHostToDevice, h2d));
        DSO_CUDA(ctx, cudaEventRecord(in_ready[s], h2d));
        DSO_CUDA(ctx, cudaStreamWaitEvent(c.stream, in_ready[s], 0));
        DSO_CUDA(ctx, launch_pipeline(c, B.cnt, B.dc, m, CH, (float)eta, K,
                                      params ? B.params : nullptr, clamped ? B.cl : nullptr,
                                      B.idx, cost ? B.cost : nullptr,
                                      energy ? B.energy : nullptr, time ? B.time : nullptr, CH));
        DSO_CUDA(ctx, cudaEventRecord(done[s], c.stream));
        DSO_CUDA(ctx, cudaStreamWaitEvent(d2h, done[s], 0));
        DSO_CUDA(ctx, cudaMemcpyAsync(idx + off, B.idx, 4 * m, cudaMemcpyDeviceToHost, d2h));
        if (cost)
            DSO_CUDA(ctx, cudaMemcpyAsync(cost + off, B.cost, 4 * m, cudaMemcpyDeviceToHost, d2h));
        if (energy)
            DSO_CUDA(ctx,
                     cudaMemcpyAsync(energy + off, B.energy, 4 * m, cudaMemcpyDeviceToHost, d2h));
        if (time)
            DSO_CUDA(ctx, cudaMemcpyAsync(time + off, B.time, 4 * m, cudaMemcpyDeviceToHost, d2h));
        if (params)
            DSO_CUDA(ctx, cudaMemcpy2DAsync(params + off, (size_t)ld * 4, B.params,
                                            (size_t)CH * 4, (size_t)m * 4, 7,
                                            cudaMemcpyDeviceToHost, d2h));
        if (clamped)
            DSO_CUDA(ctx, cudaMemcpyAsync(clamped + off, B.cl, m, cudaMemcpyDeviceToHost, d2h));
        // the input buffer s is free once the kernel is done; outputs once D2H is done
        DSO_CUDA(ctx, cudaEventRecord(drained[s], d2h));
    }
    DSO_CUDA(ctx, cudaStreamSynchronize(d2h));
    return kOk;
}

int32_t dso_gen_synthetic_csr(dso_ctx* ctx, uint64_t root, uint64_t salt_base, int64_t first,
                              int64_t n, uint64_t* row_ptr, uint32_t* entries, float* dcgm,
                              int64_t ld) {
    int32_t st = check_ctx(ctx, false, false);
    if (st) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    if (!row_ptr || (!entries && n)) return fail(ctx, kInvalidArgument, "row_ptr/entries required");
    DSO_CUDA(ctx, launch_gen_csr(ctx->c, root, salt_base, first, n, row_ptr, entries, dcgm, ld));
    return kOk;
}

int32_t dso_pipeline_csr(dso_ctx* ctx, const uint64_t* row_ptr, const uint32_t* entries,
                         uint64_t ent_base, const float* dcgm, int64_t n, int64_t ld, double eta,
                         double pmax, float* params, uint8_t* clamped, int32_t* idx, float* cost,
                         float* energy, float* time, uint32_t flags) {
    int32_t st = check_ctx(ctx, true, true);
    if (st) return st;
    if ((st = check_eta(ctx, eta))) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    if (!idx || !row_ptr || !dcgm) return fail(ctx, kInvalidArgument, "idx, row_ptr, dcgm required");
    Ctx& c = ctx->c;
    const float K = (float)((1.0 - eta) * pmax);
    if (!(flags & DSO_HOST)) {
        DSO_CUDA(ctx, launch_pipeline_csr(c, row_ptr, entries, ent_base, dcgm, n, ld, (float)eta,
                                          K, params, clamped, idx, cost, energy, time, ld));
        return kOk;
    }
    // ---- host buffers: chunked, double-buffered H2D / compute / D2H ----------------
#ifndef DSO_HOST_CSR_CHUNK_LOG2
#define DSO_HOST_CSR_CHUNK_LOG2 20
#endif
    const int64_t CH = std::min<int64_t>(n, (int64_t)1 << DSO_HOST_CSR_CHUNK_LOG2);
    uint64_t max_ent = 0;
    for (int64_t off = 0; off < n; off += CH) {
        const int64_t m = std::min(CH, n - off);
        max_ent = std::max<uint64_t>(max_ent, row_ptr[off + m] - row_ptr[off]);
    }
    const size_t in_b = (size_t)(CH + 1) * 8 + (size_t)max_ent * 4 + (size_t)CH * 8 * 4 + 64;
    const size_t out_b = (size_t)CH * (4 + 4 + 4 + 4 + 7 * 4) + (size_t)CH + 64;
    const size_t need = 2 * (in_b + out_b) + 512;
    if (c.scratch_bytes < need) {
        DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
        cudaFree(c.scratch);
        c.scratch = nullptr;
        c.scratch_bytes = 0;
        DSO_CUDA(ctx, cudaMalloc(&c.scratch, need));
        c.scratch_bytes = need;
    }
    struct Buf {
        uint64_t* rp;
        uint32_t* ent;
        float* dc;
        int32_t* idx;
        float *cost, *energy, *time, *params;
        uint8_t* cl;
    } buf[2];
    auto align = [](char* p) { return (char*)(((uintptr_t)p + 15) & ~(uintptr_t)15); };
    char* p = (char*)c.scratch;
    for (int s = 0; s < 2; ++s) {
        p = align(p);
        buf[s].rp = (uint64_t*)p;
        p = align(p + (size_t)(CH + 1) * 8);
        buf[s].ent = (uint32_t*)p;
        p = align(p + (size_t)max_ent * 4);
        buf[s].dc = (float*)p;
        p = align(p + (size_t)CH * 8 * 4);
        buf[s].idx = (int32_t*)p;
        p = align(p + (size_t)CH * 4);
        buf[s].cost = (float*)p;
        p = align(p + (size_t)CH * 4);
        buf[s].energy = (float*)p;
        p = align(p + (size_t)CH * 4);
        buf[s].time = (float*)p;
        p = align(p + (size_t)CH * 4);
        buf[s].params = (float*)p;
        p = align(p + (size_t)CH * 7 * 4);
        buf[s].cl = (uint8_t*)p;
        p += CH;
    }
    cudaStream_t h2d = c.aux[0], d2h = c.aux[1];
    cudaEvent_t in_ready[2] = {c.ev[0], c.ev[1]};
    cudaEvent_t done[2] = {c.ev[2], c.ev[3]};
    cudaEvent_t drained[2] = {c.ev[4], c.ev[5]};
    DSO_CUDA(ctx, cudaEventRecord(drained[0], c.stream));
    DSO_CUDA(ctx, cudaEventRecord(drained[1], c.stream));
    int64_t chunk_i = 0;
    for (int64_t off = 0; off < n; off += CH, ++chunk_i) {
        const int s = (int)(chunk_i & 1);
        const int64_t m = std::min(CH, n - off);
        Buf& B = buf[s];
        const uint64_t e0 = row_ptr[off], e1 = row_ptr[off + m];
        DSO_CUDA(ctx, cudaStreamWaitEvent(h2d, drained[s], 0));
        DSO_CUDA(ctx, cudaMemcpyAsync(B.rp, row_ptr + off, (size_t)(m + 1) * 8,
                                      cudaMemcpyHostToDevice, h2d));
        if (e1 > e0)
            DSO_CUDA(ctx, cudaMemcpyAsync(B.ent, entries + (e0 - ent_base), (size_t)(e1 - e0) * 4,
                                          cudaMemcpyHostToDevice, h2d));
        DSO_CUDA(ctx, cudaMemcpy2DAsync(B.dc, (size_t)CH * 4, dcgm + off, (size_t)ld * 4,
                                        (size_t)m * 4, 8, cudaMemcpyHostToDevice, h2d));
        DSO_CUDA(ctx, cudaEventRecord(in_ready[s], h2d));
        DSO_CUDA(ctx, cudaStreamWaitEvent(c.stream, in_ready[s], 0));
        DSO_CUDA(ctx, launch_pipeline_csr(c, B.rp, B.ent, e0, B.dc, m, CH, (float)eta, K,
                                          params ? B.params : nullptr, clamped ? B.cl : nullptr,
                                          B.idx, cost ? B.cost : nullptr,
                                          energy ? B.energy : nullptr, time ? B.time : nullptr,
                                          CH));
        DSO_CUDA(ctx, cudaEventRecord(done[s], c.stream));
        DSO_CUDA(ctx, cudaStreamWaitEvent(d2h, done[s], 0));
        DSO_CUDA(ctx, cudaMemcpyAsync(idx + off, B.idx, 4 * m, cudaMemcpyDeviceToHost, d2h));
        if (cost)
            DSO_CUDA(ctx, cudaMemcpyAsync(cost + off, B.cost, 4 * m, cudaMemcpyDeviceToHost, d2h));
        if (energy)
            DSO_CUDA(ctx,
                     cudaMemcpyAsync(energy + off, B.energy, 4 * m, cudaMemcpyDeviceToHost, d2h));
        if (time)
            DSO_CUDA(ctx, cudaMemcpyAsync(time + off, B.time, 4 * m, cudaMemcpyDeviceToHost, d2h));
        if (params)
            DSO_CUDA(ctx, cudaMemcpy2DAsync(params + off, (size_t)ld * 4, B.params,
                                            (size_t)CH * 4, (size_t)m * 4, 7,
                                            cudaMemcpyDeviceToHost, d2h));
        if (clamped)
            DSO_CUDA(ctx, cudaMemcpyAsync(clamped + off, B.cl, m, cudaMemcpyDeviceToHost, d2h));
        DSO_CUDA(ctx, cudaEventRecord(drained[s], d2h));
    }
    DSO_CUDA(ctx, cudaStreamSynchronize(d2h));
    return kOk;
}

int32_t dso_train_grad(dso_ctx* ctx, const float* x, const float* y, int64_t n, int64_t ld,
                       float* grad, double* loss_sum) {
    int32_t st = check_ctx(ctx, false, true);
    if (st) return st;
    if ((st = check_batch(ctx, n, ld))) return st;
    if (!grad || !loss_sum) return fail(ctx, kInvalidArgument, "grad and loss_sum required");
    DSO_CUDA(ctx, launch_train_grad(ctx->c, x, y, n, ld, grad, loss_sum));
    return kOk;
}

int32_t dso_train_apply(dso_ctx* ctx, const float* grad, double lr, double scale) {
    int32_t st = check_ctx(ctx, false, true);
    if (st) return st;
    if (!grad) return fail(ctx, kInvalidArgument, "grad required");
    DSO_CUDA(ctx, launch_train_apply(ctx->c, grad, (float)(lr * scale)));
    return kOk;
}

}  // extern "C"
