// common.cuh — shared definitions for the sm_100a DSO kernels and the C-ABI.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <set>
#include <string>
#include <utility>

#include "../../include/dso_b200.h"

namespace dso_b200 {

// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) is per device: remember, per
// (kernel, device), that it has been applied. Thread-safe; contexts on several
// devices of one process each get the attribute on their own device.
inline cudaError_t ensure_smem_attr(const void* func, int device, int bytes) {
    static std::mutex mu;
    static std::set<std::pair<const void*, int>> done;
    std::lock_guard<std::mutex> lock(mu);
    if (done.count({func, device})) return cudaSuccess;
    cudaError_t e = cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes);
    if (e == cudaSuccess) done.insert({func, device});
    return e;
}

// 1 + dso::ErrorKind (reference proj/include/dso/error.hpp:10-25)
enum Status : int32_t {
    kOk = 0,
    kMalformedPtx = 1,
    kEmptyTrace = 2,
    kOutOfRange = 3,
    kSchemaMismatch = 4,
    kNonPositivePower = 5,
    kEtaOutOfRange = 6,
    kVoltageBelowKappa = 7,
    kFrequencyBelowKappa = 8,
    kRankDeficient = 9,
    kUnderdetermined = 10,
    kDatasetTooSmall = 11,
    kInvalidArgument = 12,
    kInvalidModel = 13,
    kIoError = 14,
    kCuda = DSO_ERR_CUDA,
};

constexpr int kMaxCore = 1024;  // core levels per domain (sweep tables live in smem)
constexpr int kMaxMem = 64;

// Per-domain tables, precomputed in double on the host (abi.cu) exactly as
// the reference computes them per evaluation (optimizer.cpp:36,
// dvfs_model.hpp:117-128), then stored in both precisions.
struct DomainDev {
    int nc, nm;
    // f32 path: per core level {vc, vc*vc*fc, 1/fc, fc}; per mem level {fm, 1/fm}
    float4* core4;   // [nc]
    float2* mem2;    // [nm]
    // f64 exact path: per core level {vc, fc}; per mem level fm
    double2* core_d;  // [nc]
    double* mem_d;    // [nm]
    // optimal_config: g1 = to_mhz(max_core_freq(vc)) per level and its
    // snap_down(cores, g1) index (optimizer.cpp:141-145), host double
    double* g1_d;     // [nc]
    int* sd_g1;       // [nc]
    // the f32 tables are within the bounds under which the fast exact sweep's
    // costs stay finite (sweep_core.cuh sweep_best)
    bool fast_ok;
    // vc and vc^2 fc non-decreasing and 1/fc non-increasing along the core
    // levels, fm non-decreasing and 1/fm non-increasing along the memory levels
    // (ascending frequency lists): the eta sweep's candidate pruning applies
    bool sorted_ok;
};

// Device model: transposed, zero-padded weights for the FP32 MLP kernels.
// Only the default topology 134-100-50-25-7 (mlp.cpp:177) runs on the fused
// kernels; other topologies are rejected by dso_set_model with InvalidModel
// for the device path (the reference trains probe nets only in unit tests).
constexpr int kGenMaxLayers = 8, kGenMaxWidth = 256, kGenMaxSumWidths = 700;

struct ModelDev {
    int sizes[kGenMaxLayers + 1];
    int n_layers = 5;  // entries of sizes (layers + 1)
    // any chain other than 134-100-50-25-7 runs on the generic engine (mlp_gen.cu)
    // from w_master; gstats = target mean[out] then std[out] (device)
    bool generic = false;
    float* gstats = nullptr;
    float* wt;       // packed per-layer transposed weights (see mlp.cu layout)
    float* bias;     // packed biases (padded)
    float mean[8], std_[8];
    int64_t wt_floats, bias_floats;
    // master copy in the reference layout (row-major W, concatenated), f32
    float* w_master;  // [n_weights + n_biases]
    int64_t w_master_cap = 0;
    // the training kernel's shared-memory image of the weights (train.cu), rebuilt
    // from w_master before the next gradient after any change of w_master
    float* w_train;
    bool train_dirty;
    // the tensor-core engine's packed model (mlp_tc.cuh): weights split hi/lo
    // for 3xTF32; tc_state 1 = finite (host-checked), 0 = non-finite, -1 =
    // repacked on the device (the kernels read the flag)
    float* wtc;
    int tc_state;
    // wt / wtc are rebuilt from w_master lazily: a training update only marks
    // them stale, the next inference launch repacks (launch_ws)
    bool infer_dirty = false;
    int64_t n_weights, n_biases;
};

// Layer chain of a generic model (mlp_gen.cu): offsets into the master layout.
struct GenNet {
    int layers;                     // weight layers
    int sizes[kGenMaxLayers + 1];
    int woff[kGenMaxLayers], boff[kGenMaxLayers];
    int aoff[kGenMaxLayers + 1];    // activation rows of layer l in the grad kernel
    int maxw, sum_widths;
    int64_t nw, nb;
};

struct Ctx {
    int device = 0;
    cudaStream_t own_stream = nullptr;
    cudaStream_t stream = nullptr;
    std::string last_error;
    int64_t launches = 0;
    bool has_domain = false;
    bool has_model = false;
    DomainDev dom{};
    double dom_core[kMaxCore];
    double dom_mem[kMaxMem];
    double dom_dev[5];
    ModelDev model{};
    // staging for DSO_HOST calls and scratch
    void* scratch = nullptr;
    size_t scratch_bytes = 0;
    cudaStream_t aux[3] = {nullptr, nullptr, nullptr};
    cudaEvent_t ev[8] = {};
    int num_sms = 148;
    bool fast_sweep = true;         // dso_set_option("fast_sweep")
    bool eta_prune = true;          // dso_set_option("eta_prune"): pruned eta sweep
    bool train_tc = true;           // dso_set_option("train_tc"): weight gradients on tcgen05
    int mlp_engine = 2;             // dso_set_option("mlp_engine"): 0 FMA pipe, 1 tensor cores,
                                    // 2 auto (tensor cores for predict / CSR, FMA pipe for dense)
    float2* eta_dev = nullptr;      // dso_eta_sweep's (eta, K) table
    int eta_cap = 0;
    int* flag_dev = nullptr;        // dso_dcgm_mean's out-of-range flag
    void* fit_plan = nullptr;       // dso_param_fit's factored designs (fit.cu)
    void* train_scratch = nullptr;  // per-CTA partial gradients
    size_t train_scratch_bytes = 0;
    // device evidence counters (dso_get_counters): work the kernels actually issued
    unsigned long long* counters_dev = nullptr;
    // dso_train_step / dso_fit_model (dp.cu): gradient and loss buffers
    float* dp_grad = nullptr;
    double* dp_dbl = nullptr;
    int64_t dp_np = 0;
    // the generic-chain pipeline's staging (mlp_gen.cu)
    void* gen_scratch = nullptr;
    size_t gen_scratch_bytes = 0;
    // dense counts -> CSR for the tensor-core pipeline (dense_csr.cu)
    bool dense_csr = true;          // dso_set_option("dense_csr")
    void* dcsr_scratch = nullptr;
    size_t dcsr_bytes = 0;
};

}  // namespace dso_b200

// The opaque handle of the C-ABI.
struct dso_ctx {
    dso_b200::Ctx c;
};

namespace dso_b200 {

// ---- launchers (defined in the kernel .cu files) ------------------------------
cudaError_t launch_sweep_f32(Ctx& c, const float* params, int64_t n, int64_t ld, float eta,
                             float K, int32_t* idx, float* cost, float* energy, float* time,
                             int32_t* kstatus);
cudaError_t launch_sweep_f64(Ctx& c, const double* params, int64_t n, double eta, double K,
                             int32_t* idx, double* cost, double* energy, double* time,
                             int32_t* kstatus);
cudaError_t launch_eta_sweep(Ctx& c, const float* params, int64_t n, int64_t ld,
                             const float2* etaK_dev, int n_eta, int32_t* idx, float* cost,
                             int64_t ld_out, bool fast, bool prune);
cudaError_t launch_optimal_config(Ctx& c, const double* params, int64_t n, double eta,
                                  double K, int32_t* idx, double* cost, double* energy,
                                  double* time, int64_t* candidates, uint8_t* fallback,
                                  double* presnap, int32_t* kstatus);
cudaError_t fit_prepare(Ctx& c, const double* cfg, int S);
void fit_plan_free(Ctx& c);
cudaError_t launch_param_fit(Ctx& c, const double* power, const double* time, int64_t n,
                             int64_t ld, double* pfit, int32_t* pstatus, double* tfit,
                             int32_t* tstatus);
cudaError_t launch_gen(Ctx& c, uint64_t root, uint64_t salt_base, int64_t first, int64_t n,
                       int64_t ld, float* params, uint32_t* counts, float* dcgm);
cudaError_t launch_featurize(Ctx& c, const uint32_t* counts, const float* dcgm, int64_t n,
                             int64_t ld, float* fused);
cudaError_t launch_dcgm_mean(Ctx& c, const double* samples, int64_t rows, int64_t n,
                             int64_t ld, float* out, int64_t* bad_row, int* any_bad_dev);
cudaError_t launch_predict(Ctx& c, const float* fused, int64_t n, int64_t ld, float* params,
                           uint8_t* clamped, float* raw);
cudaError_t launch_pipeline(Ctx& c, const uint32_t* counts, const float* dcgm, int64_t n,
                            int64_t ld, float eta, float K, float* params, uint8_t* clamped,
                            int32_t* idx, float* cost, float* energy, float* time,
                            int64_t ld_out);
cudaError_t launch_pipeline_csr(Ctx& c, const uint64_t* row_ptr, const uint32_t* entries,
                                uint64_t ent_base, const float* dcgm, int64_t n, int64_t ld,
                                float eta, float K, float* params, uint8_t* clamped, int32_t* idx,
                                float* cost, float* energy, float* time, int64_t ld_out);
cudaError_t launch_gen_csr(Ctx& c, uint64_t root, uint64_t salt_base, int64_t first, int64_t n,
                           uint64_t* row_ptr, uint32_t* entries, float* dcgm, int64_t ld);
cudaError_t model_upload(Ctx& c, const double* W, const double* b);
cudaError_t launch_train_grad(Ctx& c, const float* x, const float* y, int64_t n, int64_t ld,
                              float* grad, double* loss_sum_dev);
// repack = false leaves the inference kernels' packed weights stale (training
// loops repack once at the end, dp.cu)
cudaError_t launch_train_apply(Ctx& c, const float* grad, float lr_scale, bool repack = true);
// allocations (scratch, weight image) and kernel attributes for batches of up to
// n samples, without launching: makes the next gradients capturable
cudaError_t train_prepare(Ctx& c, int64_t n);
cudaError_t launch_repack(Ctx& c);
// true when the tensor-core engine would run the CSR pipeline for the context's
// model and domain (mlp.cu)
bool tc_csr_eligible(const Ctx& c);
// dso_pipeline on device buffers through the CSR form (dense_csr.cu): the dense
// counts are compacted to slot-sorted CSR rows on the device and the tensor-core
// CSR pipeline runs on them.  *done = false (nothing launched) when a count does
// not fit the CSR field (>= 2^25).
cudaError_t launch_pipeline_dense_via_csr(Ctx& c, const uint32_t* counts, const float* dcgm,
                                          int64_t n, int64_t ld, float eta, float K,
                                          float* params, uint8_t* clamped, int32_t* idx,
                                          float* cost, float* energy, float* time, bool* done);
// generic-chain engine and 64-bit-count features (mlp_gen.cu)
GenNet gen_net_of(const ModelDev& md);
cudaError_t launch_gen_forward(Ctx& c, const float* x, int64_t n, int64_t ld, float* raw,
                               float* params, uint8_t* clamped, int64_t ld_out);
cudaError_t launch_gen_grad(Ctx& c, const float* x, const float* y, int64_t n, int64_t ld,
                            float* grad, double* loss_sum_dev);
cudaError_t launch_gen_apply(Ctx& c, const float* grad, float lr_scale);
cudaError_t launch_featurize_u64(Ctx& c, const uint64_t* counts, const float* dcgm, int64_t n,
                                 int64_t ld, float* fused);
cudaError_t launch_csr_to_dense(Ctx& c, const uint64_t* row_ptr, const uint32_t* entries,
                                uint64_t ent_base, int64_t n, int64_t ld, uint32_t* counts);
cudaError_t launch_gen_pipeline(Ctx& c, const uint32_t* counts, const uint64_t* row_ptr,
                                const uint32_t* entries, uint64_t ent_base, const float* dcgm,
                                int64_t n, int64_t ld, float eta, float K, float* params,
                                uint8_t* clamped, int32_t* idx, float* cost, float* energy,
                                float* time, int64_t ld_out);  // w_master (f32, reference layout) -> packed wt
size_t mlp_smem_bytes();

// ---- device helpers ---------------------------------------------------------
// Packed FP32x2 FMA (Blackwell FFMA2): d = a * b + c lane-wise.  A scalar
// broadcast a is expressed as {a, a}; ptxas folds it to the .F32 operand form.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long A, B, Cc, D;
    A = *reinterpret_cast<unsigned long long*>(&a);
    B = *reinterpret_cast<unsigned long long*>(&b);
    Cc = *reinterpret_cast<unsigned long long*>(&c);
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(D) : "l"(A), "l"(B), "l"(Cc));
    return *reinterpret_cast<float2*>(&D);
}

// Packed FP32x2 add / mul (FADD2 / FMUL2): same IEEE round-to-nearest result as
// the scalar __fadd_rn / __fmul_rn on each lane.  Unlike the scalar forms they
// are contractable: ptxas fuses an fmul2 feeding an fadd2 into one FFMA2 (.rn
// is mandatory on f32x2, so it cannot mark the pair), so bit-exact paths never
// chain the two.
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
    unsigned long long A = *reinterpret_cast<unsigned long long*>(&a);
    unsigned long long B = *reinterpret_cast<unsigned long long*>(&b), D;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
    return *reinterpret_cast<float2*>(&D);
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
    unsigned long long A = *reinterpret_cast<unsigned long long*>(&a);
    unsigned long long B = *reinterpret_cast<unsigned long long*>(&b), D;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(D) : "l"(A), "l"(B));
    return *reinterpret_cast<float2*>(&D);
}

// FP32 pair evaluation shared by every sweep kernel (sweep, eta sweep, fused
// pipeline) so all of them round identically.  Explicit _rn intrinsics stop
// nvcc from re-contracting the expressions differently per kernel.
//   Pc = p0 + kp*vc + c*(vc^2 fc)         (per core level; t = {vc, vc^2 fc, 1/fc, fc})
//   P  = Pc + g*fm,  T = t0 + max(a/fm, b/fc),  C = (eta*P + (1-eta)*pmax) * T
__device__ __forceinline__ float pc_f32(float p0, float kp, float c, float4 t) {
    return fmaf(c, t.y, fmaf(kp, t.x, p0));
}
__device__ __forceinline__ float time_f32(float t0, float ta, float tb) {
    return __fadd_rn(t0, fmaxf(ta, tb));
}
__device__ __forceinline__ float cost_f32(float eta, float K, float P, float T) {
    return __fmul_rn(fmaf(eta, P, K), T);
}

// sigmoid (mlp.cpp:17-20) in FP32: 1 / (1 + 2^(-z log2 e)) with the
// approximate MUFU ex2/rcp (rel. error ~2^-22 each; no denormal fix-up code).
__device__ __forceinline__ float sigmoidf_fast(float z) {
    float e, r;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e) : "f"(z * -1.4426950408889634f));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(1.0f + e));
    return r;
}

// Fast-sweep precondition on the domain and the objective constant K = (1-eta)*pmax.
inline bool fast_sweep_ok(const Ctx& cx, float K) {
    return cx.fast_sweep && cx.dom.fast_ok && K == K && K <= 1e21f && K >= -1e21f;
}

// Two sigmoids of (acc + bias) with packed FP32x2 arithmetic around the MUFU
// ex2/rcp: nbl = -bias*log2(e) per neuron; 1/(1 + 2^(acc*(-log2 e) + nbl)).
__device__ __forceinline__ float2 sigmoid2_bias(float2 acc, float nbl) {
    constexpr float kNL2E = -1.4426950408889634f;
    const float2 z = ffma2(acc, make_float2(kNL2E, kNL2E), make_float2(nbl, nbl));
    float e0, e1, r0, r1;
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e0) : "f"(z.x));
    asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(e1) : "f"(z.y));
    const float2 d = fadd2(make_float2(1.f, 1.f), make_float2(e0, e1));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r0) : "f"(d.x));
    asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r1) : "f"(d.y));
    return make_float2(r0, r1);
}
__device__ __forceinline__ float neg_bias_log2e(float b) { return b * -1.4426950408889634f; }

inline int grid_for(int64_t n, int block, int num_sms, int per_sm) {
    int64_t blocks = (n + block - 1) / block;
    int64_t cap = (int64_t)num_sms * per_sm;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    return (int)blocks;
}

}  // namespace dso_b200
