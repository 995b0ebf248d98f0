/*
 * dso_b200.h — C-ABI of the B200-native DSO hot path (libdso_b200.so).
 *
 * The reference (arxiv 2407.13096, /root/reference/proj) has no FFI: its
 * interface is the C++ API in proj/include/dso/.  Each entry point below
 * replaces one reference function for a whole batch of GPU kernels; the
 * replaced interface is cited as  <file>:<line>  (relative to proj/).  The C++
 * drop-in wrappers with the reference's own signatures and dso::Error
 * behaviour are in include/dso/batch.hpp; INTEGRATION.md shows the bindings.
 *
 * Conventions
 *   - Plain pointers and sizes only.  Every call returns int32 status:
 *       0                      ok
 *       1 + dso::ErrorKind     the reference's error kinds (error.hpp:10-25),
 *                              e.g. 12 = InvalidArgument, 6 = EtaOutOfRange
 *       DSO_ERR_CUDA (100)     CUDA runtime failure (mapped to IoError in C++)
 *     dso_last_error(ctx) returns the message of the last failure on ctx.
 *   - Device arrays are structure-of-arrays with a leading dimension ld >= n:
 *     element (row r, kernel k) lives at base[r*ld + k].  A shard [a, b) of a
 *     larger batch is passed as base + a with the batch's ld — no copy.
 *       params  float [7][ld]   p0, kappa_pow, gamma, c, t0, alpha, beta
 *                               (KernelModelParams field order, dvfs_model.hpp:23-31)
 *       counts  uint32 [126][ld] instr 0..100 | dtype 101..117 | memspace 118..125
 *                               (category order ptx_features.cpp:18-49)
 *       dcgm    float [8][ld]   smact smocc tenso drama fp64a fp32a fp16a intac
 *                               (telemetry.hpp:13-28)
 *       fused   float [134][ld] FusedFeatures::as_vector order (mlp.cpp:158-165)
 *     idx = fc_idx * nm + fm_idx (brute_force loop order, optimizer.cpp:99-100).
 *   - All launches are asynchronous on the context stream; dso_sync() waits.
 *     Pass DSO_HOST in flags (where offered) for host buffers: the call then
 *     stages the batch through the device in overlapped chunks and returns
 *     after the results are back in host memory.
 *   - One host thread per context at a time (the reference is re-entrant and
 *     stateless; a context is the per-device state it lacks).
 */
#ifndef DSO_B200_H
#define DSO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DSO_OK 0
#define DSO_ERR_CUDA 100

#define DSO_HOST 1u          /* pointers are host memory (pinned for full speed) */

#define DSO_INSTR_SLOTS 101  /* ptx_features.hpp:21 */
#define DSO_DTYPE_SLOTS 17   /* ptx_features.hpp:22 */
#define DSO_MEMSPACE_SLOTS 8 /* ptx_features.hpp:23 */
#define DSO_COUNT_ROWS 126
#define DSO_FUSED_ROWS 134   /* kFusedFeatureCount, mlp.hpp:15 */
#define DSO_PARAM_ROWS 7     /* kParamCount, mlp.hpp:16 */

typedef struct dso_ctx dso_ctx;

/* ---- context ------------------------------------------------------------- */
int32_t dso_ctx_create(int32_t device, dso_ctx** out);
int32_t dso_ctx_destroy(dso_ctx* ctx);
/* Launch on an external cudaStream_t (e.g. torch's current stream).  NULL is
 * the legacy default stream (torch's default stream); a context starts on its
 * own non-blocking stream. */
int32_t dso_ctx_set_stream(dso_ctx* ctx, void* cuda_stream);
int32_t dso_sync(dso_ctx* ctx);
const char* dso_last_error(const dso_ctx* ctx);
/* Name of the dso::ErrorKind a status maps to ("InvalidArgument", ...). */
const char* dso_status_name(int32_t status);
/* Number of device kernel launches issued on ctx so far (evidence counter). */
int64_t dso_launch_count(const dso_ctx* ctx);

/* Device evidence counters: the work the kernels actually issued (accumulated
 * per context; the call synchronises the context stream).  Indices:
 *   DSO_CTR_TC_L1_KSTEPS  tcgen05 layer-1 k-steps (3 kind::tf32 MMAs of
 *                         M128 x N112 x K8 each; CSR tiles skip all-zero chunks)
 *   DSO_CTR_TC_L2_KSTEPS  tcgen05 layer-2 k-steps (3 MMAs of M128 x N64 x K8)
 *   DSO_CTR_TC_TILES      128-kernel tiles processed by the tcgen05 engine
 * reset != 0 zeroes them after the read.  Not a reference interface (bench
 * evidence for roofline.achieved). */
#define DSO_CTR_TC_L1_KSTEPS 0
#define DSO_CTR_TC_L2_KSTEPS 1
#define DSO_CTR_TC_TILES 2
#define DSO_N_COUNTERS 8
int32_t dso_get_counters(dso_ctx* ctx, uint64_t* out, int32_t n, int32_t reset);
/* Tuning / verification switches (no reference counterpart; results never
 * depend on them).  key "fast_sweep": 1 (default) lets the FP32 sweeps use the
 * group-minimum argmin (bit-identical, see sweep_core.cuh), 0 forces the
 * pair-by-pair lexicographic scan.  key "eta_prune": 1 (default) lets
 * dso_eta_sweep on an ascending-frequency domain with 2-4 memory levels sweep
 * only the nc + nm candidate pairs no other pair can beat (bit-identical, see
 * sweep.cu), 0 sweeps all pairs.  key "dense_csr": 1 (default) lets
 * dso_pipeline on device buffers with the auto engine compact the dense counts
 * to CSR on the device and run the tensor-core CSR pipeline (one host sync per
 * call), 0 keeps the FMA-pipe dense kernel.  key "train_tc": 1 (default) computes the
 * training weight gradients on the tensor cores (3xTF32, tcgen05), 0 on the
 * FMA pipe.  key "mlp_engine": the predictor engine of
 * dso_predict / dso_pipeline / dso_pipeline_csr: 0 = FP32 FMA-pipe kernel,
 * 1 = tcgen05 3xTF32 tensor-core kernel, 2 = auto (default: tensor cores for
 * predict and CSR input, FMA pipe for dense counts).  Unknown key or value ->
 * InvalidArgument. */
int32_t dso_set_option(dso_ctx* ctx, const char* key, int64_t value);

/* ---- domain: replaces the DvfsDomain argument + validate(DvfsDomain) ------
 * optimizer.hpp:14-20, optimizer.cpp:58-88, dvfs_model.hpp:60-70.
 * dev = [kappa_vf, pmax_w, vmin_v, vmax_v, mhz_per_unit] (dvfs_model.hpp:36-42).
 * Validates exactly like the reference (same kinds), then uploads the
 * per-level tables (vc, vc^2*fc, 1/fc; fm, 1/fm) computed in double. */
int32_t dso_set_domain(dso_ctx* ctx, const double* core_mhz, int32_t nc,
                       const double* mem_mhz, int32_t nm, const double* dev);
/* validate(DvfsDomain) alone (host only, no device needed); the message of a
 * failure is copied into msg (NUL-terminated, at most msg_len bytes). */
int32_t dso_validate_domain(const double* core_mhz, int32_t nc, const double* mem_mhz,
                            int32_t nm, const double* dev, char* msg, int32_t msg_len);

/* ---- model: replaces the MlpModel argument + validate(MlpModel) -----------
 * mlp.hpp:35-42, mlp.cpp:209-226.  weights: per layer l, sizes[l+1] x sizes[l]
 * row-major, concatenated (model.schema.json order, json_io.cpp:154-160);
 * biases concatenated; mean/std of size sizes[n_sizes-1], std > 0. */
int32_t dso_set_model(dso_ctx* ctx, const int32_t* layer_sizes, int32_t n_sizes,
                      const double* weights, const double* biases,
                      const double* target_mean, const double* target_std);
/* Read back the device model (after training) in the same layout. */
int32_t dso_get_model(dso_ctx* ctx, double* weights, double* biases);

/* ---- host helpers (host C++ inside the library, no device work) ----------- */
/* init_mlp (mlp.cpp:184-207): Glorot-uniform from Rng(seed), zero biases. */
int32_t dso_init_mlp(const int32_t* layer_sizes, int32_t n_sizes, uint64_t seed,
                     double* weights, double* biases);
/* shuffled_indices (rng.hpp:58-64) from Rng(seed) state; advances *state. */
int32_t dso_shuffled_indices(uint64_t n, uint64_t* rng_state, uint64_t* out);

/* ---- feature stage ---------------------------------------------------------
 * featurize (ptx_features.cpp:311-329) + FusedFeatures::as_vector
 * (mlp.cpp:158-165): per category count/total (all-zero for a zero total),
 * fused with the already-averaged DCGM vector.  Results equal the reference's
 * double features rounded once to float. */
int32_t dso_featurize(dso_ctx* ctx, const uint32_t* counts, const float* dcgm, int64_t n,
                      int64_t ld, float* fused);

/* load_dcgm_samples mean (telemetry.cpp:73-89) over parsed rows:
 * samples double [rows][8][ld] -> out float [8][ld].  bad_row[k] = first
 * 1-based row with a value outside [0,1] (0 if none); status OutOfRange if any. */
/* featurize + as_vector on the reference's 64-bit counts (KernelInstructionCounts
 * maps are std::uint64_t, ptx_features.hpp:31-37): counts uint64 [126][ld], dcgm
 * float [8][ld] -> fused float [134][ld].  Exact integer category totals, one
 * FP64 division per count (the reference's double quotient), rounded once to
 * float; equal to the reference for totals < 2^53. */
int32_t dso_featurize_u64(dso_ctx* ctx, const uint64_t* counts, const float* dcgm, int64_t n,
                          int64_t ld, float* fused);

int32_t dso_dcgm_mean(dso_ctx* ctx, const double* samples, int64_t rows, int64_t n,
                      int64_t ld, float* out, int64_t* bad_row);

/* ---- predictor inference ---------------------------------------------------
 * predict_params (mlp.cpp:237-253) = forward_raw (mlp.cpp:232-235) + clamp:
 * negative outputs -> 0, alpha+beta <= 0 -> beta = 1e-12; clamped[k] flags it.
 * raw (optional, float [7][ld]) receives forward_raw before clamping. */
int32_t dso_predict(dso_ctx* ctx, const float* fused, int64_t n, int64_t ld, float* params,
                    uint8_t* clamped, float* raw);

/* ---- grid sweep + eta objective + argmin ------------------------------------
 * brute_force_config (optimizer.cpp:90-117) for n kernels at one eta.
 * FP32 evaluation with tables precomputed in double; outputs at the chosen
 * pair.  kstatus[k] = 0 or 1+InvalidArgument (validate(params),
 * dvfs_model.hpp:50-58) with idx -1 and NaN outputs.  Returns EtaOutOfRange
 * for eta outside [0,1] (dvfs_model.hpp:101-102). */
int32_t dso_sweep(dso_ctx* ctx, const float* params, int64_t n, int64_t ld, double eta,
                  double pmax_w, int32_t* idx, float* cost, float* energy, float* time,
                  int32_t* kstatus);

/* Bit-exact variant on the reference's own layout: params is
 * KernelModelParams[n] (7 doubles each, dvfs_model.hpp:23-31); evaluation in
 * FP64 in the reference's operation order, so idx/cost/energy/time equal
 * brute_force_config's exactly. */
int32_t dso_sweep_f64(dso_ctx* ctx, const double* params_aos, int64_t n, double eta,
                      double pmax_w, int32_t* idx, double* cost, double* energy,
                      double* time, int32_t* kstatus, uint32_t flags);

/* optimal_config (optimizer.cpp:119-205, optimizer.hpp:39-46): the structured
 * Theorem-1 search, FP64, bit-identical to the reference per kernel.  params
 * AoS [n][7] double like dso_sweep_f64.  Outputs per kernel: idx (fc_idx*nm +
 * fm_idx), cost, energy, time, candidates (candidates_evaluated), fallback
 * (0/1), presnap [n][3] = {presnap_vc, presnap_fc_mhz, presnap_fm_mhz}, kstatus.
 * Every output but idx may be NULL.  flags: DSO_HOST for host buffers. */
int32_t dso_optimal_config(dso_ctx* ctx, const double* params_aos, int64_t n, double eta,
                           double pmax_w, int32_t* idx, double* cost, double* energy,
                           double* time, int64_t* candidates, uint8_t* fallback,
                           double* presnap, int32_t* kstatus, uint32_t flags);

/* param_fit for a batch of kernels measured on one configuration grid:
 * fit_power (param_fit.cpp:43-77) and fit_time (param_fit.cpp:79-247), the
 * regressions run_campaign applies to every measurement sweep
 * (sim_harness.cpp:269-270).  cfg [S][3] host = {vc, fc_mhz, fm_mhz} per sample
 * (shared by all kernels); power / time [S][ld] (either may be NULL to skip that
 * fit).  Outputs [rows][ld]:
 *   pfit [6]: p0, kappa_pow, gamma, c, mape_pct, constraint_active
 *   tfit [8]: t0, alpha, beta, mape_pct, constraint_active,
 *             partial_identifiability, iterations, final rss
 * and per-kernel status (0, or 1 + ErrorKind: RankDeficient / InvalidArgument /
 * Underdetermined as the reference throws).  FP64; coefficients equal the
 * reference's to rounding (the QR solve operator is applied as a matrix).
 * flags: DSO_HOST for host power/time/outputs. */
int32_t dso_param_fit(dso_ctx* ctx, const double* cfg, int32_t S, const double* power,
                      const double* time, int64_t n, int64_t ld, double* pfit,
                      int32_t* pstatus, double* tfit, int32_t* tstatus, uint32_t flags);

/* eta sweep: brute_force_config at n_eta etas in one pass over the grid.
 * idx/cost are [n_eta][ld_out]. */
int32_t dso_eta_sweep(dso_ctx* ctx, const float* params, int64_t n, int64_t ld,
                      const double* etas, int32_t n_eta, double pmax_w, int32_t* idx,
                      float* cost, int64_t ld_out);

/* ---- fused pipeline: counts + DCGM -> features -> MLP -> sweep -> argmin ----
 * One persistent kernel; nothing intermediate touches HBM.  params/clamped
 * optional (NULL).  flags: DSO_HOST for host buffers (chunked, overlapped
 * H2D / compute / D2H). */
int32_t dso_pipeline(dso_ctx* ctx, const uint32_t* counts, const float* dcgm, int64_t n,
                     int64_t ld, double eta, double pmax_w, float* params, uint8_t* clamped,
                     int32_t* idx, float* cost, float* energy, float* time, uint32_t flags);

/* Same pipeline on SPARSE counts — the reference's own shape, one map of
 * non-zero category counts per kernel (KernelInstructionCounts,
 * ptx_features.hpp:31-37).  Kernel k's entries are
 * entries[row_ptr[k] - ent_base .. row_ptr[k+1] - ent_base), each
 * (count << 7) | slot with slot the count-row index (< 126, see counts above)
 * and count < 2^25; slots listed twice are added.  dcgm is [8][ld].  With
 * DSO_HOST, row_ptr/entries/dcgm/outputs are host memory (row_ptr[0..n]). */
int32_t dso_pipeline_csr(dso_ctx* ctx, const uint64_t* row_ptr, const uint32_t* entries,
                         uint64_t ent_base, const float* dcgm, int64_t n, int64_t ld,
                         double eta, double pmax_w, float* params, uint8_t* clamped,
                         int32_t* idx, float* cost, float* energy, float* time, uint32_t flags);

/* ---- synthetic inputs (sim_harness.cpp:118-144 gen_kernel, on device) -------
 * Kernel k (0 <= k < n) is gen_kernel(Rng(root).fork(salt_base+first+k)
 * .next_u64()), as run_campaign seeds its corpus (sim_harness.cpp:241-242).
 * Outputs optional: truth params (float [7][ld]), raw PTX counts, DCGM vector.
 * Bit-identical to the host generator (counts exact, params/dcgm = double
 * values rounded once to float). */
int32_t dso_gen_synthetic(dso_ctx* ctx, uint64_t root, uint64_t salt_base, int64_t first,
                          int64_t n, int64_t ld, float* params, uint32_t* counts,
                          float* dcgm);

/* The synthetic stream in the sparse format: 24 entries per kernel (the slots
 * features_from fills), row_ptr[k] = 24k for k <= n, dcgm [8][ld]. */
int32_t dso_gen_synthetic_csr(dso_ctx* ctx, uint64_t root, uint64_t salt_base, int64_t first,
                              int64_t n, uint64_t* row_ptr, uint32_t* entries, float* dcgm,
                              int64_t ld);

/* ---- predictor training (data-parallel) ------------------------------------
 * Mini-batch gradient of mse_loss (mlp.cpp:259-289) on the device model.
 * x float [in][ld] (fused features), y_std float [out][ld] (standardized
 * targets).  grad (device, weights then biases, same layout as dso_set_model)
 * receives the SUM over the batch of per-sample gradients of
 * 0.5*||out-y||^2 (i.e. analytic_gradients times B*out); loss_sum receives
 * sum ||out-y||^2 * 0.5.  Scaling by 1/(B_global*out) happens in apply, so a
 * data-parallel step is: grad -> allreduce(sum) -> apply. */
int32_t dso_train_grad(dso_ctx* ctx, const float* x, const float* y_std, int64_t n,
                       int64_t ld, float* grad, double* loss_sum);
/* W -= lr * scale * grad  (sgd update, mlp.cpp:105-108). */
int32_t dso_train_apply(dso_ctx* ctx, const float* grad, double lr, double scale);

/* One synchronous data-parallel SGD step inside the library (SURVEY.md §8(b),
 * §8(e)): the batch-sum gradient of this rank's n samples -> ncclAllReduce(sum)
 * of the gradient and the loss over `nccl_comm` (an ncclComm_t; NULL = one
 * process) -> W -= lr / (global_batch * out) * g on every rank (mse_loss's
 * 1/(B*out), mlp.cpp:259-289; update mlp.cpp:105-108).  loss (host, optional:
 * NULL keeps the call asynchronous) receives mse_loss of the global batch on
 * the pre-update weights. */
int32_t dso_train_step(dso_ctx* ctx, const float* x, const float* y_std, int64_t n, int64_t ld,
                       double lr, int64_t global_batch, void* nccl_comm, double* loss);

/* fit_model's epoch loop (mlp.cpp:84-130) on the device model set with
 * dso_set_model (the caller does init_mlp + target stats, as fit_model does):
 * per epoch the order shuffled_indices(Rng(seed).fork(0x5d0)) (rng.hpp:58-64,
 * mlp.cpp:87,123), contiguous batches of `batch` (last one partial), each
 * batch's mse_loss on the pre-update weights, W -= lr * g; epoch_loss[e]
 * (host, optional, >= epochs entries) = the mean batch loss; stops after a
 * NaN epoch (mlp.cpp:126), *epochs_run = epochs completed.  x [in][ld],
 * y_std [out][ld] device, the WHOLE dataset on every rank; with nranks > 1 each
 * rank takes the contiguous share [b*rank/nranks, b*(rank+1)/nranks) of every
 * batch and the gradients are summed over nccl_comm, so replicas stay
 * identical and equal the single-device run up to FP32 summation order.
 * Single-process epochs run as one CUDA graph replay each. */
int32_t dso_fit_model(dso_ctx* ctx, const float* x, const float* y_std, int64_t n, int64_t ld,
                      double lr, int32_t batch, int32_t epochs, uint64_t seed, void* nccl_comm,
                      int32_t rank, int32_t nranks, double* epoch_loss, int32_t* epochs_run);

/* NCCL, reached through dlopen (the copy already loaded in the process if any):
 * a unique id (DSO_NCCL_ID_BYTES bytes, broadcast by the host over any channel),
 * a communicator for (nranks, rank) on `device`, its destruction, the version.
 * IoError when no libnccl.so.2 is available. */
#define DSO_NCCL_ID_BYTES 128
int32_t dso_nccl_unique_id(uint8_t* id);
int32_t dso_nccl_comm_init(int32_t nranks, const uint8_t* id, int32_t rank, int32_t device,
                           void** comm);
int32_t dso_nccl_comm_destroy(void* comm);
int32_t dso_nccl_version(int32_t* version);
/* Number of parameters (weights + biases) of the device model. */
int64_t dso_model_param_count(const dso_ctx* ctx);

/* ---- diagnostics --------------------------------------------------------------
 * Measured FP32 FMA-pipe peak of this device (the roofline denominator of the
 * FP32-bound kernels): mode 0 = scalar FFMA, 1 = packed FFMA2.  TFLOP/s. */
int32_t dso_probe_fp32_peak(dso_ctx* ctx, int32_t mode, double* tflops);

/* ---- host feature ingestion (no device; thread-safe) ----------------------
 * parse_ptx (ptx_features.cpp:238-309): PTX text -> per-kernel category counts
 * in source order, rows = instr 0..100 | dtype 101..117 | memspace 118..125.
 * Fails with MalformedPtx (status 1) and a line number in msg on an
 * unterminated block comment or kernel body. */
typedef struct dso_ptx dso_ptx;
int32_t dso_ptx_parse(const char* text, int64_t len, dso_ptx** out, char* msg, int32_t msg_len);
void dso_ptx_free(dso_ptx* parsed);
int64_t dso_ptx_kernel_count(const dso_ptx* parsed);
const char* dso_ptx_kernel_name(const dso_ptx* parsed, int64_t k);
/* counts126 = kernel k's raw tallies (KernelInstructionCounts maps, ptx_features.hpp:31-37) */
int32_t dso_ptx_kernel_counts(const dso_ptx* parsed, int64_t k, uint64_t* counts126,
                              uint64_t* total_instructions);
/* dense uint32 [126][ld] counts for dso_featurize / dso_pipeline */
int32_t dso_ptx_counts(const dso_ptx* parsed, uint32_t* counts, int64_t ld);
/* CSR for dso_pipeline_csr: row_ptr [n+1], entries [nnz] = (count << 7) | row
 * (InvalidArgument if a count >= 2^25) */
int64_t dso_ptx_nnz(const dso_ptx* parsed);
int32_t dso_ptx_csr(const dso_ptx* parsed, uint64_t* row_ptr, uint32_t* entries);
/* Canonical category name of count row r (ptx_features.cpp:18-49 lists; the last
 * entry of each category is "other"), NULL outside 0..125. */
const char* dso_category_name(int32_t row);
/* load_dcgm_samples (telemetry.cpp:63-101): header, >= 1 row, 9 fields, values in
 * [0, 1] (OutOfRange with the row in msg), per-metric mean in double ->
 * mean8 in DcgmMetricVector order. */
int32_t dso_load_dcgm_csv(const char* text, int64_t len, double* mean8, char* msg,
                          int32_t msg_len);

#ifdef __cplusplus
}
#endif
#endif /* DSO_B200_H */
