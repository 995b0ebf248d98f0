/*
 * dso_oracle.h — CPU restatement of the DSO reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product (paper_2407_13096_b200/,
 * include/) links, loads or calls this code.  It is used by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg,
 * always as the checker, never as the thing measured or shipped.
 *
 * Every function restates a reference function in plain C, double precision,
 * in the same operation order; each definition in dso_oracle.c cites the
 * reference file:line it follows (paths relative to /root/reference/proj).
 *
 * Pinning (see DESIGN.md §3 and tests/test_oracle_*.py):
 *   - sweep / RNG / DVFS maths: checked against the reference itself
 *     (oracle/_ref/libdso_ref.so, built from proj/src/optimizer.cpp and the
 *     reference headers by oracle/Makefile);
 *   - MLP forward: proj/tests/fixtures/mlp_forward_golden.json (<= 4 ulp);
 *   - generator: acceptance KAT AC6 (24.1 % / 2.00 %, proj/test_output.txt:20);
 *   - gradients: central finite differences (proj/src/mlp.cpp:291-322).
 *
 * Layouts here are row-major per kernel ("AoS"): params [n][7],
 * counts [n][126], dcgm [n][8], fused [n][134].
 *
 * Status codes: 0 = ok, otherwise 1 + dso::ErrorKind (proj/include/dso/error.hpp:10-25).
 */
#ifndef DSO_ORACLE_H
#define DSO_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
    ORC_OK = 0,
    ORC_MalformedPtx = 1,
    ORC_EmptyTrace = 2,
    ORC_OutOfRange = 3,
    ORC_SchemaMismatch = 4,
    ORC_NonPositivePower = 5,
    ORC_EtaOutOfRange = 6,
    ORC_VoltageBelowKappa = 7,
    ORC_FrequencyBelowKappa = 8,
    ORC_RankDeficient = 9,
    ORC_Underdetermined = 10,
    ORC_DatasetTooSmall = 11,
    ORC_InvalidArgument = 12,
    ORC_InvalidModel = 13,
    ORC_IoError = 14,
};

/* ---- RNG (rng.hpp:11-64) ------------------------------------------------ */
uint64_t orc_rng_next(uint64_t* state);
double orc_rng_uniform01(uint64_t* state);
double orc_rng_uniform(uint64_t* state, double lo, double hi);
uint64_t orc_rng_below(uint64_t* state, uint64_t n);
uint64_t orc_rng_fork(const uint64_t* state, uint64_t salt); /* returns child state */
void orc_shuffled_indices(uint64_t n, uint64_t* state, uint64_t* out);

/* ---- DVFS model (dvfs_model.hpp:72-128) ---------------------------------- */
double orc_power(const double* p, double vc, double fc, double fm);
double orc_exec_time(const double* p, double vc, double fc, double fm);
double orc_required_voltage_mhz(double fc_mhz, const double* dev);
int orc_validate_params(const double* p);
int orc_validate_domain(const double* core, int nc, const double* mem, int nm,
                        const double* dev);

/* ---- generator (sim_harness.cpp:17-144) ---------------------------------- */
/* Kernel i of the synthetic stream: seed_i = Rng(root).fork(first+i).next_u64(),
 * as run_campaign does (sim_harness.cpp:241-242).  Any output may be NULL. */
void orc_gen_stream(uint64_t root, uint64_t salt_base, int64_t first, int64_t n,
                    double* params, uint32_t* counts, double* dcgm, double* fused,
                    int threads);
/* gen_kernel(seed) for explicit seeds. */
void orc_gen_seeded(const uint64_t* seeds, int64_t n, double* params, uint32_t* counts,
                    double* dcgm, double* fused);
/* gen_kernel(seed, rho) */
int orc_gen_kernel_rho(uint64_t seed, double rho, double* params, uint32_t* counts,
                       double* dcgm, double* fused);

/* ---- features (ptx_features.cpp:311-329, telemetry.cpp:63-101, mlp.cpp:158-165) */
void orc_featurize(const uint32_t* counts, int64_t n, double* out126);
/* samples [rows][8]; returns status, *bad_row = 1-based offending row */
int orc_dcgm_mean(const double* samples, int64_t rows, double* out, int64_t* bad_row);
void orc_fuse(const uint32_t* counts, const double* dcgm, int64_t n, double* fused);

/* ---- MLP (mlp.cpp:17-253) ----------------------------------------------- */
/* Model: nl = number of layer sizes; weights concatenated row-major per layer
 * (shape sizes[l+1] x sizes[l]); biases concatenated; mean/std size sizes[nl-1]. */
int64_t orc_mlp_weight_count(const int* sizes, int nl);
int64_t orc_mlp_bias_count(const int* sizes, int nl);
int orc_init_mlp(const int* sizes, int nl, uint64_t seed, double* W, double* b);
void orc_forward_raw(const int* sizes, int nl, const double* W, const double* b,
                     const double* mean, const double* std, const double* x, int64_t n,
                     double* out);
void orc_predict_params(const int* sizes, int nl, const double* W, const double* b,
                        const double* mean, const double* std, const double* x, int64_t n,
                        double* params, uint8_t* clamped, int threads);

/* ---- training (mlp.cpp:35-130, 259-346) ---------------------------------- */
/* x [B][in], y_std [B][out]; gW/gb same layout as W/b */
double orc_mse_loss(const int* sizes, int nl, const double* W, const double* b,
                    const double* x, const double* y, int64_t B);
void orc_analytic_gradients(const int* sizes, int nl, const double* W, const double* b,
                            const double* x, const double* y, int64_t B, double* gW,
                            double* gb);
void orc_numeric_gradients(const int* sizes, int nl, const double* W, const double* b,
                           const double* x, const double* y, int64_t B, double eps,
                           double* gW, double* gb);
/* One SGD epoch over examples (features [n][in], targets [n][out], raw units)
 * with stats mean/std, order from shuffled_indices(n, rng).  Updates W/b in place;
 * returns mean batch loss (NaN if non-finite). */
double orc_sgd_epoch(const int* sizes, int nl, double* W, double* b, const double* feats,
                     const double* targets, int64_t n, const double* mean,
                     const double* std, double lr, int batch, uint64_t* rng_state);
/* target_stats (mlp.cpp:57-79): returns number of degenerate dims */
int orc_target_stats(const double* targets, int64_t n, int out, double* mean, double* std);

/* ---- sweep (optimizer.cpp:18-117) ---------------------------------------- */
/* brute_force_config over n kernels; idx = fc_idx*nm + fm_idx; status per kernel */
int orc_brute_force(const double* params, int64_t n, const double* core, int nc,
                    const double* mem, int nm, const double* dev, double eta,
                    double pmax, int32_t* idx, double* cost, double* energy, double* time,
                    int32_t* kstatus, int threads);
/* eta sweep: out idx/cost [n_eta][n] */
int orc_eta_sweep(const double* params, int64_t n, const double* core, int nc,
                  const double* mem, int nm, const double* dev, const double* etas,
                  int n_eta, double pmax, int32_t* idx, double* cost, int threads);

/* ---- pipeline: counts+dcgm -> featurize -> predict -> brute force ---------- */
int orc_pipeline(const uint32_t* counts, const double* dcgm, int64_t n, const int* sizes,
                 int nl, const double* W, const double* b, const double* mean,
                 const double* std, const double* core, int nc, const double* mem, int nm,
                 const double* dev, double eta, double pmax, double* params_out,
                 uint8_t* clamped, int32_t* idx, double* cost, double* energy, double* time,
                 int threads);

/* ---- param_fit (param_fit.cpp:43-247): cfg [S][3] = vc, fc_mhz, fm_mhz ---- */
int orc_fit_power(const double* cfg, const double* power, int S, double* out /* [6] */);
int orc_fit_time(const double* cfg, const double* time_s, int S, double* out /* [8] */,
                 uint8_t* branch_out /* [S] or NULL */);

#ifdef __cplusplus
}
#endif
#endif
