/*
 * dso_oracle.c — CPU restatement of the DSO reference hot path (double precision).
 *
 * TEST INFRASTRUCTURE ONLY — see dso_oracle.h.  Never linked into the product.
 * Compiled with -ffp-contract=off so no a*b+c is fused: the reference build
 * (proj/src/CMakeLists.txt:13, plain -O2 on x86-64) never emits FMA, and the
 * restatement must round exactly like it.
 *
 * Reference paths below are relative to /root/reference/proj.
 */
#include "dso_oracle.h"

#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>

/* ====================================================================== */
/* RNG: include/dso/rng.hpp:11-64                                          */
/* ====================================================================== */

/* rng.hpp:18-23 splitmix64 */
uint64_t orc_rng_next(uint64_t* s) {
    uint64_t z = (*s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

/* rng.hpp:26 */
double orc_rng_uniform01(uint64_t* s) { return (double)(orc_rng_next(s) >> 11) * 0x1.0p-53; }

/* rng.hpp:29 */
double orc_rng_uniform(uint64_t* s, double lo, double hi) {
    return lo + (hi - lo) * orc_rng_uniform01(s);
}

/* rng.hpp:33-46 Lemire */
uint64_t orc_rng_below(uint64_t* s, uint64_t n) {
    uint64_t x = orc_rng_next(s);
    __uint128_t m = (__uint128_t)x * n;
    uint64_t l = (uint64_t)m;
    if (l < n) {
        uint64_t t = (0ULL - n) % n;
        while (l < t) {
            x = orc_rng_next(s);
            m = (__uint128_t)x * n;
            l = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}

/* rng.hpp:50-54 fork */
uint64_t orc_rng_fork(const uint64_t* s, uint64_t salt) {
    uint64_t child = *s ^ (0xd1342543de82ef95ULL * (salt + 1));
    orc_rng_next(&child);
    return child;
}

/* rng.hpp:58-64 Fisher-Yates */
void orc_shuffled_indices(uint64_t n, uint64_t* s, uint64_t* idx) {
    for (uint64_t i = 0; i < n; ++i) idx[i] = i;
    for (uint64_t i = n; i > 1; --i) {
        uint64_t j = orc_rng_below(s, i);
        uint64_t t = idx[i - 1];
        idx[i - 1] = idx[j];
        idx[j] = t;
    }
}

/* ====================================================================== */
/* DVFS model: include/dso/dvfs_model.hpp:50-128                           */
/* params order [p0, kappa_pow, gamma, c, t0, alpha, beta] (mlp.hpp:27-30)  */
/* dev order    [kappa_vf, pmax_w, vmin_v, vmax_v, mhz_per_unit] (:36-42)   */
/* ====================================================================== */

/* dvfs_model.hpp:81-84 */
double orc_power(const double* p, double vc, double fc, double fm) {
    return p[0] + p[1] * vc + p[2] * fm + p[3] * vc * vc * fc;
}

/* dvfs_model.hpp:88-90; std::max(a, b) == (a < b) ? b : a */
double orc_exec_time(const double* p, double vc, double fc, double fm) {
    (void)vc;
    double a = p[5] / fm, b = p[6] / fc;
    return p[4] + ((a < b) ? b : a);
}

/* dvfs_model.hpp:117-128 (caller guarantees fc/mpu >= kappa_vf) */
double orc_required_voltage_mhz(double fc_mhz, const double* dev) {
    double norm = fc_mhz / dev[4];
    double d = norm - dev[0];
    return 2.0 * d * d + dev[0];
}

/* dvfs_model.hpp:50-58 */
int orc_validate_params(const double* p) {
    if (p[0] < 0.0 || p[1] < 0.0 || p[2] < 0.0 || p[3] < 0.0 || p[4] < 0.0 || p[5] < 0.0 ||
        p[6] < 0.0)
        return ORC_InvalidArgument;
    if (!(p[5] + p[6] > 0.0)) return ORC_InvalidArgument;
    return ORC_OK;
}

/* dvfs_model.hpp:60-70 + optimizer.cpp:58-88 */
int orc_validate_domain(const double* core, int nc, const double* mem, int nm,
                        const double* dev) {
    if (!(dev[2] > 0.0) || !(dev[2] <= dev[3])) return ORC_InvalidArgument;
    if (!(dev[1] > 0.0)) return ORC_InvalidArgument;
    if (!(dev[0] < dev[2])) return ORC_InvalidArgument;
    if (!(dev[4] > 0.0)) return ORC_InvalidArgument;
    const double* tabs[2] = {core, mem};
    int lens[2] = {nc, nm};
    for (int t = 0; t < 2; ++t) {
        if (lens[t] <= 0) return ORC_InvalidArgument;
        double prev = 0.0;
        for (int i = 0; i < lens[t]; ++i) {
            if (!(tabs[t][i] > prev)) return ORC_InvalidArgument;
            prev = tabs[t][i];
        }
    }
    for (int i = 0; i < nc; ++i) {
        double norm = core[i] / dev[4];
        if (norm < dev[0]) return ORC_FrequencyBelowKappa;
        double d = norm - dev[0];
        double vc = 2.0 * d * d + dev[0];
        if (vc < dev[2] || vc > dev[3]) return ORC_OutOfRange;
    }
    return ORC_OK;
}

/* ====================================================================== */
/* Synthetic generator: src/sim_harness.cpp:17-144                          */
/* ====================================================================== */

typedef struct {
    double lo, hi, jitter;
} Range;

/* sim_harness.cpp:24-30 */
static const Range kAlpha = {40.0, 400.0, 0.10};
static const Range kBeta = {40.0, 400.0, 0.10};
static const Range kT0 = {0.04, 0.30, 0.05};
static const Range kGamma = {0.004, 0.020, 0.10};
static const Range kC = {0.002, 0.0055, 0.10};
static const Range kP0 = {40.0, 90.0, 0.05};
static const Range kKappa = {5.0, 15.0, 0.05};

/* sim_harness.cpp:19-21 */
static double r_floor(Range r) { return r.lo * (1.0 - r.jitter); }
static double r_span(Range r) { return r.hi * (1.0 + r.jitter) - r_floor(r); }
static double r_encode(Range r, double v) { return (v - r_floor(r)) / r_span(r); }
/* sim_harness.cpp:32-36 */
static double lerp(Range r, double w) { return r.lo + (r.hi - r.lo) * w; }
static double jittered(Range r, double w, uint64_t* s) {
    return lerp(r, w) * (1.0 + r.jitter * orc_rng_uniform(s, -1.0, 1.0));
}

/* Category slot indices (ptx_features.cpp:18-49); the 126-wide count vector
 * is [instr 0..100 | dtype 101..117 | memspace 118..125]. */
enum {
    SL_ADD = 0, SL_MUL = 4, SL_FMA = 37, SL_SETP = 39, SL_MOV = 51, SL_LD = 54, SL_ST = 56,
    SL_CVT = 61, SL_BRA = 71, SL_RET = 74, SL_BAR = 76,
    DT = 101, DT_S32 = DT + 2, DT_U32 = DT + 6, DT_U64 = DT + 7, DT_F32 = DT + 10,
    DT_F64 = DT + 11, DT_B32 = DT + 14, DT_B64 = DT + 15,
    MS = 118, MS_REG = MS + 0, MS_CONST = MS + 2, MS_GLOBAL = MS + 3, MS_LOCAL = MS + 4,
    MS_PARAM = MS + 5, MS_SHARED = MS + 6,
};

static uint32_t slot(double w) { return (uint32_t)llround(w * 1e6); }

/* features_from, sim_harness.cpp:42-99: DCGM vector and raw PTX counts. */
static void features_from(const double* p, uint32_t* counts, double* dcgm) {
    const double za = r_encode(kAlpha, p[5]);
    const double zb = r_encode(kBeta, p[6]);
    const double zt = r_encode(kT0, p[4]);
    const double zg = r_encode(kGamma, p[2]);
    const double zc = r_encode(kC, p[3]);
    const double zp = r_encode(kP0, p[0]);
    const double zk = r_encode(kKappa, p[1]);
    dcgm[0] = 0.30 + 0.65 * zt;
    dcgm[1] = 0.10 + 0.80 * zp;
    dcgm[2] = 0.02 + 0.60 * zg;
    dcgm[3] = 0.05 + 0.90 * za;
    dcgm[4] = 0.02 + 0.70 * zk;
    dcgm[5] = 0.05 + 0.90 * zb;
    dcgm[6] = 0.02 + 0.90 * zc;
    dcgm[7] = 0.05 + 0.45 * zb + 0.45 * zc;

    const double s = p[6] / (p[5] + p[6]);
    const double arith = 0.70 * s;
    const double mem = 0.70 * (1.0 - s);
    memset(counts, 0, 126 * sizeof(uint32_t));
    counts[SL_ADD] = slot(0.35 * arith);
    counts[SL_MUL] = slot(0.25 * arith);
    counts[SL_FMA] = slot(0.40 * arith);
    counts[SL_LD] = slot(0.60 * mem);
    counts[SL_ST] = slot(0.40 * mem);
    counts[SL_MOV] = slot(0.12);
    counts[SL_SETP] = slot(0.06);
    counts[SL_BRA] = slot(0.06);
    counts[SL_CVT] = slot(0.03);
    counts[SL_BAR] = slot(0.02);
    counts[SL_RET] = slot(0.01);

    counts[DT_F32] = slot(0.35 + 0.25 * s);
    counts[DT_S32] = slot(0.30 - 0.15 * s);
    counts[DT_U32] = slot(0.10);
    counts[DT_B32] = slot(0.05);
    counts[DT_F64] = slot(0.08 - 0.05 * s);
    counts[DT_U64] = slot(0.07);
    counts[DT_B64] = slot(0.05 - 0.05 * s);

    counts[MS_GLOBAL] = slot(0.50 - 0.25 * s);
    counts[MS_SHARED] = slot(0.12 + 0.10 * s);
    counts[MS_PARAM] = slot(0.08);
    counts[MS_REG] = slot(0.20 + 0.15 * s);
    counts[MS_LOCAL] = slot(0.05);
    counts[MS_CONST] = slot(0.05);
}

/* gen_kernel(seed, rho), sim_harness.cpp:124-144 */
int orc_gen_kernel_rho(uint64_t seed, double rho, double* p, uint32_t* counts, double* dcgm,
                       double* fused) {
    if (!(rho >= 0.0 && rho <= 1.0)) return ORC_InvalidArgument;
    uint64_t base = seed;
    uint64_t s = orc_rng_fork(&base, 0x6e6b);
    double q[7];
    q[5] = jittered(kAlpha, 1.0 - rho, &s);
    q[6] = jittered(kBeta, rho, &s);
    q[4] = jittered(kT0, orc_rng_uniform01(&s), &s);
    q[2] = jittered(kGamma, 1.0 - rho, &s);
    q[3] = jittered(kC, rho, &s);
    q[0] = jittered(kP0, orc_rng_uniform01(&s), &s);
    q[1] = jittered(kKappa, orc_rng_uniform01(&s), &s);
    int st = orc_validate_params(q);
    if (st) return st;
    if (p) memcpy(p, q, sizeof q);
    uint32_t c[126];
    double d[8];
    features_from(q, c, d);
    if (counts) memcpy(counts, c, sizeof c);
    if (dcgm) memcpy(dcgm, d, sizeof d);
    if (fused) orc_fuse(c, d, 1, fused);
    return ORC_OK;
}

/* gen_kernel(seed), sim_harness.cpp:118-122 */
static void gen_one(uint64_t seed, double* p, uint32_t* counts, double* dcgm, double* fused) {
    uint64_t s = seed;
    double rho = orc_rng_uniform01(&s);
    orc_gen_kernel_rho(seed, rho, p, counts, dcgm, fused);
}

void orc_gen_seeded(const uint64_t* seeds, int64_t n, double* params, uint32_t* counts,
                    double* dcgm, double* fused) {
    for (int64_t i = 0; i < n; ++i)
        gen_one(seeds[i], params ? params + 7 * i : NULL, counts ? counts + 126 * i : NULL,
                dcgm ? dcgm + 8 * i : NULL, fused ? fused + 134 * i : NULL);
}

/* ====================================================================== */
/* Features: ptx_features.cpp:311-329, telemetry.cpp:63-101, mlp.cpp:158-165 */
/* ====================================================================== */

static const int kCatBase[3] = {0, 101, 118};
static const int kCatLen[3] = {101, 17, 8};

/* featurize, ptx_features.cpp:311-329: per category v[i] = count[i] / total,
 * all-zero when the total is 0.  The total is a double sum of integer counts
 * (exact below 2^53, so independent of std::map iteration order). */
void orc_featurize(const uint32_t* counts, int64_t n, double* out) {
    for (int64_t k = 0; k < n; ++k) {
        const uint32_t* c = counts + 126 * k;
        double* v = out + 126 * k;
        for (int cat = 0; cat < 3; ++cat) {
            double total = 0.0;
            for (int i = 0; i < kCatLen[cat]; ++i) total += (double)c[kCatBase[cat] + i];
            for (int i = 0; i < kCatLen[cat]; ++i)
                v[kCatBase[cat] + i] =
                    total == 0.0 ? 0.0 : (double)c[kCatBase[cat] + i] / total;
        }
    }
}

/* load_dcgm_samples mean, telemetry.cpp:73-89 (CSV parsing is out of scope:
 * rows arrive as parsed doubles). */
int orc_dcgm_mean(const double* samples, int64_t rows, double* out, int64_t* bad_row) {
    if (bad_row) *bad_row = 0;
    if (rows < 1) return ORC_EmptyTrace;
    double sum[8] = {0};
    for (int64_t r = 0; r < rows; ++r) {
        for (int m = 0; m < 8; ++m) {
            double v = samples[8 * r + m];
            if (v < 0.0 || v > 1.0) {
                if (bad_row) *bad_row = r + 1;
                return ORC_OutOfRange;
            }
            sum[m] += v;
        }
    }
    for (int m = 0; m < 8; ++m) out[m] = sum[m] / (double)rows;
    return ORC_OK;
}

/* FusedFeatures::as_vector, mlp.cpp:158-165: [dcgm 8 | instr 101 | dtype 17 | memspace 8] */
void orc_fuse(const uint32_t* counts, const double* dcgm, int64_t n, double* fused) {
    for (int64_t k = 0; k < n; ++k) {
        double* f = fused + 134 * k;
        for (int m = 0; m < 8; ++m) f[m] = dcgm[8 * k + m];
        orc_featurize(counts + 126 * k, 1, f + 8);
    }
}

/* ====================================================================== */
/* MLP: src/mlp.cpp:17-253                                                 */
/* ====================================================================== */

int64_t orc_mlp_weight_count(const int* sizes, int nl) {
    int64_t t = 0;
    for (int l = 0; l + 1 < nl; ++l) t += (int64_t)sizes[l] * sizes[l + 1];
    return t;
}

int64_t orc_mlp_bias_count(const int* sizes, int nl) {
    int64_t t = 0;
    for (int l = 1; l < nl; ++l) t += sizes[l];
    return t;
}

/* init_mlp, mlp.cpp:184-207: Glorot-uniform drawn row-major from Rng(seed). */
int orc_init_mlp(const int* sizes, int nl, uint64_t seed, double* W, double* b) {
    if (nl < 2) return ORC_InvalidModel;
    for (int l = 0; l < nl; ++l)
        if (sizes[l] <= 0) return ORC_InvalidModel;
    uint64_t s = seed;
    for (int l = 0; l + 1 < nl; ++l) {
        const int fan_in = sizes[l], fan_out = sizes[l + 1];
        const double limit = sqrt(6.0 / (fan_in + fan_out));
        for (int r = 0; r < fan_out; ++r)
            for (int c = 0; c < fan_in; ++c) *W++ = orc_rng_uniform(&s, -limit, limit);
        for (int r = 0; r < fan_out; ++r) *b++ = 0.0;
    }
    return ORC_OK;
}

/* sigmoid, mlp.cpp:17-20 */
static double sigmoid(double z) { return 1.0 / (1.0 + exp(-z)); }

static int max_width(const int* sizes, int nl) {
    int w = 0;
    for (int l = 0; l < nl; ++l)
        if (sizes[l] > w) w = sizes[l];
    return w;
}

/* forward_trace, mlp.cpp:22-32, one column.  acts must hold sum(sizes)
 * doubles; returns pointer to the (standardized) output activations. */
static double* forward_trace1(const int* sizes, int nl, const double* W, const double* b,
                              const double* x, double* acts) {
    double* a = acts;
    memcpy(a, x, sizeof(double) * sizes[0]);
    for (int l = 0; l + 1 < nl; ++l) {
        const int in = sizes[l], out = sizes[l + 1];
        double* z = a + in;
        for (int r = 0; r < out; ++r) {
            double acc = 0.0;
            const double* w = W + (int64_t)r * in;
            for (int c = 0; c < in; ++c) acc += w[c] * a[c];
            z[r] = acc + b[r];
            if (l + 2 < nl) z[r] = sigmoid(z[r]);
        }
        W += (int64_t)in * out;
        b += out;
        a = z;
    }
    return a;
}

static int64_t act_total(const int* sizes, int nl) {
    int64_t t = 0;
    for (int l = 0; l < nl; ++l) t += sizes[l];
    return t;
}

/* forward_raw, mlp.cpp:232-235: (out .* std) + mean */
void orc_forward_raw(const int* sizes, int nl, const double* W, const double* b,
                     const double* mean, const double* std, const double* x, int64_t n,
                     double* out) {
    const int in = sizes[0], od = sizes[nl - 1];
    double* acts = malloc(sizeof(double) * act_total(sizes, nl));
    for (int64_t k = 0; k < n; ++k) {
        const double* o = forward_trace1(sizes, nl, W, b, x + (int64_t)in * k, acts);
        for (int i = 0; i < od; ++i) out[(int64_t)od * k + i] = o[i] * std[i] + mean[i];
    }
    free(acts);
}

/* predict_params, mlp.cpp:237-253 (kBetaFloor mlp.cpp:15) */
static void predict_one(const int* sizes, int nl, const double* W, const double* b,
                        const double* mean, const double* std, const double* x, double* acts,
                        double* p, uint8_t* clamped) {
    const double* o = forward_trace1(sizes, nl, W, b, x, acts);
    int cl = 0;
    for (int i = 0; i < 7; ++i) {
        double r = o[i] * std[i] + mean[i];
        if (r < 0.0) {
            r = 0.0;
            cl = 1;
        }
        p[i] = r;
    }
    if (p[5] + p[6] <= 0.0) {
        p[6] = 1e-12;
        cl = 1;
    }
    if (clamped) *clamped = (uint8_t)cl;
}

/* ---- tiny thread pool helper ---------------------------------------------- */
typedef void (*range_fn)(void* ctx, int64_t lo, int64_t hi);
typedef struct {
    range_fn fn;
    void* ctx;
    int64_t lo, hi;
} Job;
static void* job_main(void* a) {
    Job* j = (Job*)a;
    j->fn(j->ctx, j->lo, j->hi);
    return NULL;
}
static void parallel_for(int64_t n, int threads, range_fn fn, void* ctx) {
    if (threads < 1) threads = 1;
    if (threads > 512) threads = 512;
    if ((int64_t)threads > n) threads = (int)(n > 0 ? n : 1);
    if (threads == 1) {
        fn(ctx, 0, n);
        return;
    }
    pthread_t tid[512];
    Job jobs[512];
    for (int t = 0; t < threads; ++t) {
        jobs[t].fn = fn;
        jobs[t].ctx = ctx;
        jobs[t].lo = n * t / threads;
        jobs[t].hi = n * (t + 1) / threads;
        pthread_create(&tid[t], NULL, job_main, &jobs[t]);
    }
    for (int t = 0; t < threads; ++t) pthread_join(tid[t], NULL);
}

typedef struct {
    const int* sizes;
    int nl;
    const double *W, *b, *mean, *std, *x;
    double* params;
    uint8_t* clamped;
} PredictCtx;

static void predict_range(void* c, int64_t lo, int64_t hi) {
    PredictCtx* p = (PredictCtx*)c;
    double* acts = malloc(sizeof(double) * act_total(p->sizes, p->nl));
    for (int64_t k = lo; k < hi; ++k)
        predict_one(p->sizes, p->nl, p->W, p->b, p->mean, p->std,
                    p->x + (int64_t)p->sizes[0] * k, acts, p->params + 7 * k,
                    p->clamped ? p->clamped + k : NULL);
    free(acts);
}

void orc_predict_params(const int* sizes, int nl, const double* W, const double* b,
                        const double* mean, const double* std, const double* x, int64_t n,
                        double* params, uint8_t* clamped, int threads) {
    PredictCtx c = {sizes, nl, W, b, mean, std, x, params, clamped};
    parallel_for(n, threads, predict_range, &c);
}

/* ====================================================================== */
/* Training: mlp.cpp:57-130,259-289 (target stats, SGD epoch, loss, backprop)      */
/* ====================================================================== */

/* mse_loss, mlp.cpp:259-263: 0.5 * ||out - y||^2 / (B * out_dim) */
double orc_mse_loss(const int* sizes, int nl, const double* W, const double* b,
                    const double* x, const double* y, int64_t B) {
    const int in = sizes[0], od = sizes[nl - 1];
    double* acts = malloc(sizeof(double) * act_total(sizes, nl));
    double sq = 0.0;
    for (int64_t k = 0; k < B; ++k) {
        const double* o = forward_trace1(sizes, nl, W, b, x + (int64_t)in * k, acts);
        for (int i = 0; i < od; ++i) {
            double d = o[i] - y[(int64_t)od * k + i];
            sq += d * d;
        }
    }
    free(acts);
    return 0.5 * sq / (double)(B * od);
}

/* analytic_gradients, mlp.cpp:265-289 */
void orc_analytic_gradients(const int* sizes, int nl, const double* W, const double* b,
                            const double* x, const double* y, int64_t B, double* gW,
                            double* gb) {
    const int L = nl - 1, in = sizes[0], od = sizes[nl - 1];
    const double scale = 1.0 / (double)(B * od);
    const int64_t nw = orc_mlp_weight_count(sizes, nl), nb = orc_mlp_bias_count(sizes, nl);
    memset(gW, 0, sizeof(double) * nw);
    memset(gb, 0, sizeof(double) * nb);
    int64_t woff[64], boff[64], aoff[65];
    woff[0] = boff[0] = aoff[0] = 0;
    for (int l = 0; l < L; ++l) {
        woff[l + 1] = woff[l] + (int64_t)sizes[l] * sizes[l + 1];
        boff[l + 1] = boff[l] + sizes[l + 1];
        aoff[l + 1] = aoff[l] + sizes[l];
    }
    aoff[L + 1] = aoff[L] + sizes[L];
    const int wmax = max_width(sizes, nl);
    double* acts = malloc(sizeof(double) * act_total(sizes, nl));
    double* delta = malloc(sizeof(double) * wmax);
    double* nd = malloc(sizeof(double) * wmax);
    for (int64_t k = 0; k < B; ++k) {
        forward_trace1(sizes, nl, W, b, x + (int64_t)in * k, acts);
        const double* out = acts + aoff[L];
        for (int i = 0; i < od; ++i) delta[i] = (out[i] - y[(int64_t)od * k + i]) * scale;
        for (int l = L - 1; l >= 0; --l) {
            const int fi = sizes[l], fo = sizes[l + 1];
            const double* a = acts + aoff[l];
            double* g = gW + woff[l];
            for (int r = 0; r < fo; ++r) {
                for (int c = 0; c < fi; ++c) g[(int64_t)r * fi + c] += delta[r] * a[c];
                gb[boff[l] + r] += delta[r];
            }
            if (l > 0) {
                const double* w = W + woff[l];
                for (int c = 0; c < fi; ++c) {
                    double acc = 0.0;
                    for (int r = 0; r < fo; ++r) acc += w[(int64_t)r * fi + c] * delta[r];
                    nd[c] = acc * a[c] * (1.0 - a[c]);
                }
                memcpy(delta, nd, sizeof(double) * fi);
            }
        }
    }
    free(acts);
    free(delta);
    free(nd);
}

/* numeric_gradients, mlp.cpp:291-322 (central differences) */
void orc_numeric_gradients(const int* sizes, int nl, const double* W, const double* b,
                           const double* x, const double* y, int64_t B, double eps,
                           double* gW, double* gb) {
    const int64_t nw = orc_mlp_weight_count(sizes, nl), nb = orc_mlp_bias_count(sizes, nl);
    double* Wp = malloc(sizeof(double) * nw);
    double* bp = malloc(sizeof(double) * nb);
    memcpy(Wp, W, sizeof(double) * nw);
    memcpy(bp, b, sizeof(double) * nb);
    for (int64_t i = 0; i < nw; ++i) {
        double saved = Wp[i];
        Wp[i] = saved + eps;
        double up = orc_mse_loss(sizes, nl, Wp, bp, x, y, B);
        Wp[i] = saved - eps;
        double down = orc_mse_loss(sizes, nl, Wp, bp, x, y, B);
        Wp[i] = saved;
        gW[i] = (up - down) / (2.0 * eps);
    }
    for (int64_t i = 0; i < nb; ++i) {
        double saved = bp[i];
        bp[i] = saved + eps;
        double up = orc_mse_loss(sizes, nl, Wp, bp, x, y, B);
        bp[i] = saved - eps;
        double down = orc_mse_loss(sizes, nl, Wp, bp, x, y, B);
        bp[i] = saved;
        gb[i] = (up - down) / (2.0 * eps);
    }
    free(Wp);
    free(bp);
}

/* target_stats, mlp.cpp:57-79 (population std; zero variance -> std 1, mean 0) */
int orc_target_stats(const double* t, int64_t n, int od, double* mean, double* std) {
    int degenerate = 0;
    for (int i = 0; i < od; ++i) mean[i] = 0.0;
    for (int64_t k = 0; k < n; ++k)
        for (int i = 0; i < od; ++i) mean[i] += t[(int64_t)od * k + i];
    for (int i = 0; i < od; ++i) mean[i] /= (double)n;
    for (int i = 0; i < od; ++i) std[i] = 0.0;
    for (int64_t k = 0; k < n; ++k)
        for (int i = 0; i < od; ++i) {
            double d = t[(int64_t)od * k + i] - mean[i];
            std[i] += d * d;
        }
    for (int i = 0; i < od; ++i) {
        std[i] = sqrt(std[i] / (double)n);
        if (std[i] == 0.0) {
            std[i] = 1.0;
            mean[i] = 0.0;
            ++degenerate;
        }
    }
    return degenerate;
}

/* sgd_epoch, mlp.cpp:84-112 */
double orc_sgd_epoch(const int* sizes, int nl, double* W, double* b, const double* feats,
                     const double* targets, int64_t n, const double* mean, const double* std,
                     double lr, int batch, uint64_t* rng_state) {
    const int in = sizes[0], od = sizes[nl - 1];
    const int64_t nw = orc_mlp_weight_count(sizes, nl), nb = orc_mlp_bias_count(sizes, nl);
    uint64_t* order = malloc(sizeof(uint64_t) * (size_t)n);
    orc_shuffled_indices((uint64_t)n, rng_state, order);
    double* x = malloc(sizeof(double) * (size_t)batch * in);
    double* y = malloc(sizeof(double) * (size_t)batch * od);
    double* gW = malloc(sizeof(double) * nw);
    double* gb = malloc(sizeof(double) * nb);
    double loss_sum = 0.0;
    int64_t batches = 0;
    for (int64_t start = 0; start < n; start += batch) {
        int64_t bsz = n - start < batch ? n - start : batch;
        for (int64_t k = 0; k < bsz; ++k) {
            const int64_t e = (int64_t)order[start + k];
            memcpy(x + in * k, feats + in * e, sizeof(double) * in);
            for (int i = 0; i < od; ++i)
                y[od * k + i] = (targets[od * e + i] - mean[i]) / std[i];
        }
        orc_analytic_gradients(sizes, nl, W, b, x, y, bsz, gW, gb);
        loss_sum += orc_mse_loss(sizes, nl, W, b, x, y, bsz);
        ++batches;
        for (int64_t i = 0; i < nw; ++i) W[i] -= lr * gW[i];
        for (int64_t i = 0; i < nb; ++i) b[i] -= lr * gb[i];
    }
    free(order);
    free(x);
    free(y);
    free(gW);
    free(gb);
    double mean_loss = loss_sum / (double)batches;
    return isfinite(mean_loss) ? mean_loss : NAN;
}

/* ====================================================================== */
/* Sweep: src/optimizer.cpp:18-117                                          */
/* ====================================================================== */

typedef struct {
    double cost, energy, time;
    int idx;
} Cand;

/* better(), optimizer.cpp:27-32.  vc is strictly increasing in fc_idx (the
 * domain is validated), so comparing vc then fm equals comparing the index. */
static int better(const Cand* a, const Cand* b) {
    if (a->cost != b->cost) return a->cost < b->cost;
    if (a->energy != b->energy) return a->energy < b->energy;
    return a->idx < b->idx;
}

typedef struct {
    const double* params;
    const double *core, *mem, *dev;
    int nc, nm;
    const double* etas;
    int n_eta;
    double pmax;
    int32_t* idx;
    double *cost, *energy, *time;
    int32_t* kstatus;
    int64_t n;
    double* vc; /* per core level, required_voltage_mhz */
} SweepCtx;

/* brute_force_config, optimizer.cpp:90-117; evaluate() at :34-39. */
static void sweep_one(const SweepCtx* c, const double* p, double eta, Cand* best) {
    int have = 0;
    for (int i = 0; i < c->nc; ++i) {
        const double fc = c->core[i], vc = c->vc[i];
        for (int j = 0; j < c->nm; ++j) {
            const double fm = c->mem[j];
            Cand cand;
            const double P = orc_power(p, vc, fc, fm);
            const double T = orc_exec_time(p, vc, fc, fm);
            cand.cost = (eta * P + (1.0 - eta) * c->pmax) * T; /* dvfs_model.hpp:103 */
            cand.energy = P * T;                               /* dvfs_model.hpp:94 */
            cand.time = T;
            cand.idx = i * c->nm + j;
            if (!have || better(&cand, best)) {
                *best = cand;
                have = 1;
            }
        }
    }
}

static void sweep_range(void* v, int64_t lo, int64_t hi) {
    const SweepCtx* c = (const SweepCtx*)v;
    for (int64_t k = lo; k < hi; ++k) {
        const double* p = c->params + 7 * k;
        int st = orc_validate_params(p);
        if (c->kstatus) c->kstatus[k] = st;
        for (int e = 0; e < c->n_eta; ++e) {
            const int64_t o = (int64_t)e * c->n + k;
            if (st) {
                c->idx[o] = -1;
                if (c->cost) c->cost[o] = NAN;
                if (c->energy) c->energy[o] = NAN;
                if (c->time) c->time[o] = NAN;
                continue;
            }
            Cand best;
            sweep_one(c, p, c->etas[e], &best);
            c->idx[o] = best.idx;
            if (c->cost) c->cost[o] = best.cost;
            if (c->energy) c->energy[o] = best.energy;
            if (c->time) c->time[o] = best.time;
        }
    }
}

static int sweep_common(SweepCtx* c, int threads) {
    int st = orc_validate_domain(c->core, c->nc, c->mem, c->nm, c->dev);
    if (st) return st;
    for (int e = 0; e < c->n_eta; ++e)
        if (!(c->etas[e] >= 0.0 && c->etas[e] <= 1.0)) return ORC_EtaOutOfRange;
    c->vc = malloc(sizeof(double) * c->nc);
    for (int i = 0; i < c->nc; ++i) c->vc[i] = orc_required_voltage_mhz(c->core[i], c->dev);
    parallel_for(c->n, threads, sweep_range, c);
    free(c->vc);
    return ORC_OK;
}

int orc_brute_force(const double* params, int64_t n, const double* core, int nc,
                    const double* mem, int nm, const double* dev, double eta, double pmax,
                    int32_t* idx, double* cost, double* energy, double* time, int32_t* kstatus,
                    int threads) {
    SweepCtx c = {params, core, mem, dev, nc, nm, &eta, 1, pmax, idx, cost, energy, time,
                  kstatus, n, NULL};
    return sweep_common(&c, threads);
}

int orc_eta_sweep(const double* params, int64_t n, const double* core, int nc,
                  const double* mem, int nm, const double* dev, const double* etas, int n_eta,
                  double pmax, int32_t* idx, double* cost, int threads) {
    SweepCtx c = {params, core, mem, dev, nc, nm, etas, n_eta, pmax, idx, cost, NULL, NULL,
                  NULL, n, NULL};
    return sweep_common(&c, threads);
}

/* ====================================================================== */
/* Synthetic stream (run_campaign seeding, sim_harness.cpp:241-242)         */
/* ====================================================================== */

typedef struct {
    uint64_t root, salt_base;
    int64_t first;
    double* params;
    uint32_t* counts;
    double *dcgm, *fused;
} GenCtx;

static void gen_range(void* v, int64_t lo, int64_t hi) {
    const GenCtx* g = (const GenCtx*)v;
    for (int64_t k = lo; k < hi; ++k) {
        uint64_t child = orc_rng_fork(&g->root, g->salt_base + (uint64_t)(g->first + k));
        uint64_t seed = orc_rng_next(&child);
        gen_one(seed, g->params ? g->params + 7 * k : NULL,
                g->counts ? g->counts + 126 * k : NULL, g->dcgm ? g->dcgm + 8 * k : NULL,
                g->fused ? g->fused + 134 * k : NULL);
    }
}

void orc_gen_stream(uint64_t root, uint64_t salt_base, int64_t first, int64_t n,
                    double* params, uint32_t* counts, double* dcgm, double* fused,
                    int threads) {
    GenCtx g = {root, salt_base, first, params, counts, dcgm, fused};
    parallel_for(n, threads, gen_range, &g);
}

/* ====================================================================== */
/* Pipeline: featurize + as_vector + predict_params + brute_force_config    */
/* ====================================================================== */

typedef struct {
    const uint32_t* counts;
    const double* dcgm;
    const int* sizes;
    int nl;
    const double *W, *b, *mean, *std;
    SweepCtx* sweep;
    double* params_out;
    uint8_t* clamped;
} PipeCtx;

static void pipe_range(void* v, int64_t lo, int64_t hi) {
    const PipeCtx* c = (const PipeCtx*)v;
    double* acts = malloc(sizeof(double) * act_total(c->sizes, c->nl));
    double fused[134], p[7];
    for (int64_t k = lo; k < hi; ++k) {
        orc_fuse(c->counts + 126 * k, c->dcgm + 8 * k, 1, fused);
        uint8_t cl;
        predict_one(c->sizes, c->nl, c->W, c->b, c->mean, c->std, fused, acts, p, &cl);
        if (c->params_out) memcpy(c->params_out + 7 * k, p, sizeof p);
        if (c->clamped) c->clamped[k] = cl;
        Cand best;
        sweep_one(c->sweep, p, c->sweep->etas[0], &best);
        c->sweep->idx[k] = best.idx;
        if (c->sweep->cost) c->sweep->cost[k] = best.cost;
        if (c->sweep->energy) c->sweep->energy[k] = best.energy;
        if (c->sweep->time) c->sweep->time[k] = best.time;
    }
    free(acts);
}

int orc_pipeline(const uint32_t* counts, const double* dcgm, int64_t n, const int* sizes,
                 int nl, const double* W, const double* b, const double* mean,
                 const double* std, const double* core, int nc, const double* mem, int nm,
                 const double* dev, double eta, double pmax, double* params_out,
                 uint8_t* clamped, int32_t* idx, double* cost, double* energy, double* time,
                 int threads) {
    if (nl < 2 || sizes[0] != 134 || sizes[nl - 1] != 7) return ORC_InvalidModel;
    int st = orc_validate_domain(core, nc, mem, nm, dev);
    if (st) return st;
    if (!(eta >= 0.0 && eta <= 1.0)) return ORC_EtaOutOfRange;
    SweepCtx s = {NULL, core, mem, dev, nc, nm, &eta, 1, pmax, idx, cost, energy, time,
                  NULL, n, NULL};
    s.vc = malloc(sizeof(double) * nc);
    for (int i = 0; i < nc; ++i) s.vc[i] = orc_required_voltage_mhz(core[i], dev);
    PipeCtx c = {counts, dcgm, sizes, nl, W, b, mean, std, &s, params_out, clamped};
    parallel_for(n, threads, pipe_range, &c);
    free(s.vc);
    return ORC_OK;
}

/* ===========================================================================
 * param_fit (proj/src/param_fit.cpp) — TEST INFRASTRUCTURE ONLY.
 *
 * The reference solves its least-squares problems with Eigen's
 * ColPivHouseholderQR (threshold 1e-10, param_fit.cpp:29-31,108-110).  Eigen is
 * absent here; orc_cpqr_* restate that algorithm (Householder QR with column
 * pivoting by updated column norms, Eigen 3.4 ColPivHouseholderQR::computeInPlace,
 * rank() = #|R_ii| > threshold * maxpivot among the nonzero pivots, solve() =
 * Q^T b, upper-triangular solve on the nonzero pivots, permute back) with naive
 * summation (Eigen vectorises its reductions, so results agree to rounding).
 * ======================================================================== */
#define ORC_QR_MAXC 4

typedef struct {
    int rows, cols, nonzero, perm[ORC_QR_MAXC];
    double maxpivot, hcoef[ORC_QR_MAXC];
    double* a; /* column-major rows x cols, overwritten by R (upper) + Householder essentials */
} orc_qr;

static double orc_colnorm(const double* a, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += a[i] * a[i];
    return sqrt(s);
}

/* Eigen 3.4 ColPivHouseholderQR<MatrixXd>::computeInPlace */
static void orc_cpqr_compute(orc_qr* q) {
    const int rows = q->rows, cols = q->cols, size = rows < cols ? rows : cols;
    double* a = q->a;
    double normsU[ORC_QR_MAXC], normsD[ORC_QR_MAXC], maxn = 0.0;
    for (int k = 0; k < cols; ++k) {
        normsD[k] = normsU[k] = orc_colnorm(a + (size_t)k * rows, rows);
        if (normsU[k] > maxn) maxn = normsU[k];
        q->perm[k] = k;
    }
    const double eps = 2.220446049250313e-16;
    const double thr_helper = (maxn * eps) * (maxn * eps) / (double)rows;
    const double downdate_thr = sqrt(eps);
    q->nonzero = size;
    q->maxpivot = 0.0;
    for (int k = 0; k < size; ++k) {
        int big = k;
        for (int j = k + 1; j < cols; ++j)
            if (normsU[j] > normsU[big]) big = j;
        const double big_sq = normsU[big] * normsU[big];
        if (q->nonzero == size && big_sq < thr_helper * (double)(rows - k)) q->nonzero = k;
        if (big != k) {
            for (int i = 0; i < rows; ++i) {
                double t = a[(size_t)k * rows + i];
                a[(size_t)k * rows + i] = a[(size_t)big * rows + i];
                a[(size_t)big * rows + i] = t;
            }
            double t = normsU[k]; normsU[k] = normsU[big]; normsU[big] = t;
            t = normsD[k]; normsD[k] = normsD[big]; normsD[big] = t;
            int tp = q->perm[k]; q->perm[k] = q->perm[big]; q->perm[big] = tp;
        }
        /* makeHouseholderInPlace on column k, rows k.. */
        double* v = a + (size_t)k * rows + k;
        const int m = rows - k;
        double tail = 0.0;
        for (int i = 1; i < m; ++i) tail += v[i] * v[i];
        const double c0 = v[0];
        double tau, beta;
        if (tail <= 2.2250738585072014e-308) {
            tau = 0.0;
            beta = c0;
            for (int i = 1; i < m; ++i) v[i] = 0.0;
        } else {
            beta = sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            for (int i = 1; i < m; ++i) v[i] = v[i] / (c0 - beta);
            tau = (beta - c0) / beta;
        }
        v[0] = beta;
        q->hcoef[k] = tau;
        if (fabs(beta) > q->maxpivot) q->maxpivot = fabs(beta);
        /* apply H = I - tau [1; v] [1; v]^T to the remaining columns */
        for (int j = k + 1; j < cols; ++j) {
            double* c = a + (size_t)j * rows + k;
            double w = c[0];
            for (int i = 1; i < m; ++i) w += v[i] * c[i];
            w *= tau;
            c[0] -= w;
            for (int i = 1; i < m; ++i) c[i] -= w * v[i];
        }
        /* column norm downdates */
        for (int j = k + 1; j < cols; ++j) {
            if (normsU[j] != 0.0) {
                double t = fabs(a[(size_t)j * rows + k]) / normsU[j];
                t = (1.0 + t) * (1.0 - t);
                if (t < 0.0) t = 0.0;
                const double r = normsU[j] / normsD[j];
                const double t2 = t * r * r;
                if (t2 <= downdate_thr) {
                    normsD[j] = orc_colnorm(a + (size_t)j * rows + k + 1, rows - k - 1);
                    normsU[j] = normsD[j];
                } else {
                    normsU[j] *= sqrt(t);
                }
            }
        }
    }
}

static int orc_cpqr_rank(const orc_qr* q, double threshold) {
    const double pt = fabs(q->maxpivot) * threshold;
    int r = 0;
    for (int i = 0; i < q->nonzero; ++i) r += fabs(q->a[(size_t)i * q->rows + i]) > pt;
    return r;
}

/* solve(b): x = P [R11^-1 (Q^T b)_top; 0] */
static void orc_cpqr_solve(const orc_qr* q, const double* b, double* x, double* work) {
    const int rows = q->rows, cols = q->cols, size = rows < cols ? rows : cols;
    for (int i = 0; i < rows; ++i) work[i] = b[i];
    for (int k = 0; k < size; ++k) {
        const double* v = q->a + (size_t)k * rows + k;
        double w = work[k];
        for (int i = 1; i < rows - k; ++i) w += v[i] * work[k + i];
        w *= q->hcoef[k];
        work[k] -= w;
        for (int i = 1; i < rows - k; ++i) work[k + i] -= w * v[i];
    }
    const int nz = q->nonzero;
    double c[ORC_QR_MAXC];
    for (int i = nz - 1; i >= 0; --i) {
        double s = work[i];
        for (int j = i + 1; j < nz; ++j) s -= q->a[(size_t)j * rows + i] * c[j];
        c[i] = s / q->a[(size_t)i * rows + i];
    }
    for (int i = nz; i < cols; ++i) c[i] = 0.0;
    for (int i = 0; i < cols; ++i) x[q->perm[i]] = c[i];
}

static double orc_mape_pct(const double* pred, const double* obs, int n) { /* param_fit.cpp:19-24 */
    double acc = 0.0;
    for (int i = 0; i < n; ++i) acc += fabs(pred[i] - obs[i]) / fabs(obs[i]);
    return 100.0 * acc / (double)n;
}

/* fit_power (param_fit.cpp:43-77).  cfg [S][3] = vc, fc_mhz, fm_mhz.
 * out = p0, kappa_pow, gamma, c, mape_pct, constraint_active. */
int orc_fit_power(const double* cfg, const double* power, int S, double* out) {
    if (S < 4) return ORC_RankDeficient;
    for (int i = 0; i < S; ++i)
        if (!(power[i] > 0.0)) return ORC_InvalidArgument;
    double* a = (double*)malloc(sizeof(double) * 4 * S + sizeof(double) * 2 * S);
    double* work = a + 4 * S;
    double* pred = work + S;
    for (int i = 0; i < S; ++i) {
        const double vc = cfg[3 * i], fc = cfg[3 * i + 1], fm = cfg[3 * i + 2];
        a[i] = 1.0;
        a[S + i] = vc;
        a[2 * S + i] = fm;
        a[3 * S + i] = vc * vc * fc;
    }
    orc_qr q = {S, 4, 0, {0}, 0.0, {0}, a};
    orc_cpqr_compute(&q);
    if (orc_cpqr_rank(&q, 1e-10) < 4) {
        free(a);
        return ORC_RankDeficient;
    }
    double coef[4];
    orc_cpqr_solve(&q, power, coef, work);
    int active = 0;
    for (int j = 0; j < 4; ++j)
        if (coef[j] < 0.0) {
            coef[j] = 0.0;
            active = 1;
        }
    for (int i = 0; i < S; ++i) {  /* design * coef (design rebuilt: a was overwritten) */
        const double vc = cfg[3 * i], fc = cfg[3 * i + 1], fm = cfg[3 * i + 2];
        pred[i] = coef[0] * 1.0 + coef[1] * vc + coef[2] * fm + coef[3] * (vc * vc * fc);
    }
    for (int j = 0; j < 4; ++j) out[j] = coef[j];
    out[4] = orc_mape_pct(pred, power, S);
    out[5] = active;
    free(a);
    return ORC_OK;
}

/* solve_assignment / the iteration solve of fit_time for a branch assignment
 * (mem[i] = 1: memory branch).  Returns the rank-deficiency flag. */
static int orc_time_solve(const double* y, const double* ifm, const double* ifc, const uint8_t* mem,
                          int n, double* coef3, int* any_mem, int* any_core, double* scratch) {
    *any_mem = *any_core = 0;
    for (int i = 0; i < n; ++i) {
        if (mem[i]) *any_mem = 1; else *any_core = 1;
    }
    const int cols = 1 + *any_mem + *any_core;
    const int mc = *any_mem ? 1 : -1, cc = *any_core ? (*any_mem ? 2 : 1) : -1;
    double* a = scratch;
    double* work = scratch + 3 * n;
    for (int i = 0; i < cols * n; ++i) a[i] = 0.0;
    for (int i = 0; i < n; ++i) {
        a[i] = 1.0;
        if (mem[i]) a[(size_t)mc * n + i] = ifm[i]; else a[(size_t)cc * n + i] = ifc[i];
    }
    orc_qr q = {n, cols, 0, {0}, 0.0, {0}, a};
    orc_cpqr_compute(&q);
    if (orc_cpqr_rank(&q, 1e-10) < cols) return 1;
    double c[3] = {0, 0, 0};
    orc_cpqr_solve(&q, y, c, work);
    coef3[0] = c[0];
    coef3[1] = *any_mem ? c[mc] : 0.0;
    coef3[2] = *any_core ? c[cc] : 0.0;
    return 0;
}

static int orc_cmp_double(const void* x, const void* y) {
    const double a = *(const double*)x, b = *(const double*)y;
    return a < b ? -1 : (a > b ? 1 : 0);
}

/* fit_time (param_fit.cpp:79-247).  out = t0, alpha, beta, mape_pct,
 * constraint_active, partial_identifiability, iterations, final rss;
 * branch_out (optional) [S] = 1 for the memory branch. */
int orc_fit_time(const double* cfg, const double* tm, int S, double* out, uint8_t* branch_out) {
    if (S < 3) return ORC_Underdetermined;
    for (int i = 0; i < S; ++i)
        if (!(tm[i] > 0.0)) return ORC_InvalidArgument;
    double* buf = (double*)malloc(sizeof(double) * (size_t)S * 10);
    double *ifm = buf, *ifc = buf + S, *ratios = buf + 2 * S, *cuts = buf + 3 * S,
           *scratch = buf + 4 * S;
    uint8_t* branch = (uint8_t*)malloc((size_t)S * 2);
    uint8_t* assign = branch + S;
    double ysq = 0.0;
    for (int i = 0; i < S; ++i) {
        ifm[i] = 1.0 / cfg[3 * i + 2];
        ifc[i] = 1.0 / cfg[3 * i + 1];
        ysq += tm[i] * tm[i];
    }
    for (int i = 0; i < S; ++i) ratios[i] = ifm[i] / ifc[i];
    for (int i = 0; i < S; ++i) cuts[i] = ratios[i];
    qsort(cuts, S, sizeof(double), orc_cmp_double);
    int nu = 0;
    for (int i = 0; i < S; ++i)
        if (nu == 0 || cuts[i] != cuts[nu - 1]) cuts[nu++] = cuts[i];
    const double inf = 1.0 / 0.0;
    for (int i = 0; i < S; ++i) branch[i] = 0; /* Core */
    double best = inf;
    const double slack = 1e-12 * (ysq + 1.0);
    for (int c = 0; c <= nu; ++c) {  /* ordered: inf, cuts[0], cuts[1..] */
        const double cut = c == 0 ? inf : cuts[c - 1];
        for (int i = 0; i < S; ++i) assign[i] = ratios[i] >= cut;
        double co[3];
        int am, ac;
        double rss = inf;
        if (!orc_time_solve(tm, ifm, ifc, assign, S, co, &am, &ac, scratch)) {
            const double t0 = co[0], al = am ? (co[1] > 0.0 ? co[1] : 0.0) : 0.0,
                         be = ac ? (co[2] > 0.0 ? co[2] : 0.0) : 0.0;
            rss = 0.0;
            for (int i = 0; i < S; ++i) {
                const double x = al * ifm[i], z = be * ifc[i];
                const double pred = t0 + (x < z ? z : x);
                rss += (pred - tm[i]) * (pred - tm[i]);
            }
        }
        if (rss < best - slack) {
            best = rss;
            memcpy(branch, assign, (size_t)S);
        }
    }
    if (!(best < inf) && !(best > -inf)) { /* not finite */ }
    if (!isfinite(best)) {
        free(buf); free(branch);
        return ORC_Underdetermined;
    }
    double t0 = 0.0, al = 0.0, be = 0.0, rss = 0.0;
    int iters = 0, active = 0;
    for (int it = 0; it < 50; ++it) {
        ++iters;
        double co[3];
        int am, ac;
        if (orc_time_solve(tm, ifm, ifc, branch, S, co, &am, &ac, scratch)) {
            free(buf); free(branch);
            return ORC_Underdetermined;
        }
        t0 = co[0];
        al = am ? co[1] : 0.0;
        be = ac ? co[2] : 0.0;
        active = 0;
        if (al < 0.0) { al = 0.0; active = 1; }
        if (be < 0.0) { be = 0.0; active = 1; }
        rss = 0.0;
        for (int i = 0; i < S; ++i) {
            const double x = al * ifm[i], z = be * ifc[i];
            const double pred = t0 + (x < z ? z : x);
            rss += (pred - tm[i]) * (pred - tm[i]);
        }
        int changed = 0;
        for (int i = 0; i < S; ++i) {
            const uint8_t want = al * ifm[i] >= be * ifc[i];
            if (want != branch[i]) { branch[i] = want; changed = 1; }
        }
        if (!changed) break;
    }
    int all_mem = 1, all_core = 1;
    for (int i = 0; i < S; ++i) { if (branch[i]) all_core = 0; else all_mem = 0; }
    const int partial = all_mem || all_core;
    if (t0 < 0.0) { t0 = 0.0; active = 1; }
    if (partial) { if (all_mem) be = 0.0; else al = 0.0; }
    double* pred = scratch;
    for (int i = 0; i < S; ++i) {
        const double x = al * ifm[i], z = be * ifc[i];
        pred[i] = t0 + (x < z ? z : x);
    }
    out[0] = t0; out[1] = al; out[2] = be;
    out[3] = orc_mape_pct(pred, tm, S);
    out[4] = active; out[5] = partial; out[6] = iters; out[7] = rss;
    if (branch_out) memcpy(branch_out, branch, (size_t)S);
    free(buf); free(branch);
    return ORC_OK;
}
