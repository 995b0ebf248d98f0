// fit.cu — batched param_fit (sm_100a): fit_power and fit_time for many kernels
// measured on the same configuration grid (reference proj/src/param_fit.cpp).
//
// run_campaign measures every training kernel over the whole DVFS grid
// (measure_sweep, sim_harness.cpp:157-170) and fits each sweep with fit_power /
// fit_time (sim_harness.cpp:269-270) to get the MLP's training targets.  With a
// shared grid every least-squares design is shared by all kernels:
//   * fit_power (param_fit.cpp:43-77): one design [1, vc, fm, vc^2 fc];
//   * fit_time (param_fit.cpp:79-247): the candidate branch assignments are the
//     threshold splits of the grid's fc/fm ratios (":128-145"), and every
//     reassignment of the alternating iterations (":211-219") is again such a
//     split, so all designs the algorithm can meet are known up front.
// The host factors each design once with the reference's solver (Eigen's
// ColPivHouseholderQR, restated below: column pivoting by updated norms,
// threshold 1e-10 rank decision) and stores its solve operator as a matrix
// (solve() is linear in the right-hand side).  The device then runs the
// reference's per-kernel control flow — the ordered split search with its tie
// slack, the alternating iterations with clamping, partial identifiability,
// MAPE — in FP64, one thread per kernel, with coef = M * y in place of
// qr.solve(y) (same linear map; rounding differs at the 1e-15 level).
#include <math.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "common.cuh"

namespace dso_b200 {

// ---------------------------------------------------------------------------
// Host: Householder QR with column pivoting (Eigen 3.4 ColPivHouseholderQR).
namespace {

struct CpQr {
    int rows = 0, cols = 0, nonzero = 0;
    std::vector<double> a;  // column-major; R in the upper triangle, essentials below
    std::vector<double> hcoef;
    std::vector<int> perm;
    double maxpivot = 0.0;
};

double colnorm(const double* v, int n) {
    double s = 0.0;
    for (int i = 0; i < n; ++i) s += v[i] * v[i];
    return std::sqrt(s);
}

void cpqr_compute(CpQr& q) {
    const int rows = q.rows, cols = q.cols, size = std::min(rows, cols);
    std::vector<double> nu(cols), nd(cols);
    double maxn = 0.0;
    q.perm.resize(cols);
    q.hcoef.assign(size, 0.0);
    for (int k = 0; k < cols; ++k) {
        nd[k] = nu[k] = colnorm(&q.a[(size_t)k * rows], rows);
        maxn = std::max(maxn, nu[k]);
        q.perm[k] = k;
    }
    const double eps = 2.220446049250313e-16;
    const double thr = (maxn * eps) * (maxn * eps) / rows;
    const double dthr = std::sqrt(eps);
    q.nonzero = size;
    q.maxpivot = 0.0;
    for (int k = 0; k < size; ++k) {
        int big = k;
        for (int j = k + 1; j < cols; ++j)
            if (nu[j] > nu[big]) big = j;
        if (q.nonzero == size && nu[big] * nu[big] < thr * (rows - k)) q.nonzero = k;
        if (big != k) {
            for (int i = 0; i < rows; ++i)
                std::swap(q.a[(size_t)k * rows + i], q.a[(size_t)big * rows + i]);
            std::swap(nu[k], nu[big]);
            std::swap(nd[k], nd[big]);
            std::swap(q.perm[k], q.perm[big]);
        }
        double* v = &q.a[(size_t)k * rows + k];
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
            beta = std::sqrt(c0 * c0 + tail);
            if (c0 >= 0.0) beta = -beta;
            for (int i = 1; i < m; ++i) v[i] = v[i] / (c0 - beta);
            tau = (beta - c0) / beta;
        }
        v[0] = beta;
        q.hcoef[k] = tau;
        q.maxpivot = std::max(q.maxpivot, std::fabs(beta));
        for (int j = k + 1; j < cols; ++j) {
            double* c = &q.a[(size_t)j * rows + k];
            double w = c[0];
            for (int i = 1; i < m; ++i) w += v[i] * c[i];
            w *= tau;
            c[0] -= w;
            for (int i = 1; i < m; ++i) c[i] -= w * v[i];
        }
        for (int j = k + 1; j < cols; ++j) {
            if (nu[j] != 0.0) {
                double t = std::fabs(q.a[(size_t)j * rows + k]) / nu[j];
                t = (1.0 + t) * (1.0 - t);
                if (t < 0.0) t = 0.0;
                const double r = nu[j] / nd[j];
                if (t * r * r <= dthr) {
                    nd[j] = colnorm(&q.a[(size_t)j * rows + k + 1], rows - k - 1);
                    nu[j] = nd[j];
                } else {
                    nu[j] *= std::sqrt(t);
                }
            }
        }
    }
}

int cpqr_rank(const CpQr& q, double threshold) {
    const double pt = std::fabs(q.maxpivot) * threshold;
    int r = 0;
    for (int i = 0; i < q.nonzero; ++i) r += std::fabs(q.a[(size_t)i * q.rows + i]) > pt;
    return r;
}

void cpqr_solve(const CpQr& q, const double* b, double* x, std::vector<double>& w) {
    const int rows = q.rows, cols = q.cols, size = std::min(rows, cols);
    w.assign(b, b + rows);
    for (int k = 0; k < size; ++k) {
        const double* v = &q.a[(size_t)k * rows + k];
        double s = w[k];
        for (int i = 1; i < rows - k; ++i) s += v[i] * w[k + i];
        s *= q.hcoef[k];
        w[k] -= s;
        for (int i = 1; i < rows - k; ++i) w[k + i] -= s * v[i];
    }
    std::vector<double> c(cols, 0.0);
    for (int i = q.nonzero - 1; i >= 0; --i) {
        double s = w[i];
        for (int j = i + 1; j < q.nonzero; ++j) s -= q.a[(size_t)j * rows + i] * c[j];
        c[i] = s / q.a[(size_t)i * rows + i];
    }
    for (int i = 0; i < cols; ++i) x[q.perm[i]] = c[i];
}

// The solve operator of a full-rank design as a [cols][S] matrix.
void solve_matrix(const CpQr& q, double* M /* [3 or 4][S] */, int mrows) {
    const int S = q.rows;
    std::vector<double> e(S, 0.0), x(q.cols), w;
    for (int s = 0; s < S; ++s) {
        e[s] = 1.0;
        cpqr_solve(q, e.data(), x.data(), w);
        e[s] = 0.0;
        for (int j = 0; j < mrows; ++j) M[(size_t)j * S + s] = j < q.cols ? x[j] : 0.0;
    }
}

// ---------------------------------------------------------------------------
// Device: one thread per kernel.
struct FitDev {
    int S, ncut;          // samples per kernel, ordered split candidates (1 + unique ratios)
    const double* cfg;    // [S][3] vc, fc, fm
    const double* ifm;    // [S] 1/fm
    const double* ifc;    // [S] 1/fc
    const double* ratio;  // [S] ifm/ifc (= fc/fm)
    const double* cuts;   // [ncut] split values (ordered[0] = +inf)
    const int* cmeta;     // [ncut] bit0 solvable, bit1 any_mem, bit2 any_core
    const double* Mt;     // [ncut][3][S] time solve operators (t0, alpha, beta rows)
    const double* Mp;     // [4][S] power solve operator
    int pstatus_all;      // S < 4: RankDeficient for every kernel (checked first)
    int prank_bad;        // design rank < 4: RankDeficient after the positivity check
    int tstatus_all;      // S < 3: Underdetermined
};

constexpr int kFitBlock = 128;

__device__ __forceinline__ double dmax_ref(double a, double b) { return (a < b) ? b : a; }

__global__ void __launch_bounds__(kFitBlock) fit_kernel(FitDev F, const double* __restrict__ power,
                                                        const double* __restrict__ tm, int64_t n,
                                                        int64_t ld, double* __restrict__ pfit,
                                                        int32_t* __restrict__ pst,
                                                        double* __restrict__ tfit,
                                                        int32_t* __restrict__ tst) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int S = F.S;
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    // ---- fit_power (param_fit.cpp:43-77) ---------------------------------------------
    if (power) {
        int st = F.pstatus_all;
        if (st == 0)
            for (int s = 0; s < S; ++s)
                if (!(power[(int64_t)s * ld + k] > 0.0)) {
                    st = kInvalidArgument;
                    break;
                }
        if (st == 0 && F.prank_bad) st = kRankDeficient;  // QR rank after positivity (":62")
        double c[4] = {0, 0, 0, 0};
        double mape = 0.0;
        int active = 0;
        if (st == 0) {
            for (int s = 0; s < S; ++s) {
                const double y = power[(int64_t)s * ld + k];
#pragma unroll
                for (int j = 0; j < 4; ++j) c[j] = fma(F.Mp[(size_t)j * S + s], y, c[j]);
            }
#pragma unroll
            for (int j = 0; j < 4; ++j)
                if (c[j] < 0.0) {
                    c[j] = 0.0;
                    active = 1;
                }
            double acc = 0.0;
            for (int s = 0; s < S; ++s) {
                const double vc = F.cfg[3 * s], fc = F.cfg[3 * s + 1], fm = F.cfg[3 * s + 2];
                const double pred = __dadd_rn(
                    __dadd_rn(__dadd_rn(c[0], __dmul_rn(c[1], vc)), __dmul_rn(c[2], fm)),
                    __dmul_rn(c[3], __dmul_rn(__dmul_rn(vc, vc), fc)));
                const double y = power[(int64_t)s * ld + k];
                acc += fabs(pred - y) / fabs(y);
            }
            mape = 100.0 * acc / S;
        }
        if (pfit) {
#pragma unroll
            for (int j = 0; j < 4; ++j) pfit[(int64_t)j * ld + k] = c[j];
            pfit[4 * ld + k] = mape;
            pfit[5 * ld + k] = active;
        }
        if (pst) pst[k] = st;
    }
    // ---- fit_time (param_fit.cpp:79-247) ----------------------------------------------
    if (tm) {
        int st = F.tstatus_all;
        double ysq = 0.0;
        if (st == 0)
            for (int s = 0; s < S; ++s) {
                const double y = tm[(int64_t)s * ld + k];
                if (!(y > 0.0)) {
                    st = kInvalidArgument;
                    break;
                }
                ysq += y * y;
            }
        double out[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        // coefficients of split c (the solve operator applied to this kernel's times)
        auto coef = [&](int c, double& t0, double& a, double& b) {
            const double* M = F.Mt + (size_t)c * 3 * S;
            t0 = a = b = 0.0;
            for (int s = 0; s < S; ++s) {
                const double y = tm[(int64_t)s * ld + k];
                t0 = fma(M[s], y, t0);
                a = fma(M[S + s], y, a);
                b = fma(M[2 * S + s], y, b);
            }
        };
        auto rss_of = [&](double t0, double a, double b) {
            double r = 0.0;
            for (int s = 0; s < S; ++s) {
                const double pred = t0 + dmax_ref(a * F.ifm[s], b * F.ifc[s]);
                const double y = tm[(int64_t)s * ld + k];
                r += (pred - y) * (pred - y);
            }
            return r;
        };
        if (st == 0) {
            // ordered split search (":128-158"): strict improvement beyond the tie slack
            const double slack = 1e-12 * (ysq + 1.0);
            double best = kInf;
            int cur = 0;
            for (int c = 0; c < F.ncut; ++c) {
                double rss = kInf;
                const int meta = F.cmeta[c];
                if (meta & 1) {
                    double t0, a, b;
                    coef(c, t0, a, b);
                    a = (meta & 2) ? dmax_ref(a, 0.0) : 0.0;
                    b = (meta & 4) ? dmax_ref(b, 0.0) : 0.0;
                    rss = rss_of(t0, a, b);
                }
                if (rss < best - slack) {
                    best = rss;
                    cur = c;
                }
            }
            if (!(fabs(best) < kInf)) st = kUnderdetermined;
            double t0 = 0.0, a = 0.0, b = 0.0, rss = 0.0;
            int iters = 0, active = 0;
            for (int it = 0; st == 0 && it < 50; ++it) {
                ++iters;
                const int meta = F.cmeta[cur];
                if (!(meta & 1)) {  // solve_full_rank throws (":183")
                    st = kUnderdetermined;
                    break;
                }
                coef(cur, t0, a, b);
                if (!(meta & 2)) a = 0.0;
                if (!(meta & 4)) b = 0.0;
                active = 0;
                if (a < 0.0) {
                    a = 0.0;
                    active = 1;
                }
                if (b < 0.0) {
                    b = 0.0;
                    active = 1;
                }
                rss = rss_of(t0, a, b);
                // reassignment (":211-219"): memory iff a/fm >= b/fc; as a split of the
                // ratios it is "ratio >= smallest memory ratio" (rounding-level
                // non-monotone assignments take the split with the same memory count)
                int nmem = 0;
                double rmin = kInf;
                for (int s = 0; s < S; ++s)
                    if (a * F.ifm[s] >= b * F.ifc[s]) {
                        ++nmem;
                        rmin = fmin(rmin, F.ratio[s]);
                    }
                int next;
                if (nmem == 0) {
                    next = 0;
                } else {
                    next = 1;
                    for (int c = 1; c < F.ncut; ++c)
                        if (F.cuts[c] <= rmin) next = c;
                }
                if (next == cur) break;
                cur = next;
            }
            if (st == 0) {
                const int meta = F.cmeta[cur];
                const bool all_mem = (meta & 2) && !(meta & 4);
                const bool all_core = !(meta & 2);
                const bool partial = all_mem || all_core;
                if (t0 < 0.0) {
                    t0 = 0.0;
                    active = 1;
                }
                if (partial) {
                    if (all_mem)
                        b = 0.0;
                    else
                        a = 0.0;
                }
                double acc = 0.0;
                for (int s = 0; s < S; ++s) {
                    const double pred = t0 + dmax_ref(a * F.ifm[s], b * F.ifc[s]);
                    const double y = tm[(int64_t)s * ld + k];
                    acc += fabs(pred - y) / fabs(y);
                }
                out[0] = t0;
                out[1] = a;
                out[2] = b;
                out[3] = 100.0 * acc / S;
                out[4] = active;
                out[5] = partial;
                out[6] = iters;
                out[7] = rss;
            }
        }
        if (tfit)
#pragma unroll
            for (int j = 0; j < 8; ++j) tfit[(int64_t)j * ld + k] = out[j];
        if (tst) tst[k] = st;
    }
}

}  // namespace

// Host side: factor the shared designs (cached per context for the same grid).
struct FitPlan {
    std::vector<double> cfg;
    int S = 0, ncut = 0;
    int pstatus_all = 0, prank_bad = 0, tstatus_all = 0;
    double* dev = nullptr;  // cfg | ifm | ifc | ratio | cuts | Mp | Mt (doubles) then cmeta (int)
    size_t dev_bytes = 0;
    FitDev fd{};
};

static FitPlan* plan_of(Ctx& cx) { return reinterpret_cast<FitPlan*>(cx.fit_plan); }

void fit_plan_free(Ctx& cx) {
    FitPlan* p = plan_of(cx);
    if (!p) return;
    cudaFree(p->dev);
    delete p;
    cx.fit_plan = nullptr;
}

cudaError_t fit_prepare(Ctx& cx, const double* cfg, int S) {
    FitPlan* p = plan_of(cx);
    if (p && p->S == S && std::memcmp(p->cfg.data(), cfg, sizeof(double) * 3 * S) == 0)
        return cudaSuccess;
    fit_plan_free(cx);
    p = new FitPlan();
    cx.fit_plan = p;
    p->S = S;
    p->cfg.assign(cfg, cfg + 3 * S);
    std::vector<double> ifm(S), ifc(S), ratio(S);
    for (int s = 0; s < S; ++s) {
        ifm[s] = 1.0 / cfg[3 * s + 2];  // param_fit.cpp:93-94
        ifc[s] = 1.0 / cfg[3 * s + 1];
        ratio[s] = ifm[s] / ifc[s];     // ":131"
    }
    // fit_power design and operator
    std::vector<double> Mp(4 * (size_t)S, 0.0);
    if (S < 4) {
        p->pstatus_all = kRankDeficient;
    } else {
        CpQr q;
        q.rows = S;
        q.cols = 4;
        q.a.resize(4 * (size_t)S);
        for (int s = 0; s < S; ++s) {
            const double vc = cfg[3 * s], fc = cfg[3 * s + 1], fm = cfg[3 * s + 2];
            q.a[s] = 1.0;
            q.a[S + s] = vc;
            q.a[2 * S + s] = fm;
            q.a[3 * S + s] = vc * vc * fc;
        }
        cpqr_compute(q);
        if (cpqr_rank(q, 1e-10) < 4)
            p->prank_bad = 1;
        else
            solve_matrix(q, Mp.data(), 4);
    }
    // fit_time: ordered splits (":133-145"): +inf (all core), then the unique ratios
    std::vector<double> cuts(ratio);
    std::sort(cuts.begin(), cuts.end());
    cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
    std::vector<double> ordered;
    ordered.push_back(HUGE_VAL);
    for (double c : cuts) ordered.push_back(c);
    const int ncut = S >= 3 ? (int)ordered.size() : 0;
    p->ncut = ncut;
    p->tstatus_all = S < 3 ? kUnderdetermined : 0;
    std::vector<double> Mt(3 * (size_t)S * ncut, 0.0);
    std::vector<int> meta(ncut > 0 ? ncut : 1, 0);
    for (int c = 0; c < ncut; ++c) {
        bool any_mem = false, any_core = false;
        std::vector<char> mem(S);
        for (int s = 0; s < S; ++s) {
            mem[s] = ratio[s] >= ordered[c];
            (mem[s] ? any_mem : any_core) = true;
        }
        const int cols = 1 + (any_mem ? 1 : 0) + (any_core ? 1 : 0);
        const int mc = any_mem ? 1 : -1, cc = any_core ? (any_mem ? 2 : 1) : -1;
        CpQr q;
        q.rows = S;
        q.cols = cols;
        q.a.assign((size_t)cols * S, 0.0);
        for (int s = 0; s < S; ++s) {
            q.a[s] = 1.0;
            if (mem[s])
                q.a[(size_t)mc * S + s] = ifm[s];
            else
                q.a[(size_t)cc * S + s] = ifc[s];
        }
        cpqr_compute(q);
        const bool ok = cpqr_rank(q, 1e-10) >= cols;
        meta[c] = (ok ? 1 : 0) | (any_mem ? 2 : 0) | (any_core ? 4 : 0);
        if (ok) {
            std::vector<double> M((size_t)cols * S);
            solve_matrix(q, M.data(), cols);
            double* dst = &Mt[(size_t)c * 3 * S];
            for (int s = 0; s < S; ++s) {
                dst[s] = M[s];                                           // t0
                if (any_mem) dst[S + s] = M[(size_t)mc * S + s];         // alpha
                if (any_core) dst[2 * S + s] = M[(size_t)cc * S + s];    // beta
            }
        }
    }
    // upload
    const size_t nd = 3 * (size_t)S + 3 * (size_t)S + (size_t)ordered.size() + Mp.size() + Mt.size();
    const size_t bytes = nd * sizeof(double) + meta.size() * sizeof(int) + 64;
    cudaError_t e = cudaMalloc(&p->dev, bytes);
    if (e != cudaSuccess) return e;
    p->dev_bytes = bytes;
    double* d = p->dev;
    auto put = [&](const double* src, size_t cnt) {
        double* at = d;
        cudaMemcpy(at, src, cnt * sizeof(double), cudaMemcpyHostToDevice);
        d += cnt;
        return at;
    };
    p->fd.S = S;
    p->fd.ncut = ncut;
    p->fd.cfg = put(cfg, 3 * (size_t)S);
    p->fd.ifm = put(ifm.data(), S);
    p->fd.ifc = put(ifc.data(), S);
    p->fd.ratio = put(ratio.data(), S);
    p->fd.cuts = put(ordered.data(), ordered.size());
    p->fd.Mp = put(Mp.data(), Mp.size());
    p->fd.Mt = put(Mt.data(), Mt.size());
    int* mi = reinterpret_cast<int*>(d);
    cudaMemcpy(mi, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice);
    p->fd.cmeta = mi;
    p->fd.pstatus_all = p->pstatus_all;
    p->fd.prank_bad = p->prank_bad;
    p->fd.tstatus_all = p->tstatus_all;
    return cudaGetLastError();
}

cudaError_t launch_param_fit(Ctx& cx, const double* power, const double* tm, int64_t n,
                             int64_t ld, double* pfit, int32_t* pst, double* tfit, int32_t* tst) {
    if (n <= 0) return cudaSuccess;
    FitPlan* p = plan_of(cx);
    const int64_t blocks = (n + kFitBlock - 1) / kFitBlock;
    fit_kernel<<<(unsigned)blocks, kFitBlock, 0, cx.stream>>>(p->fd, power, tm, n, ld, pfit, pst,
                                                            tfit, tst);
    ++cx.launches;
    return cudaGetLastError();
}

}  // namespace dso_b200
