// opt.cu — optimal_config for a batch of kernels (sm_100a), FP64, bit-exact.
//
// Replaces dso::optimal_config (reference proj/src/optimizer.cpp:119-205,
// declared optimizer.hpp:39-46): the structured Theorem-1 search over the
// induced voltage levels that the CLI and run_campaign call.  Per level i
// (one per core clock):
//   g1      = to_mhz(max_core_freq(vc_i))                (optimizer.cpp:141-142)
//   target  = min(g1, knee),  knee = alpha > 0 ? (beta/alpha)*fm_max : inf
//   fc_base = snap_down(cores, target)  (skip the level if -1)
//   for fc_idx in fc_base-1..fc_base+1, fm_base = snap_up(mems, (alpha/beta)*fc)
//     (last level if -1; 0 when beta == 0), for fm_idx in fm_base-1..fm_base+1:
//       evaluate, ++evaluated, keep if better() (cost, energy, vc, fm)
// then the fallback to brute_force_config when no level produced a candidate,
// and presnap_{vc,fc,fm} from the winning level (optimizer.cpp:188-203).
//
// The domain-only terms (vc_i, g1_i, snap_down(cores, g1_i)) are computed once
// on the host in double with the reference's expressions (abi.cu).  Per
// kernel, a candidate (fc_idx, fm_idx) seen at an earlier level can never be
// strictly better than the state it already produced, so each distinct
// candidate is evaluated once (fc_base is non-decreasing in the level, so
// "seen" is fc_idx <= the previous level's fc_base + 1); evaluated still
// counts every visit like the reference.  All arithmetic is explicit
// round-to-nearest FP64 in the reference's operation order (no contraction),
// so every output is bit-identical to the reference's.
#include <math.h>

#include "common.cuh"

namespace dso_b200 {

namespace {

constexpr int kBlock = 128;

struct Cand {
    double cost, energy, time, vc, fm;
    int fc_idx, fm_idx;
};

// better() (optimizer.cpp:27-32): cost, energy, vc, fm — all ascending.
__device__ __forceinline__ bool better(const Cand& a, const Cand& b) {
    if (a.cost != b.cost) return a.cost < b.cost;
    if (a.energy != b.energy) return a.energy < b.energy;
    if (a.vc != b.vc) return a.vc < b.vc;
    return a.fm < b.fm;
}

struct P64 {
    double p0, kp, g, c, t0, a, b;
};

// evaluate() (optimizer.cpp:34-39) with power/exec_time/energy/cost of
// dvfs_model.hpp:81-104, operation by operation.
__device__ __forceinline__ Cand evaluate(const P64& p, double vc, double fc, double fm,
                                         double eta, double K) {
    const double P = __dadd_rn(__dadd_rn(__dadd_rn(p.p0, __dmul_rn(p.kp, vc)), __dmul_rn(p.g, fm)),
                               __dmul_rn(__dmul_rn(__dmul_rn(p.c, vc), vc), fc));
    const double ta = __ddiv_rn(p.a, fm), tb = __ddiv_rn(p.b, fc);
    const double T = __dadd_rn(p.t0, (ta < tb) ? tb : ta);  // std::max
    Cand r;
    r.cost = __dmul_rn(__dadd_rn(__dmul_rn(eta, P), K), T);
    r.energy = __dmul_rn(P, T);
    r.time = T;
    r.vc = vc;
    r.fm = fm;
    return r;
}

__global__ void __launch_bounds__(kBlock) optimal_config_kernel(
    const double* __restrict__ params, int64_t n, const double2* __restrict__ core_d,
    const double* __restrict__ g1_d, const int* __restrict__ sd_g1, int nc,
    const double* __restrict__ mem_d, int nm, double eta, double K, double up, double down,
    int32_t* __restrict__ idx_out, double* __restrict__ cost_out, double* __restrict__ energy_out,
    double* __restrict__ time_out, int64_t* __restrict__ cand_out, uint8_t* __restrict__ fb_out,
    double* __restrict__ presnap_out, int32_t* __restrict__ kstatus) {
    __shared__ double2 s_core[kMaxCore];  // {vc, fc}
    __shared__ double s_g1[kMaxCore];
    __shared__ int s_sd[kMaxCore];
    __shared__ double s_mem[kMaxMem];
    for (int i = threadIdx.x; i < nc; i += blockDim.x) {
        s_core[i] = core_d[i];
        s_g1[i] = g1_d[i];
        s_sd[i] = sd_g1[i];
    }
    for (int j = threadIdx.x; j < nm; j += blockDim.x) s_mem[j] = mem_d[j];
    __syncthreads();
    const double kInf = __longlong_as_double(0x7ff0000000000000LL);
    const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        const double* q = params + 7 * k;
        const P64 p{q[0], q[1], q[2], q[3], q[4], q[5], q[6]};
        if (p.p0 < 0.0 || p.kp < 0.0 || p.g < 0.0 || p.c < 0.0 || p.t0 < 0.0 || p.a < 0.0 ||
            p.b < 0.0 || !(__dadd_rn(p.a, p.b) > 0.0)) {  // validate(params), dvfs_model.hpp:50-58
            idx_out[k] = -1;
            if (cost_out) cost_out[k] = kNaN;
            if (energy_out) energy_out[k] = kNaN;
            if (time_out) time_out[k] = kNaN;
            if (cand_out) cand_out[k] = 0;
            if (fb_out) fb_out[k] = 0;
            if (presnap_out) presnap_out[3 * k] = presnap_out[3 * k + 1] = presnap_out[3 * k + 2] = 0.0;
            if (kstatus) kstatus[k] = kInvalidArgument;
            continue;
        }
        const double fm_max = s_mem[nm - 1], fm_min = s_mem[0];
        const double knee = p.a > 0.0 ? __dmul_rn(__ddiv_rn(p.b, p.a), fm_max) : kInf;
        // snap_down(cores, knee) for the levels whose g1 exceeds the knee
        int sd_knee = -1;
        {
            const double x = __dmul_rn(knee, up);
            for (int j = 0; j < nc; ++j)
                if (s_core[j].y <= x) sd_knee = j;
        }
        const double ab = p.b > 0.0 ? __ddiv_rn(p.a, p.b) : 0.0;
        bool have = false;
        Cand best{};
        int best_level = -1;
        int64_t evaluated = 0;
        int prev_base = -3;  // fc_base of the previous level with candidates
        for (int i = 0; i < nc; ++i) {
            const double g1 = s_g1[i];
            const bool capped = knee < g1;  // std::min(g1, knee) picks the knee
            const int base = capped ? sd_knee : s_sd[i];
            if (base < 0) continue;
            for (int dfc = -1; dfc <= 1; ++dfc) {
                const int fi = base + dfc;
                if (fi < 0 || fi >= nc) continue;
                const double fc = s_core[fi].y;
                int fm_base;
                if (p.b > 0.0) {
                    const double x = __dmul_rn(__dmul_rn(ab, fc), down);
                    fm_base = -1;
                    for (int j = 0; j < nm; ++j)
                        if (s_mem[j] >= x) {
                            fm_base = j;
                            break;
                        }
                    if (fm_base < 0) fm_base = nm - 1;
                } else {
                    fm_base = 0;
                }
                const int jlo = fm_base > 0 ? fm_base - 1 : 0;
                const int jhi = fm_base + 1 < nm ? fm_base + 1 : nm - 1;
                evaluated += jhi - jlo + 1;
                if (fi <= prev_base + 1) continue;  // seen at an earlier level
                for (int fj = jlo; fj <= jhi; ++fj) {
                    Cand c = evaluate(p, s_core[fi].x, fc, s_mem[fj], eta, K);
                    c.fc_idx = fi;
                    c.fm_idx = fj;
                    if (!have || better(c, best)) {
                        best = c;
                        have = true;
                        best_level = i;
                    }
                }
            }
            prev_base = base;
        }
        bool fallback = false;
        if (!have) {
            // brute_force_config (optimizer.cpp:90-117), flagged
            fallback = true;
            evaluated = (int64_t)nc * nm;
            for (int fi = 0; fi < nc; ++fi)
                for (int fj = 0; fj < nm; ++fj) {
                    Cand c = evaluate(p, s_core[fi].x, s_core[fi].y, s_mem[fj], eta, K);
                    c.fc_idx = fi;
                    c.fm_idx = fj;
                    if (!have || better(c, best)) {
                        best = c;
                        have = true;
                    }
                }
        }
        idx_out[k] = best.fc_idx * nm + best.fm_idx;
        if (cost_out) cost_out[k] = best.cost;
        if (energy_out) energy_out[k] = best.energy;
        if (time_out) time_out[k] = best.time;
        if (cand_out) cand_out[k] = evaluated;
        if (fb_out) fb_out[k] = fallback ? 1 : 0;
        if (presnap_out) {
            double pv = 0.0, pf = 0.0, pm = 0.0;
            if (!fallback) {
                // optimizer.cpp:196-203 (g1 of the winning level == s_g1[best_level])
                const double g1w = s_g1[best_level];
                const double fcc = (knee < g1w) ? knee : g1w;
                double fmc = fm_min;
                if (p.b > 0.0) {
                    const double x = __dmul_rn(ab, fcc);
                    fmc = (fm_min < x) ? x : fm_min;  // std::max(fm_min, x)
                }
                pv = s_core[best_level].x;
                pf = fcc;
                pm = fmc;
            }
            presnap_out[3 * k] = pv;
            presnap_out[3 * k + 1] = pf;
            presnap_out[3 * k + 2] = pm;
        }
        if (kstatus) kstatus[k] = 0;
    }
}

}  // namespace

cudaError_t launch_optimal_config(Ctx& cx, const double* params, int64_t n, double eta,
                                  double K, int32_t* idx, double* cost, double* energy,
                                  double* time, int64_t* candidates, uint8_t* fallback,
                                  double* presnap, int32_t* kstatus) {
    if (n <= 0) return cudaSuccess;
    const int grid = grid_for(n, kBlock, cx.num_sms, 8);
    const DomainDev& d = cx.dom;
    optimal_config_kernel<<<grid, kBlock, 0, cx.stream>>>(
        params, n, d.core_d, d.g1_d, d.sd_g1, d.nc, d.mem_d, d.nm, eta, K, 1.0 + 1e-12,
        1.0 - 1e-12, idx, cost, energy, time, candidates, fallback, presnap, kstatus);
    ++cx.launches;
    return cudaGetLastError();
}

}  // namespace dso_b200
