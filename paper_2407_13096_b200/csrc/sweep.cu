// sweep.cu — grid sweep + eta objective + lexicographic argmin (sm_100a).
//
// Replaces brute_force_config (reference proj/src/optimizer.cpp:90-117) for a
// batch of kernels.  Reference semantics kept exactly:
//   * pairs visited fc-outer / fm-inner (optimizer.cpp:99-100), idx = i*nm + j;
//   * better() (optimizer.cpp:27-32): cost, then energy, then vc (strictly
//     increasing in i), then fm — in visit order that is
//     (C < bc) || (C == bc && E < be), keeping the earlier pair otherwise;
//   * P = p0 + kp*vc + g*fm + c*vc^2*fc, T = t0 + max(a/fm, b/fc),
//     C = (eta*P + (1-eta)*pmax)*T, E = P*T (dvfs_model.hpp:81-104);
//   * validate(params) (dvfs_model.hpp:50-58) per kernel -> kstatus.
// The first pair seeds the running best unconditionally, as have_best does
// (optimizer.cpp:96-106), so NaN/inf semantics match too.
//
// Work mapping: one thread per kernel, the per-domain tables in shared memory
// (uniform across the warp -> broadcast LDS), per-kernel terms hoisted out of
// the pair loop:  per fc level Pc = p0 + kp*vc + c*vc^2*fc and Tb = b/fc; per
// fm level G = g*fm and Ta = a/fm.  Per pair: FADD, FMNMX, FADD, FFMA, FMUL,
// FMUL + the comparator.  Issue-bound on the FP32/ALU pipes; no HBM pressure
// (28 B in, 16 B out per kernel for nc*nm pairs).
#include <math.h>

#include <type_traits>

#include "common.cuh"
#include "sweep_core.cuh"

namespace dso_b200 {

namespace {

constexpr int kBlock = 256;
#ifndef DSO_ETA_CH
#define DSO_ETA_CH 26
#endif
#ifndef DSO_ETA_GROUP_UNROLL
#define DSO_ETA_GROUP_UNROLL 1
#endif
#ifndef DSO_ETA_PRUNE_MINB
#define DSO_ETA_PRUNE_MINB 4
#endif
#ifndef DSO_ETA_PRUNE_CH
#define DSO_ETA_PRUNE_CH 34
#endif
constexpr int kEtaGroupUnroll = DSO_ETA_GROUP_UNROLL;  // eta-sweep groups per unrolled step

__device__ __forceinline__ bool params_invalid(float p0, float kp, float g, float c, float t0,
                                               float a, float b) {
    // dvfs_model.hpp:51-57 (NaN passes the >= 0 tests there too; a NaN in
    // alpha or beta fails alpha + beta > 0)
    return p0 < 0.f || kp < 0.f || g < 0.f || c < 0.f || t0 < 0.f || a < 0.f || b < 0.f ||
           !(a + b > 0.f);
}

template <int NM>
__global__ void __launch_bounds__(kBlock) sweep_f32_kernel(
    const float* __restrict__ params, int64_t n, int64_t ld, const float4* __restrict__ core4,
    int nc, const float2* __restrict__ mem2, int nm_rt, float eta, float K,
    int32_t* __restrict__ idx, float* __restrict__ cost, float* __restrict__ energy,
    float* __restrict__ time, int32_t* __restrict__ kstatus, bool fast) {
    __shared__ float4 s_core[kMaxCore];
    __shared__ float4 s_pair[kMaxCore + 2];
    __shared__ float2 s_mem[kMaxMem];
    const int nm = NM > 0 ? NM : nm_rt;
    for (int i = threadIdx.x; i < nc; i += blockDim.x) s_core[i] = core4[i];
    for (int j = threadIdx.x; j < nm; j += blockDim.x) s_mem[j] = mem2[j];
    build_pairs(s_pair, core4, nc);
    __syncthreads();

    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        KParams p;
        p.p0 = __ldg(params + k);
        p.kp = __ldg(params + ld + k);
        p.g = __ldg(params + 2 * ld + k);
        p.c = __ldg(params + 3 * ld + k);
        p.t0 = __ldg(params + 4 * ld + k);
        p.a = __ldg(params + 5 * ld + k);
        p.b = __ldg(params + 6 * ld + k);
        if (params_invalid(p.p0, p.kp, p.g, p.c, p.t0, p.a, p.b)) {
            idx[k] = -1;
            if (cost) cost[k] = __int_as_float(0x7fc00000);
            if (energy) energy[k] = __int_as_float(0x7fc00000);
            if (time) time[k] = __int_as_float(0x7fc00000);
            if (kstatus) kstatus[k] = kInvalidArgument;
            continue;
        }
        const Best b = sweep_best<NM>(p, s_core, s_mem, nm, 0, nc, eta, K, fast, s_pair);
        idx[k] = b.i;
        if (cost) cost[k] = b.c;
        if (energy) energy[k] = b.e;
        if (time) time[k] = time_at(p, s_core, s_mem, nm, b.i);
        if (kstatus) kstatus[k] = 0;
    }
}

// ---- exact FP64 variant -------------------------------------------------------
// Same arithmetic as the reference, operation by operation, with explicit
// round-to-nearest intrinsics so nothing is contracted into an FMA:
//   power    ((p0 + kp*vc) + g*fm) + ((c*vc)*vc)*fc      dvfs_model.hpp:82-83
//   time     t0 + ((a/fm < b/fc) ? b/fc : a/fm)          dvfs_model.hpp:89 (std::max)
//   cost     (eta*P + (1-eta)*pmax) * T                   dvfs_model.hpp:103
//   energy   P * T                                        dvfs_model.hpp:94
// vc per level is computed on the host by required_voltage_mhz's expression.
// Hoisting (p0 + kp*vc), ((c*vc)*vc)*fc, b/fc and a/fm out of the pair loop
// does not change any rounding: each is a complete sub-expression.
__global__ void __launch_bounds__(kBlock) sweep_f64_kernel(
    const double* __restrict__ params, int64_t n, const double2* __restrict__ core_d, int nc,
    const double* __restrict__ mem_d, int nm, double eta, double K, int32_t* __restrict__ idx,
    double* __restrict__ cost, double* __restrict__ energy, double* __restrict__ time,
    int32_t* __restrict__ kstatus) {
    __shared__ double2 s_core[kMaxCore];
    __shared__ double s_mem[kMaxMem];
    for (int i = threadIdx.x; i < nc; i += blockDim.x) s_core[i] = core_d[i];
    for (int j = threadIdx.x; j < nm; j += blockDim.x) s_mem[j] = mem_d[j];
    __syncthreads();
    const double kNaN = __longlong_as_double(0x7ff8000000000000LL);
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        const double* p = params + 7 * k;
        const double p0 = p[0], kp = p[1], g = p[2], c = p[3], t0 = p[4], a = p[5], b = p[6];
        if (p0 < 0.0 || kp < 0.0 || g < 0.0 || c < 0.0 || t0 < 0.0 || a < 0.0 || b < 0.0 ||
            !(__dadd_rn(a, b) > 0.0)) {
            idx[k] = -1;
            if (cost) cost[k] = kNaN;
            if (energy) energy[k] = kNaN;
            if (time) time[k] = kNaN;
            if (kstatus) kstatus[k] = kInvalidArgument;
            continue;
        }
        double bc, be, bt;
        int bi = 0;
        {  // first candidate taken unconditionally (optimizer.cpp:103)
            const double vc = s_core[0].x, fc = s_core[0].y, fm = s_mem[0];
            const double P = __dadd_rn(
                __dadd_rn(__dadd_rn(p0, __dmul_rn(kp, vc)), __dmul_rn(g, fm)),
                __dmul_rn(__dmul_rn(__dmul_rn(c, vc), vc), fc));
            const double Ta = __ddiv_rn(a, fm), Tb = __ddiv_rn(b, fc);
            bt = __dadd_rn(t0, (Ta < Tb) ? Tb : Ta);
            bc = __dmul_rn(__dadd_rn(__dmul_rn(eta, P), K), bt);
            be = __dmul_rn(P, bt);
        }
        for (int i = 0; i < nc; ++i) {
            const double vc = s_core[i].x, fc = s_core[i].y;
            const double A = __dadd_rn(p0, __dmul_rn(kp, vc));
            const double W = __dmul_rn(__dmul_rn(__dmul_rn(c, vc), vc), fc);
            const double Tb = __ddiv_rn(b, fc);
            for (int j = 0; j < nm; ++j) {
                const double fm = s_mem[j];
                const double P = __dadd_rn(__dadd_rn(A, __dmul_rn(g, fm)), W);
                const double Ta = __ddiv_rn(a, fm);
                const double T = __dadd_rn(t0, (Ta < Tb) ? Tb : Ta);
                const double C = __dmul_rn(__dadd_rn(__dmul_rn(eta, P), K), T);
                const double E = __dmul_rn(P, T);
                const bool better = (C < bc) | ((C == bc) & (E < be));
                if (better) {
                    bc = C;
                    be = E;
                    bt = T;
                    bi = i * nm + j;
                }
            }
        }
        idx[k] = bi;
        if (cost) cost[k] = bc;
        if (energy) energy[k] = be;
        if (time) time[k] = bt;
        if (kstatus) kstatus[k] = 0;
    }
}

// ---- eta sweep ------------------------------------------------------------------
// brute_force_config at n_eta objective weights in one pass over the grid.
// One thread owns one kernel and a chunk of CH etas (state: 3 registers per
// eta, the eta constants in registers).  P, T and E are computed once per pair
// and shared by the chunk; per (pair, eta) the objective is one FFMA + FMUL
// with the same rounding as sweep_f32_kernel, so each eta's argmin equals
// dso_sweep at that eta bit for bit.
template <int CH>
__global__ void __launch_bounds__(128) eta_sweep_kernel(
    const float* __restrict__ params, int64_t n, int64_t ld, const float4* __restrict__ core4,
    int nc, const float2* __restrict__ mem2, int nm, const float2* __restrict__ etaK, int n_eta, int32_t* __restrict__ idx, float* __restrict__ cost, int64_t ld_out) {
    __shared__ float4 s_core[kMaxCore];
    __shared__ float2 s_mem[kMaxMem];
    for (int i = threadIdx.x; i < nc; i += blockDim.x) s_core[i] = core4[i];
    for (int j = threadIdx.x; j < nm; j += blockDim.x) s_mem[j] = mem2[j];
    __syncthreads();
    const int chunk = blockIdx.y;
    const int e0 = chunk * CH;
    float ev[CH], Kv[CH];
#pragma unroll
    for (int e = 0; e < CH; ++e) {
        const int ee = e0 + e < n_eta ? e0 + e : n_eta - 1;
        ev[e] = etaK[ee].x;
        Kv[e] = etaK[ee].y;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        const float p0 = __ldg(params + k), kp = __ldg(params + ld + k),
                    g = __ldg(params + 2 * ld + k), c = __ldg(params + 3 * ld + k),
                    t0 = __ldg(params + 4 * ld + k), a = __ldg(params + 5 * ld + k),
                    b = __ldg(params + 6 * ld + k);
        if (params_invalid(p0, kp, g, c, t0, a, b)) {
#pragma unroll
            for (int e = 0; e < CH; ++e)
                if (e0 + e < n_eta) {
                    idx[(int64_t)(e0 + e) * ld_out + k] = -1;
                    if (cost) cost[(int64_t)(e0 + e) * ld_out + k] = __int_as_float(0x7fc00000);
                }
            continue;
        }
        float bc[CH], be[CH];
        int bi[CH];
        {  // first candidate taken unconditionally (optimizer.cpp:103)
            const float4 t = s_core[0];
            const float P = __fadd_rn(pc_f32(p0, kp, c, t), __fmul_rn(g, s_mem[0].x));
            const float T = time_f32(t0, __fmul_rn(a, s_mem[0].y), __fmul_rn(b, t.z));
#pragma unroll
            for (int e = 0; e < CH; ++e) {
                bc[e] = cost_f32(ev[e], Kv[e], P, T);
                be[e] = __fmul_rn(P, T);
                bi[e] = 0;
            }
        }
        for (int i = 0; i < nc; ++i) {
            const float4 t = s_core[i];
            const float Pc = pc_f32(p0, kp, c, t);
            const float Tb = __fmul_rn(b, t.z);
            for (int j = 0; j < nm; ++j) {
                const float2 m = s_mem[j];
                const float P = __fadd_rn(Pc, __fmul_rn(g, m.x));
                const float T = time_f32(t0, __fmul_rn(a, m.y), Tb);
                const float E = __fmul_rn(P, T);
                const int id = i * nm + j;
#pragma unroll
                for (int e = 0; e < CH; ++e) {
                    const float C = cost_f32(ev[e], Kv[e], P, T);
                    const bool better = (C < bc[e]) | ((C == bc[e]) & (E < be[e]));
                    bc[e] = better ? C : bc[e];
                    be[e] = better ? E : be[e];
                    bi[e] = better ? id : bi[e];
                }
            }
        }
#pragma unroll
        for (int e = 0; e < CH; ++e)
            if (e0 + e < n_eta) {
                idx[(int64_t)(e0 + e) * ld_out + k] = bi[e];
                if (cost) cost[(int64_t)(e0 + e) * ld_out + k] = bc[e];
            }
    }
}

// Fast exact eta sweep (NM = 1..4): per group of 8 pairs, P and T are formed
// once and shared by the chunk's CH etas; per eta the group costs take 8
// packed FFMA2/FMUL2 and a min tree, and the running minimum keeps the first
// group attaining it (sweep_best's scheme, sweep_core.cuh).  Afterwards each
// eta's winning group is replayed with the lexicographic rule; an eta whose
// minimum was reached by two groups (its bit in `ties`) is rescanned in full.
// Every eta's (idx, cost) therefore equals dso_sweep's at that eta, bit for bit.
// Out of line so the unrolled per-eta calls keep the eta state in registers.
template <int NM>
__device__ __noinline__ Best replay_levels(const KParams p, const float4* s_core,
                                           const float2* s_mem, int lo, int hi, float eta,
                                           float K) {
    return sweep_levels<NM>(p, s_core, s_mem, NM, lo, hi, eta, K);
}

template <int CH, int NM>
__global__ void __launch_bounds__(128) eta_sweep_fast_kernel(
    const float* __restrict__ params, int64_t n, int64_t ld, const float4* __restrict__ core4,
    int nc, const float2* __restrict__ mem2, const float2* __restrict__ etaK, int n_eta,
    int32_t* __restrict__ idx, float* __restrict__ cost, int64_t ld_out) {
    static_assert(CH <= 32, "tie bits");
    constexpr int GL = FastGroup<NM>::GL;
    constexpr int GH = GL * NM / 2;
    __shared__ float4 s_core[kMaxCore];
    __shared__ float4 s_pair[kMaxCore + 2];
    __shared__ float2 s_mem[NM];
    for (int i = threadIdx.x; i < nc; i += blockDim.x) s_core[i] = core4[i];
    if (threadIdx.x < NM) s_mem[threadIdx.x] = mem2[threadIdx.x];
    build_pairs(s_pair, core4, nc);
    __syncthreads();
    const int e0 = blockIdx.y * CH;
    float ev[CH], Kv[CH];
#pragma unroll
    for (int e = 0; e < CH; ++e) {
        const int ee = e0 + e < n_eta ? e0 + e : n_eta - 1;
        ev[e] = etaK[ee].x;
        Kv[e] = etaK[ee].y;
    }
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        KParams p;
        p.p0 = __ldg(params + k);
        p.kp = __ldg(params + ld + k);
        p.g = __ldg(params + 2 * ld + k);
        p.c = __ldg(params + 3 * ld + k);
        p.t0 = __ldg(params + 4 * ld + k);
        p.a = __ldg(params + 5 * ld + k);
        p.b = __ldg(params + 6 * ld + k);
        if (params_invalid(p.p0, p.kp, p.g, p.c, p.t0, p.a, p.b)) {
#pragma unroll
            for (int e = 0; e < CH; ++e)
                if (e0 + e < n_eta) {
                    idx[(int64_t)(e0 + e) * ld_out + k] = -1;
                    if (cost) cost[(int64_t)(e0 + e) * ld_out + k] = __int_as_float(0x7fc00000);
                }
            continue;
        }
        const bool fast = params_fast(p);
        float bc[CH];
        int bg[CH];
        uint32_t ties = fast ? 0u : 0xffffffffu;
#pragma unroll
        for (int e = 0; e < CH; ++e) {
            bc[e] = __int_as_float(0x7f800000);
            bg[e] = 0;
        }
        if (fast) {
            float G[NM], Ta1[NM];
#pragma unroll
            for (int j = 0; j < NM; ++j) {
                G[j] = __fmul_rn(p.g, s_mem[j].x);
                Ta1[j] = __fadd_rn(p.t0, __fmul_rn(p.a, s_mem[j].y));
            }
            auto group = [&](int i, auto tail) {
                float pc[GL], tb[GL];
                if constexpr (decltype(tail)::value)
                    group_levels<NM, true>(p, s_core, i, nc, pc, tb);
                else
                    group_levels_paired<NM>(p, s_pair, i, pc, tb);  // groups start at even i
                float2 P2[GH], T2[GH];
                group_pt<NM>(pc, tb, Ta1, G, P2, T2);
#pragma unroll
                for (int e = 0; e < CH; ++e) {
                    const float m = group_min_cost<NM>(P2, T2, ev[e], Kv[e]);
                    ties |= m == bc[e] ? 1u << e : 0u;
                    bg[e] = m < bc[e] ? i : bg[e];
                    bc[e] = fminf(m, bc[e]);
                }
            };
            int i = 0;
#pragma unroll kEtaGroupUnroll
            for (; i + GL <= nc; i += GL) group(i, std::false_type{});
            if (i < nc) group(i, std::true_type{});
        }
        // replay each eta's winning group (or, on a tie, every level) exactly
#pragma unroll
        for (int e = 0; e < CH; ++e) {
            if (e0 + e < n_eta) {
                const bool full = (ties >> e) & 1u;
                const int lo = full ? 0 : bg[e];
                const int hi = full ? nc : min(bg[e] + GL, nc);
                const Best b = replay_levels<NM>(p, s_core, s_mem, lo, hi, ev[e], Kv[e]);
                idx[(int64_t)(e0 + e) * ld_out + k] = b.i;
                if (cost) cost[(int64_t)(e0 + e) * ld_out + k] = b.c;
            }
        }
    }
}

// ---- Pruned exact eta sweep (NM = 2..4) ------------------------------------
//
// Preconditions (host: DomainDev::sorted_ok, every eta >= 0 and K >= 0; device:
// params_fast): along the core levels vc and vc^2 fc are non-decreasing and
// 1/fc non-increasing, along the memory levels fm is non-decreasing and 1/fm
// non-increasing.  With params >= 0 (validate(params)) every rounded quantity
// is then monotone: Pc_i and TB_i = t0 + b/fc_i along i (up / down), G_j = g fm_j
// and TA_j = t0 + a/fm_j along j (up / down), and C = (eta P + K) T, E = P T are
// non-decreasing in P and T (round-to-nearest is monotone; all operands >= 0).
//
// Every pair (i, j) has T = max(TA_j, TB_i), so it lies in
//   J_i = { j : TA_j <= TB_i }  (T = TB_i; a suffix of the memory levels) or
//   S_j = { i : TB_i <= TA_j }  (T = TA_j; a suffix of the core levels).
// Inside J_i the first member j0(i) has the least P and the same T as the others,
// hence C and E no larger, and it comes first in visit order: no other member of
// J_i can be strictly better than it (better(), optimizer.cpp:27-32), so none can
// be the scan's answer.  Likewise inside S_j for its first member i0(j).  The
// scan's answer is therefore among the candidates
//   (i, j0(i)) for every level i with J_i non-empty, and (i0(j), j) for every j
// with S_j non-empty: at most nc + NM points instead of nc * NM (132 of 512 on
// the 128 x 4 grids).  Over the candidates the group-minimum scheme of
// sweep_best runs unchanged (groups of 8 level candidates plus one group of the
// NM knee candidates; a minimum reached by two groups -> exact full rescan), and
// the winning group's candidates are replayed with the sequential rule: each
// eta's (idx, cost) equals dso_sweep's bit for bit.  A missing candidate is a
// NaN slot (FMNMX drops it; it never compares equal or smaller).
constexpr int kPruneL = 8;  // level candidates per group

// Candidates of the 8 levels i .. i+7 (clamped to nc-1: a repeated candidate is
// the same pair, so neither the group minimum nor the replay changes).
template <int NM, bool PAIRED>
__device__ __forceinline__ void prune_level_cands(const KParams& p,
                                                  const float4* __restrict__ s_core,
                                                  const float4* __restrict__ s_pair, int i,
                                                  int nc, const float* G, const float* TA,
                                                  float2* P2, float2* T2, int* js) {
    float pc[kPruneL], tb[kPruneL];
    if constexpr (PAIRED) {  // i even, i + 8 <= nc
#pragma unroll
        for (int l2 = 0; l2 < kPruneL / 2; ++l2) {
            const int q = (i >> 1) + l2;
            const float4 v = s_pair[2 * q], r = s_pair[2 * q + 1];
            const float2 pc2 = ffma2(make_float2(p.c, p.c), make_float2(v.z, v.w),
                                     ffma2(make_float2(p.kp, p.kp), make_float2(v.x, v.y),
                                           make_float2(p.p0, p.p0)));
            pc[2 * l2] = pc2.x;
            pc[2 * l2 + 1] = pc2.y;
            tb[2 * l2] = __fadd_rn(p.t0, __fmul_rn(p.b, r.x));
            tb[2 * l2 + 1] = __fadd_rn(p.t0, __fmul_rn(p.b, r.y));
        }
    } else {
#pragma unroll
        for (int l = 0; l < kPruneL; ++l) {
            const float4 t = s_core[min(i + l, nc - 1)];
            pc[l] = pc_f32(p.p0, p.kp, p.c, t);
            tb[l] = __fadd_rn(p.t0, __fmul_rn(p.b, t.z));
        }
    }
    float P[kPruneL];
#pragma unroll
    for (int l = 0; l < kPruneL; ++l) {
        float gs = __int_as_float(0x7fffffff);  // J_i empty -> NaN slot
        int j0 = NM;
#pragma unroll
        for (int j = NM - 1; j >= 0; --j) {
            const bool cb = TA[j] <= tb[l];
            gs = cb ? G[j] : gs;
            j0 = cb ? j : j0;
        }
        P[l] = __fadd_rn(pc[l], gs);
        js[l] = j0;
    }
#pragma unroll
    for (int q = 0; q < kPruneL / 2; ++q) {
        P2[q] = make_float2(P[2 * q], P[2 * q + 1]);
        T2[q] = make_float2(tb[2 * q], tb[2 * q + 1]);
    }
}

__device__ __forceinline__ float prune_min8(const float2* P2, const float2* T2, float eta,
                                            float K) {
    float c[8];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        const float2 C = fmul2(ffma2(make_float2(eta, eta), P2[q], make_float2(K, K)), T2[q]);
        c[2 * q] = C.x;
        c[2 * q + 1] = C.y;
    }
    return fminf(fmin3(c[0], c[1], c[2]), fmin3(c[3], c[4], fmin3(c[5], c[6], c[7])));
}

__device__ __forceinline__ float prune_min4(const float2* P2, const float2* T2, float eta,
                                            float K) {
    float c[4];
#pragma unroll
    for (int q = 0; q < 2; ++q) {
        const float2 C = fmul2(ffma2(make_float2(eta, eta), P2[q], make_float2(K, K)), T2[q]);
        c[2 * q] = C.x;
        c[2 * q + 1] = C.y;
    }
    return fminf(fmin3(c[0], c[1], c[2]), c[3]);
}

// First slot (visit order) of the exact lexicographic winner among n slots
// whose minimum cost m is known: the least energy among the slots costing m,
// the first such slot on equal energies (better(), optimizer.cpp:27-32).
template <int N>
__device__ __forceinline__ int prune_pick(const float* C, const float* E, float m) {
    float e[N];
#pragma unroll
    for (int l = 0; l < N; ++l) e[l] = C[l] == m ? E[l] : __int_as_float(0x7f800000);
    float emin = e[0];
#pragma unroll
    for (int l = 1; l < N; ++l) emin = fminf(emin, e[l]);
    int pos = N - 1;
#pragma unroll
    for (int l = N - 2; l >= 0; --l) pos = e[l] == emin ? l : pos;
    return pos;
}

constexpr int kPruneMaxCore = 256;  // pruned kernel: nc <= 256 (per-thread js cache)

template <int CH, int NM>
__global__ void __launch_bounds__(128, DSO_ETA_PRUNE_MINB) eta_sweep_pruned_kernel(
    const float* __restrict__ params, int64_t n, int64_t ld, const float4* __restrict__ core4,
    int nc, const float2* __restrict__ mem2, const float2* __restrict__ etaK, int n_eta,
    int32_t* __restrict__ idx, float* __restrict__ cost, int64_t ld_out) {
    static_assert(CH <= 64 && NM >= 2 && NM <= 4, "tie bits / memory levels");
    using TieT = std::conditional_t<(CH > 32), uint64_t, uint32_t>;
    __shared__ float4 s_core[kPruneMaxCore];
    __shared__ float4 s_pair[kPruneMaxCore + 2];
    __shared__ float2 s_mem[NM];
    __shared__ float2 s_ek[CH];
    // per thread: the 2-bit j0 of every level candidate (one 16-bit word per
    // group), each eta's winning group, and G_j — read back by the replay
    __shared__ uint16_t s_js[kPruneMaxCore / kPruneL][128];
    __shared__ uint8_t s_bg[CH][128];
    __shared__ float s_G[NM][128];
    const int tid = threadIdx.x;
    for (int i = tid; i < nc; i += blockDim.x) s_core[i] = core4[i];
    if (tid < NM) s_mem[tid] = mem2[tid];
    build_pairs(s_pair, core4, nc);
    const int e0 = blockIdx.y * CH;
    for (int e = tid; e < CH; e += blockDim.x) s_ek[e] = etaK[e0 + e < n_eta ? e0 + e : n_eta - 1];
    __syncthreads();
    float ev[CH], Kv[CH];
#pragma unroll
    for (int e = 0; e < CH; ++e) {
        ev[e] = s_ek[e].x;
        Kv[e] = s_ek[e].y;
    }
    const int ng_full = nc / kPruneL;  // paired groups; a tail group covers the rest
    const int ng = (nc + kPruneL - 1) / kPruneL;
    const int top = 1 << (31 - __clz(nc));
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + tid; k < n; k += stride) {
        KParams p;
        p.p0 = __ldg(params + k);
        p.kp = __ldg(params + ld + k);
        p.g = __ldg(params + 2 * ld + k);
        p.c = __ldg(params + 3 * ld + k);
        p.t0 = __ldg(params + 4 * ld + k);
        p.a = __ldg(params + 5 * ld + k);
        p.b = __ldg(params + 6 * ld + k);
        if (params_invalid(p.p0, p.kp, p.g, p.c, p.t0, p.a, p.b)) {
#pragma unroll
            for (int e = 0; e < CH; ++e)
                if (e0 + e < n_eta) {
                    idx[(int64_t)(e0 + e) * ld_out + k] = -1;
                    if (cost) cost[(int64_t)(e0 + e) * ld_out + k] = __int_as_float(0x7fc00000);
                }
            continue;
        }
        const bool fast = params_fast(p);
        float G[NM], TA[NM];
#pragma unroll
        for (int j = 0; j < NM; ++j) {
            G[j] = __fmul_rn(p.g, s_mem[j].x);
            TA[j] = __fadd_rn(p.t0, __fmul_rn(p.a, s_mem[j].y));
            s_G[j][tid] = G[j];
        }
        // knee candidates (i0(j), j): i0(j) = #{ i : TB_i > TA_j } (a prefix)
        int i0[4];
        float2 KP2[2], KT2[2];
        {
            float kp_[4], kt_[4];
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                kp_[j] = __int_as_float(0x7fffffff);
                kt_[j] = 1.f;
                i0[j] = 0;
            }
#pragma unroll
            for (int j = 0; j < NM; ++j) {
                int pos = 0;
                for (int s = top; s > 0; s >>= 1)
                    if (pos + s <= nc &&
                        __fadd_rn(p.t0, __fmul_rn(p.b, s_core[pos + s - 1].z)) > TA[j])
                        pos += s;
                i0[j] = pos;
                const float pc = pc_f32(p.p0, p.kp, p.c, s_core[min(pos, nc - 1)]);
                kp_[j] = pos < nc ? __fadd_rn(pc, G[j]) : __int_as_float(0x7fffffff);
                kt_[j] = TA[j];
            }
            KP2[0] = make_float2(kp_[0], kp_[1]);
            KP2[1] = make_float2(kp_[2], kp_[3]);
            KT2[0] = make_float2(kt_[0], kt_[1]);
            KT2[1] = make_float2(kt_[2], kt_[3]);
        }
        TieT ties = fast ? TieT(0) : ~TieT(0);
        if (fast) {
            float bc[CH];
            int bg[CH];
#pragma unroll
            for (int e = 0; e < CH; ++e) {
                bc[e] = fminf(prune_min4(KP2, KT2, ev[e], Kv[e]), __int_as_float(0x7f800000));
                bg[e] = ng;  // the knee group
            }
            auto group = [&](int g, auto paired) {
                float2 P2[4], T2[4];
                int js[kPruneL];
                prune_level_cands<NM, decltype(paired)::value>(p, s_core, s_pair, g * kPruneL,
                                                               nc, G, TA, P2, T2, js);
                uint32_t w = 0;
#pragma unroll
                for (int l = 0; l < kPruneL; ++l) w |= (uint32_t)(js[l] & 3) << (2 * l);
                s_js[g][tid] = (uint16_t)w;
#pragma unroll
                for (int e = 0; e < CH; ++e) {
                    const float m = prune_min8(P2, T2, ev[e], Kv[e]);
                    ties |= m == bc[e] ? TieT(1) << e : TieT(0);
                    bg[e] = m < bc[e] ? g : bg[e];
                    bc[e] = fminf(m, bc[e]);
                }
            };
            int g = 0;
#pragma unroll 1
            for (; g < ng_full; ++g) group(g, std::true_type{});
            if (g < ng) group(g, std::false_type{});
#pragma unroll
            for (int e = 0; e < CH; ++e) s_bg[e][tid] = (uint8_t)bg[e];
        }
        // replay, one eta per iteration (rolled: one copy of the code)
        const float ta_last = TA[NM - 1];
#pragma unroll 1
        for (int e = 0; e < CH && e0 + e < n_eta; ++e) {
            const float eta = s_ek[e].x, K = s_ek[e].y;
            int bi;
            float bcost;
            if ((ties >> e) & TieT(1)) {
                const Best b = replay_levels<NM>(p, s_core, s_mem, 0, nc, eta, K);
                bi = b.i;
                bcost = b.c;
            } else {
                const int g = s_bg[e][tid];
                if (g == ng) {
                    float C[4], E[4];
#pragma unroll
                    for (int q = 0; q < 2; ++q) {
                        const float2 c2 = fmul2(
                            ffma2(make_float2(eta, eta), KP2[q], make_float2(K, K)), KT2[q]);
                        const float2 e2 = fmul2(KP2[q], KT2[q]);
                        C[2 * q] = c2.x;
                        C[2 * q + 1] = c2.y;
                        E[2 * q] = e2.x;
                        E[2 * q + 1] = e2.y;
                    }
                    const float m = fminf(fmin3(C[0], C[1], C[2]), C[3]);
                    const int pos = prune_pick<4>(C, E, m);
                    int ip = i0[0];
#pragma unroll
                    for (int j = 1; j < 4; ++j) ip = pos == j ? i0[j] : ip;
                    bi = ip * NM + pos;
                    bcost = m;
                } else {
                    const uint32_t w = s_js[g][tid];
                    const int ib = g * kPruneL;
                    float C[kPruneL], P[kPruneL], T[kPruneL];
#pragma unroll
                    for (int l = 0; l < kPruneL; ++l) {
                        const float4 t = s_core[min(ib + l, nc - 1)];
                        const float pc = pc_f32(p.p0, p.kp, p.c, t);
                        T[l] = __fadd_rn(p.t0, __fmul_rn(p.b, t.z));
                        const float gj = s_G[(w >> (2 * l)) & 3][tid];
                        P[l] = ta_last > T[l] ? __int_as_float(0x7fffffff) : __fadd_rn(pc, gj);
                        C[l] = cost_f32(eta, K, P[l], T[l]);
                    }
                    const float m = fminf(fmin3(C[0], C[1], C[2]), fmin3(C[3], C[4], fmin3(C[5], C[6], C[7])));
                    // usually one slot attains m; energies only when several do
                    uint32_t eq = 0;
#pragma unroll
                    for (int l = 0; l < kPruneL; ++l) eq |= C[l] == m ? 1u << l : 0u;
                    int pos = __ffs(eq) - 1;
                    if (eq & (eq - 1)) {
                        float E[kPruneL];
#pragma unroll
                        for (int l = 0; l < kPruneL; ++l) E[l] = __fmul_rn(P[l], T[l]);
                        pos = prune_pick<kPruneL>(C, E, m);
                    }
                    bi = min(ib + pos, nc - 1) * NM + (int)((w >> (2 * pos)) & 3);
                    bcost = m;
                }
            }
            idx[(int64_t)(e0 + e) * ld_out + k] = bi;
            if (cost) cost[(int64_t)(e0 + e) * ld_out + k] = bcost;
        }
    }
}

}  // namespace

cudaError_t launch_sweep_f32(Ctx& cx, const float* params, int64_t n, int64_t ld, float eta,
                             float K, int32_t* idx, float* cost, float* energy, float* time,
                             int32_t* kstatus) {
    if (n <= 0) return cudaSuccess;
    const int grid = grid_for(n, kBlock, cx.num_sms, 8);
    const DomainDev& d = cx.dom;
#define DSO_SWEEP_CASE(NMV)                                                                    \
    sweep_f32_kernel<NMV><<<grid, kBlock, 0, cx.stream>>>(params, n, ld, d.core4, d.nc, d.mem2, \
                                                          d.nm, eta, K, idx, cost, energy,      \
                                                          time, kstatus, fast)
    const bool fast = fast_sweep_ok(cx, K);
    switch (d.nm) {
        case 1: DSO_SWEEP_CASE(1); break;
        case 2: DSO_SWEEP_CASE(2); break;
        case 3: DSO_SWEEP_CASE(3); break;
        case 4: DSO_SWEEP_CASE(4); break;
        default: DSO_SWEEP_CASE(0); break;
    }
#undef DSO_SWEEP_CASE
    ++cx.launches;
    return cudaGetLastError();
}

cudaError_t launch_sweep_f64(Ctx& cx, const double* params, int64_t n, double eta, double K,
                             int32_t* idx, double* cost, double* energy, double* time,
                             int32_t* kstatus) {
    if (n <= 0) return cudaSuccess;
    const int grid = grid_for(n, kBlock, cx.num_sms, 8);
    sweep_f64_kernel<<<grid, kBlock, 0, cx.stream>>>(params, n, cx.dom.core_d, cx.dom.nc,
                                                     cx.dom.mem_d, cx.dom.nm, eta, K, idx, cost,
                                                     energy, time, kstatus);
    ++cx.launches;
    return cudaGetLastError();
}

cudaError_t launch_eta_sweep(Ctx& cx, const float* params, int64_t n, int64_t ld,
                             const float2* etaK_dev, int n_eta, int32_t* idx, float* cost,
                             int64_t ld_out, bool fast, bool prune) {
    if (n <= 0 || n_eta <= 0) return cudaSuccess;
    const DomainDev& d = cx.dom;
    if (prune && d.nm >= 2 && d.nm <= 4 && d.nc <= kPruneMaxCore) {
        constexpr int CH = DSO_ETA_PRUNE_CH;
        const int chunks = (n_eta + CH - 1) / CH;
        const int gx = grid_for(n, 128, cx.num_sms, 16);
        dim3 grid(gx, chunks);
#define DSO_ETA_PRUNED(NMV)                                                                 \
    eta_sweep_pruned_kernel<CH, NMV><<<grid, 128, 0, cx.stream>>>(                          \
        params, n, ld, d.core4, d.nc, d.mem2, etaK_dev, n_eta, idx, cost, ld_out)
        switch (d.nm) {
            case 2: DSO_ETA_PRUNED(2); break;
            case 3: DSO_ETA_PRUNED(3); break;
            default: DSO_ETA_PRUNED(4); break;
        }
#undef DSO_ETA_PRUNED
        ++cx.launches;
        return cudaGetLastError();
    }
    if (fast && d.nm >= 1 && d.nm <= 4) {
        // chunks of up to 26 etas (101 -> 4 chunks of 26, 3 padding slots)
        constexpr int CH = DSO_ETA_CH;
        const int chunks = (n_eta + CH - 1) / CH;
        const int gx = grid_for(n, 128, cx.num_sms, 16);
        dim3 grid(gx, chunks);
#define DSO_ETA_FAST(NMV)                                                                   \
    eta_sweep_fast_kernel<CH, NMV><<<grid, 128, 0, cx.stream>>>(                            \
        params, n, ld, d.core4, d.nc, d.mem2, etaK_dev, n_eta, idx, cost, ld_out)
        switch (d.nm) {
            case 1: DSO_ETA_FAST(1); break;
            case 2: DSO_ETA_FAST(2); break;
            case 3: DSO_ETA_FAST(3); break;
            default: DSO_ETA_FAST(4); break;
        }
#undef DSO_ETA_FAST
        ++cx.launches;
        return cudaGetLastError();
    }
    // pick the chunk size with the least padding (ties -> larger chunk)
    const int cands[3] = {17, 8, 4};
    int best = 17, best_slots = 1 << 30;
    for (int ch : cands) {
        const int slots = ((n_eta + ch - 1) / ch) * ch;
        if (slots < best_slots) {
            best_slots = slots;
            best = ch;
        }
    }
    const int chunks = (n_eta + best - 1) / best;
    const int gx = grid_for(n, 128, cx.num_sms, 16);
    dim3 grid(gx, chunks);
    switch (best) {
        case 17:
            eta_sweep_kernel<17><<<grid, 128, 0, cx.stream>>>(params, n, ld, d.core4, d.nc,
                                                              d.mem2, d.nm, etaK_dev, n_eta,
                                                              idx, cost, ld_out);
            break;
        case 8:
            eta_sweep_kernel<8><<<grid, 128, 0, cx.stream>>>(params, n, ld, d.core4, d.nc,
                                                             d.mem2, d.nm, etaK_dev, n_eta,
                                                             idx, cost, ld_out);
            break;
        default:
            eta_sweep_kernel<4><<<grid, 128, 0, cx.stream>>>(params, n, ld, d.core4, d.nc,
                                                             d.mem2, d.nm, etaK_dev, n_eta,
                                                             idx, cost, ld_out);
            break;
    }
    ++cx.launches;
    return cudaGetLastError();
}

}  // namespace dso_b200
