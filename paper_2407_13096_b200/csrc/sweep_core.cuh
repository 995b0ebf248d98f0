// sweep_core.cuh — the per-kernel grid sweep shared by every sweep kernel.
//
// brute_force_config (reference proj/src/optimizer.cpp:90-117) visits pairs in
// (fc outer, fm inner) order and keeps the first candidate unless a later one
// is strictly better (better(), optimizer.cpp:27-32: cost, then energy; vc and
// fm are the visit order).  Here the visit is split into independent chains
// (one per memory level, or four interleaved core levels when nm == 1) so the
// comparator's dependency chain does not serialise the pipe; each chain keeps
// the reference's sequential rule over its own (increasing) pairs, and
// merge_best combines chains exactly as the single sequential scan would.
#pragma once

#include "common.cuh"

namespace dso_b200 {

struct Best {
    float c, e;
    int i;
};

// Sequential visit-order update: a later pair wins only when strictly better.
__device__ __forceinline__ void upd_best(Best& b, float C, float E, int id) {
    const bool better = (C < b.c) | ((C == b.c) & (E < b.e));
    b.c = better ? C : b.c;
    b.e = better ? E : b.e;
    b.i = better ? id : b.i;
}

// Merge two chains' results into what one sequential scan over both would keep.
// Equal costs: the earlier pair survives unless the later one has strictly
// lower energy (so unordered/NaN energies keep the earlier one, as better()
// does).  NaN costs never win (a NaN-cost first pair is never replaced).
__device__ __forceinline__ void merge_best(Best& a, const Best& o) {
    bool take = false;
    if (o.c < a.c) {
        take = true;
    } else if (o.c == a.c) {
        take = (o.i < a.i) ? !(a.e < o.e) : (o.e < a.e);
    }
    if (take) a = o;
}

struct KParams {
    float p0, kp, g, c, t0, a, b;
};

__device__ __forceinline__ void eval_pair(const KParams& p, float Pc, float Tb, float G, float Ta,
                                          float eta, float K, float& C, float& E) {
    const float P = __fadd_rn(Pc, G);
    const float T = time_f32(p.t0, Ta, Tb);
    C = cost_f32(eta, K, P, T);
    E = __fmul_rn(P, T);
}

// Two pairs (j, j+1) of one core level at once with packed FP32x2 ops; each
// lane rounds exactly like eval_pair.
__device__ __forceinline__ void eval_pair2(float Pc, float Tb, float t0, float2 G, float2 Ta,
                                           float eta, float K, float2& C, float2& E) {
    const float2 P = fadd2(make_float2(Pc, Pc), G);
    const float2 T = fadd2(make_float2(t0, t0), make_float2(fmaxf(Ta.x, Tb), fmaxf(Ta.y, Tb)));
    C = fmul2(ffma2(make_float2(eta, eta), P, make_float2(K, K)), T);
    E = fmul2(P, T);
}

// Sweep core levels [i_lo, i_hi) (non-empty) x all memory levels.
template <int NM>
__device__ __forceinline__ Best sweep_levels(const KParams& p, const float4* __restrict__ s_core,
                                             const float2* __restrict__ s_mem, int nm_rt, int i_lo,
                                             int i_hi, float eta, float K) {
    if constexpr (NM == 2 || NM == 4) {
        // memory levels in pairs: FADD2 / FMUL2 / FFMA2 evaluate two pairs per op
        constexpr int NP = NM / 2;
        float2 G[NP], Ta[NP];
#pragma unroll
        for (int h = 0; h < NP; ++h) {
            G[h] = make_float2(__fmul_rn(p.g, s_mem[2 * h].x), __fmul_rn(p.g, s_mem[2 * h + 1].x));
            Ta[h] = make_float2(__fmul_rn(p.a, s_mem[2 * h].y), __fmul_rn(p.a, s_mem[2 * h + 1].y));
        }
        Best ch[NM];
        {
            const float4 t = s_core[i_lo];
            const float Pc = pc_f32(p.p0, p.kp, p.c, t);
            const float Tb = __fmul_rn(p.b, t.z);
#pragma unroll
            for (int h = 0; h < NP; ++h) {
                float2 C, E;
                eval_pair2(Pc, Tb, p.t0, G[h], Ta[h], eta, K, C, E);
                ch[2 * h] = Best{C.x, E.x, i_lo * NM + 2 * h};
                ch[2 * h + 1] = Best{C.y, E.y, i_lo * NM + 2 * h + 1};
            }
        }
#pragma unroll 2
        for (int i = i_lo + 1; i < i_hi; ++i) {
            const float4 t = s_core[i];
            const float Pc = pc_f32(p.p0, p.kp, p.c, t);
            const float Tb = __fmul_rn(p.b, t.z);
#pragma unroll
            for (int h = 0; h < NP; ++h) {
                float2 C, E;
                eval_pair2(Pc, Tb, p.t0, G[h], Ta[h], eta, K, C, E);
                upd_best(ch[2 * h], C.x, E.x, i * NM + 2 * h);
                upd_best(ch[2 * h + 1], C.y, E.y, i * NM + 2 * h + 1);
            }
        }
#pragma unroll
        for (int j = 1; j < NM; ++j) merge_best(ch[0], ch[j]);
        return ch[0];
    } else if constexpr (NM == 3) {
        float G[NM], Ta[NM];
#pragma unroll
        for (int j = 0; j < NM; ++j) {
            G[j] = __fmul_rn(p.g, s_mem[j].x);
            Ta[j] = __fmul_rn(p.a, s_mem[j].y);
        }
        Best ch[NM];
        {
            const float4 t = s_core[i_lo];
            const float Pc = pc_f32(p.p0, p.kp, p.c, t);
            const float Tb = __fmul_rn(p.b, t.z);
#pragma unroll
            for (int j = 0; j < NM; ++j) {
                eval_pair(p, Pc, Tb, G[j], Ta[j], eta, K, ch[j].c, ch[j].e);
                ch[j].i = i_lo * NM + j;
            }
        }
#pragma unroll 2
        for (int i = i_lo + 1; i < i_hi; ++i) {
            const float4 t = s_core[i];
            const float Pc = pc_f32(p.p0, p.kp, p.c, t);
            const float Tb = __fmul_rn(p.b, t.z);
#pragma unroll
            for (int j = 0; j < NM; ++j) {
                float C, E;
                eval_pair(p, Pc, Tb, G[j], Ta[j], eta, K, C, E);
                upd_best(ch[j], C, E, i * NM + j);
            }
        }
#pragma unroll
        for (int j = 1; j < NM; ++j) merge_best(ch[0], ch[j]);
        return ch[0];
    } else if constexpr (NM == 1) {
        const float G = __fmul_rn(p.g, s_mem[0].x);
        const float Ta = __fmul_rn(p.a, s_mem[0].y);
        Best ch[4];
        {
            const float4 t = s_core[i_lo];
            eval_pair(p, pc_f32(p.p0, p.kp, p.c, t), __fmul_rn(p.b, t.z), G, Ta, eta, K, ch[0].c,
                      ch[0].e);
            ch[0].i = i_lo;
            ch[1] = ch[2] = ch[3] = ch[0];
        }
        int i = i_lo + 1;
        for (; i + 3 < i_hi; i += 4) {
#pragma unroll
            for (int u = 0; u < 4; ++u) {
                const float4 t = s_core[i + u];
                float C, E;
                eval_pair(p, pc_f32(p.p0, p.kp, p.c, t), __fmul_rn(p.b, t.z), G, Ta, eta, K, C, E);
                upd_best(ch[u], C, E, i + u);
            }
        }
        for (; i < i_hi; ++i) {
            const float4 t = s_core[i];
            float C, E;
            eval_pair(p, pc_f32(p.p0, p.kp, p.c, t), __fmul_rn(p.b, t.z), G, Ta, eta, K, C, E);
            upd_best(ch[0], C, E, i);
        }
        merge_best(ch[0], ch[1]);
        merge_best(ch[0], ch[2]);
        merge_best(ch[0], ch[3]);
        return ch[0];
    } else {
        const int nm = nm_rt;
        Best b;
        {
            const float4 t = s_core[i_lo];
            eval_pair(p, pc_f32(p.p0, p.kp, p.c, t), __fmul_rn(p.b, t.z),
                      __fmul_rn(p.g, s_mem[0].x), __fmul_rn(p.a, s_mem[0].y), eta, K, b.c, b.e);
            b.i = i_lo * nm;
        }
        for (int i = i_lo; i < i_hi; ++i) {
            const float4 t = s_core[i];
            const float Pc = pc_f32(p.p0, p.kp, p.c, t);
            const float Tb = __fmul_rn(p.b, t.z);
            for (int j = 0; j < nm; ++j) {
                float C, E;
                eval_pair(p, Pc, Tb, __fmul_rn(p.g, s_mem[j].x), __fmul_rn(p.a, s_mem[j].y), eta,
                          K, C, E);
                upd_best(b, C, E, i * nm + j);
            }
        }
        return b;
    }
}

// ---------------------------------------------------------------------------
// Fast exact sweep: the same argmin as sweep_levels, with about a third of its
// comparator work.
//
// The core levels are visited in groups of GL = 8/NM levels (8 pairs).  Per
// group only the minimum cost is formed (a min-tree: FMNMX), and the running
// minimum over groups keeps the FIRST group attaining it (strict <).  The
// exact lexicographic rule (cost, then energy, then visit order — better(),
// optimizer.cpp:27-32) is then replayed by sweep_levels over the 8 pairs of
// the winning group only.  This equals the full sequential scan unless another
// group reaches the same minimum cost exactly; that is detected (m == best at
// any group) and the whole range is then rescanned by sweep_levels.
//
// T is formed as max(t0 + a/fm, t0 + b/fc): round-to-nearest is monotone, so
// fl(t0 + max(x, y)) == max(fl(t0 + x), fl(t0 + y)) — every cost is
// bit-identical to eval_pair's.  Preconditions (else sweep_levels runs):
// finite params <= 1e12 per kernel and a domain / K within the bounds checked
// on the host (DomainDev::fast_ok), which keep every cost finite, so there are
// no NaNs for FMNMX to drop.
__device__ __forceinline__ bool params_fast(const KParams& p) {
    const float m = fmaxf(fmaxf(fmaxf(p.p0, p.kp), fmaxf(p.g, p.c)),
                          fmaxf(fmaxf(p.t0, p.a), p.b));
    // fmaxf drops NaN operands: test finiteness of the sum separately
    const float s = ((p.p0 + p.kp) + (p.g + p.c)) + ((p.t0 + p.a) + p.b);
    return m <= 1e12f && s == s;
}

template <int NM>
struct FastGroup {
    static constexpr int GL = NM == 3 ? 2 : 8 / NM;  // core levels per group (NM = 1..4)
};

__device__ __forceinline__ float fmin3(float a, float b, float c) {
    float r;
    asm("min.f32 %0, %1, %2, %3;" : "=f"(r) : "f"(a), "f"(b), "f"(c));
    return r;
}

// Per-level terms of a group of GL core levels starting at i: Pc and
// t0 + b/fc.  TAIL: the group is cut at i_end; missing levels repeat the last
// one (a repeated pair has the same cost, so the group minimum is unchanged).
template <int NM, bool TAIL>
__device__ __forceinline__ void group_levels(const KParams& p, const float4* __restrict__ s_core,
                                             int i, int i_end, float* pc, float* tb) {
#pragma unroll
    for (int l = 0; l < FastGroup<NM>::GL; ++l) {
        const float4 t = s_core[TAIL ? min(i + l, i_end - 1) : i + l];
        pc[l] = pc_f32(p.p0, p.kp, p.c, t);
        tb[l] = __fadd_rn(p.t0, __fmul_rn(p.b, t.z));
    }
}

// Level terms from the level-pair table (group start i even): s_pair[2q] =
// {vc, vc', vc^2 fc, vc'^2 fc'}, s_pair[2q+1] = {1/fc, 1/fc', -, -} of levels
// 2q, 2q+1, so two levels' Pc take one FFMA2 pair — lane for lane the same
// roundings as group_levels.
template <int NM>
__device__ __forceinline__ void group_levels_paired(const KParams& p,
                                                    const float4* __restrict__ s_pair, int i,
                                                    float* pc, float* tb) {
#pragma unroll
    for (int l2 = 0; l2 < FastGroup<NM>::GL / 2; ++l2) {
        const int q = (i >> 1) + l2;
        const float4 v = s_pair[2 * q], r = s_pair[2 * q + 1];
        const float2 pc2 = ffma2(make_float2(p.c, p.c), make_float2(v.z, v.w),
                                 ffma2(make_float2(p.kp, p.kp), make_float2(v.x, v.y),
                                       make_float2(p.p0, p.p0)));
        pc[2 * l2] = pc2.x;
        pc[2 * l2 + 1] = pc2.y;
        // scalar: ptxas fuses mul.rn.f32x2 + add.rn.f32x2 into FFMA2 (.rn is
        // mandatory on f32x2, so it does not mark the pair non-contractable)
        tb[2 * l2] = __fadd_rn(p.t0, __fmul_rn(p.b, r.x));
        tb[2 * l2 + 1] = __fadd_rn(p.t0, __fmul_rn(p.b, r.y));
    }
}

// Builds the level-pair table for nc levels (threads of a block cooperate).
__device__ __forceinline__ void build_pairs(float4* s_pair, const float4* __restrict__ core4,
                                            int nc) {
    for (int q = threadIdx.x; q < (nc + 1) / 2; q += blockDim.x) {
        const float4 a = core4[2 * q], b = core4[min(2 * q + 1, nc - 1)];
        s_pair[2 * q] = make_float4(a.x, b.x, a.y, b.y);
        s_pair[2 * q + 1] = make_float4(a.z, b.z, 0.f, 0.f);
    }
}

// P and T of the group's GP = GL*NM pairs, in visit order, two per packed op.
template <int NM>
__device__ __forceinline__ void group_pt(const float* pc, const float* tb, const float* Ta1,
                                         const float* G, float2* P2, float2* T2) {
    constexpr int GP = FastGroup<NM>::GL * NM;
    static_assert(GP % 2 == 0, "groups hold an even number of pairs");
#pragma unroll
    for (int q = 0; q < GP; q += 2) {
        const int l0 = q / NM, j0 = q % NM, l1 = (q + 1) / NM, j1 = (q + 1) % NM;
        P2[q / 2] = fadd2(make_float2(pc[l0], pc[l1]), make_float2(G[j0], G[j1]));
        T2[q / 2] = make_float2(fmaxf(Ta1[j0], tb[l0]), fmaxf(Ta1[j1], tb[l1]));
    }
}

// Minimum cost over the group: C = (eta*P + K) * T per pair (cost_f32's
// rounding), then a three-input min tree (FMNMX3).
template <int NM>
__device__ __forceinline__ float group_min_cost(const float2* P2, const float2* T2, float eta,
                                                float K) {
    constexpr int GP = FastGroup<NM>::GL * NM;
    float c[GP];
#pragma unroll
    for (int q = 0; q < GP / 2; ++q) {
        const float2 C = fmul2(ffma2(make_float2(eta, eta), P2[q], make_float2(K, K)), T2[q]);
        c[2 * q] = C.x;
        c[2 * q + 1] = C.y;
    }
    if constexpr (GP == 8) {
        return fminf(fmin3(c[0], c[1], c[2]), fmin3(c[3], c[4], fmin3(c[5], c[6], c[7])));
    } else {
        static_assert(GP == 6, "group sizes 8 (NM = 1, 2, 4) and 6 (NM = 3)");
        return fminf(fmin3(c[0], c[1], c[2]), fmin3(c[3], c[4], c[5]));
    }
}

template <int NM, bool TAIL, bool PAIRED = false>
__device__ __forceinline__ float group_min(const KParams& p, const float4* __restrict__ s_core,
                                           const float* Ta1, const float* G, int i, int i_end,
                                           float eta, float K,
                                           const float4* __restrict__ s_pair = nullptr) {
    constexpr int GL = FastGroup<NM>::GL;
    float pc[GL], tb[GL];
    if constexpr (PAIRED)
        group_levels_paired<NM>(p, s_pair, i, pc, tb);
    else
        group_levels<NM, TAIL>(p, s_core, i, i_end, pc, tb);
    float2 P2[GL * NM / 2], T2[GL * NM / 2];
    group_pt<NM>(pc, tb, Ta1, G, P2, T2);
    return group_min_cost<NM>(P2, T2, eta, K);
}

// Exact sweep of core levels [i_lo, i_hi) (non-empty) x all memory levels:
// identical result to sweep_levels<NM>(..., i_lo, i_hi, ...).
constexpr int DSO_SWEEP_STEP_UNROLL_C =
#ifdef DSO_SWEEP_STEP_UNROLL
    DSO_SWEEP_STEP_UNROLL;
#else
    1;
#endif
template <int NM, int UNR = 4>
__device__ __forceinline__ Best sweep_best(const KParams& p, const float4* __restrict__ s_core,
                                           const float2* __restrict__ s_mem, int nm_rt, int i_lo,
                                           int i_hi, float eta, float K, bool fast,
                                           const float4* __restrict__ s_pair = nullptr) {
    int lo = i_lo, hi = i_hi;
    if constexpr (NM >= 1 && NM <= 4) {
        constexpr int GL = FastGroup<NM>::GL;
        if (fast && params_fast(p)) {
            float G[NM], Ta1[NM];
#pragma unroll
            for (int j = 0; j < NM; ++j) {
                G[j] = __fmul_rn(p.g, s_mem[j].x);
                Ta1[j] = __fadd_rn(p.t0, __fmul_rn(p.a, s_mem[j].y));
            }
            float bc = __int_as_float(0x7f800000);
            int bg = i_lo;
            bool tie = false;
            int i = i_lo;
            // UNR independent groups per step: their loads and min trees overlap
            // (a single group is a ~80-cycle dependency chain); folded in order
            if (s_pair && !(i_lo & 1)) {  // groups start on even levels: paired level terms
#ifndef DSO_SWEEP_STEP_UNROLL
#define DSO_SWEEP_STEP_UNROLL 1
#endif
#pragma unroll DSO_SWEEP_STEP_UNROLL_C
                for (; i + UNR * GL <= i_hi; i += UNR * GL) {
                    float m[UNR];
#pragma unroll
                    for (int u = 0; u < UNR; ++u)
                        m[u] = group_min<NM, false, true>(p, s_core, Ta1, G, i + u * GL, i_hi, eta,
                                                          K, s_pair);
#pragma unroll
                    for (int u = 0; u < UNR; ++u) {
                        tie |= (m[u] == bc);
                        bg = m[u] < bc ? i + u * GL : bg;
                        bc = fminf(m[u], bc);
                    }
                }
            }
#pragma unroll 1
            for (; i + UNR * GL <= i_hi; i += UNR * GL) {
                float m[UNR];
#pragma unroll
                for (int u = 0; u < UNR; ++u)
                    m[u] = group_min<NM, false>(p, s_core, Ta1, G, i + u * GL, i_hi, eta, K);
#pragma unroll
                for (int u = 0; u < UNR; ++u) {
                    tie |= (m[u] == bc);
                    bg = m[u] < bc ? i + u * GL : bg;
                    bc = fminf(m[u], bc);
                }
            }
#pragma unroll 1
            for (; i + GL <= i_hi; i += GL) {
                const float m = group_min<NM, false>(p, s_core, Ta1, G, i, i_hi, eta, K);
                tie |= (m == bc);
                bg = m < bc ? i : bg;
                bc = fminf(m, bc);
            }
            if (i < i_hi) {
                const float m = group_min<NM, true>(p, s_core, Ta1, G, i, i_hi, eta, K);
                tie |= (m == bc);
                bg = m < bc ? i : bg;
            }
            if (!tie) {
                lo = bg;
                hi = min(bg + GL, i_hi);
            }
        }
    }
    return sweep_levels<NM>(p, s_core, s_mem, nm_rt, lo, hi, eta, K);
}

__device__ __forceinline__ float time_at(const KParams& p, const float4* s_core,
                                         const float2* s_mem, int nm, int idx) {
    const int i = idx / nm, j = idx - i * nm;
    return time_f32(p.t0, __fmul_rn(p.a, s_mem[j].y), __fmul_rn(p.b, s_core[i].z));
}

}  // namespace dso_b200
