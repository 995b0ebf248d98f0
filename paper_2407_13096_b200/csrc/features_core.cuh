// features_core.cuh — the feature stage for one tile of 128 kernels, shared by
// the standalone featurize kernel and the fused pipeline.
//
// featurize (reference proj/src/ptx_features.cpp:311-329) + as_vector
// (mlp.cpp:158-165): per category (instr 101 | dtype 17 | memspace 8)
// v[i] = count[i] / total, all-zero for a zero total, DCGM ratios first.  The
// reference divides in double; for totals < 2^24 the correctly rounded FP32
// quotient equals that double rounded to float.  Tile layout:
// act[134][128] floats, k-major (row = feature, 128 kernels contiguous).
#pragma once

#include "common.cuh"

namespace dso_b200 {

constexpr int kFeatTile = 128;

// ---------------------------------------------------------------------------
// Feature stage into act: raw counts [126][ld] + DCGM [8][ld] for kernels
// [t0, t0+128) -> act rows 0..133 (fused order).  Kernels >= n get zeros.
//   phase 1: every load of the tile in flight at once (16 x 128-bit per
//            thread; a warp covers one 512-byte row segment) — or a scalar
//            path for the ragged last tile / unaligned inputs;
//   phase 2: per (kernel, category) exact integer total and its reciprocal,
//            once — not per entry;
//   phase 3: every entry becomes count/total, correctly rounded (Markstein).
// scratch: 1024 floats: tf[3][128], rr[3][128] and the
// split instr partial sums (u64 [128]).
// Registers of one full, aligned tile: 16 x 128-bit count loads + 1 DCGM load
// per thread (a warp covers one 512-byte row segment).
struct TileRegs {
    uint4 v[16];
    float4 d;
};

__device__ __forceinline__ void tile_load(TileRegs& R, const uint32_t* __restrict__ counts,
                                          const float* __restrict__ dcgm, int64_t t0,
                                          int64_t ld) {
    const int q = threadIdx.x & 31, rp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int r = rp + 8 * j;
        if (r < DSO_COUNT_ROWS)
            R.v[j] = __ldg(reinterpret_cast<const uint4*>(counts + (int64_t)r * ld + t0) + q);
    }
    R.d = __ldg(reinterpret_cast<const float4*>(dcgm + (int64_t)rp * ld + t0) + q);
}

__device__ __forceinline__ void tile_store(float* act, const TileRegs& R) {
    uint32_t* acti = reinterpret_cast<uint32_t*>(act);
    const int q = threadIdx.x & 31, rp = threadIdx.x >> 5;
#pragma unroll
    for (int j = 0; j < 16; ++j) {
        const int r = rp + 8 * j;
        if (r < DSO_COUNT_ROWS) reinterpret_cast<uint4*>(acti + (8 + r) * kFeatTile)[q] = R.v[j];
    }
    reinterpret_cast<float4*>(act + rp * kFeatTile)[q] = R.d;
}

// Ragged last tile / unaligned inputs: scalar loads straight into act.
__device__ __forceinline__ void tile_load_scalar(float* act, const uint32_t* __restrict__ counts,
                                                 const float* __restrict__ dcgm, int64_t t0,
                                                 int64_t n, int64_t ld) {
    uint32_t* acti = reinterpret_cast<uint32_t*>(act);
    const int m = threadIdx.x & (kFeatTile - 1);
    const int h = threadIdx.x >> 7;
    const int64_t k = t0 + m;
    const bool live = k < n;
#pragma unroll 9
    for (int r = h; r < DSO_COUNT_ROWS; r += 2)
        acti[(8 + r) * kFeatTile + m] = live ? __ldg(counts + (int64_t)r * ld + k) : 0u;
#pragma unroll
    for (int r = h; r < 8; r += 2) act[r * kFeatTile + m] = live ? __ldg(dcgm + (int64_t)r * ld + k) : 0.f;
}

// Normalise a staged tile in place (phases 2 and 3 below); act holds the raw
// counts in rows 8.. and the DCGM rows 0..7 (the caller synchronised).
__device__ __forceinline__ void tile_normalise(float* act, float* scratch) {
    uint32_t* acti = reinterpret_cast<uint32_t*>(act);
    const int tid = threadIdx.x;
    // phase 2: exact totals (u64), split so both thread halves sum ~63 rows.
    // scratch (1024 floats): tf[3][128], rr[3][128], part u64[128]
    float* tfv = scratch;
    float* rrv = tfv + 3 * kFeatTile;
    uint64_t* part = reinterpret_cast<uint64_t*>(rrv + 3 * kFeatTile);
    constexpr int kSplit = 60;
    const int m = tid & (kFeatTile - 1);
    uint64_t s_a = 0, s_b = 0, s_c = 0;
    if (tid < kFeatTile) {
    #pragma unroll 10
        for (int r = 0; r < kSplit; ++r) s_a += acti[(8 + r) * kFeatTile + m];
    } else {
        for (int r = kSplit; r < DSO_INSTR_SLOTS; ++r) s_a += acti[(8 + r) * kFeatTile + m];
        for (int r = 0; r < DSO_DTYPE_SLOTS; ++r) s_b += acti[(8 + DSO_INSTR_SLOTS + r) * kFeatTile + m];
        for (int r = 0; r < DSO_MEMSPACE_SLOTS; ++r)
            s_c += acti[(8 + DSO_INSTR_SLOTS + DSO_DTYPE_SLOTS + r) * kFeatTile + m];
        part[m] = s_a;
    }
    __syncthreads();
    // tf = total as float (exact below 2^24), rr = RN(1/tf); tf = 0 marks a zero
    // total.  A total >= 2^24 is stored exactly as two 24-bit halves:
    // tf = -hi, rr = lo (total = hi * 2^24 + lo), for the FP64 path of phase 3.
    auto scale = [&](int cat, uint64_t tot) {
        float tf = 0.f, rr = 0.f;
        if (tot != 0 && tot < (1u << 24)) {
            tf = __uint2float_rn((uint32_t)tot);
            rr = __frcp_rn(tf);
        } else if (tot != 0) {
            tf = -(float)(tot >> 24);               // exact: hi < 2^24 for totals < 2^48
            rr = (float)(tot & 0xFFFFFFu);          // exact
        }
        tfv[cat * kFeatTile + m] = tf;
        rrv[cat * kFeatTile + m] = rr;
    };
    if (tid < kFeatTile) {
        scale(0, s_a + part[m]);
    } else {
        scale(1, s_b);
        scale(2, s_c);
    }
    __syncthreads();
    // phase 3: normalise in place, 4 kernels x 16 rows per thread
    {
        const int q = tid & 31;
        const int rp = tid >> 5;
#pragma unroll 4
        for (int j = 0; j < 16; ++j) {
            const int r = rp + 8 * j;
            if (r >= DSO_COUNT_ROWS) break;
            const int cat = r < DSO_INSTR_SLOTS ? 0 : (r < DSO_INSTR_SLOTS + DSO_DTYPE_SLOTS ? 1 : 2);
            uint4* cp = reinterpret_cast<uint4*>(acti + (8 + r) * kFeatTile) + q;
            const uint4 c = *cp;
            const float4 tf = reinterpret_cast<const float4*>(tfv + cat * kFeatTile)[q];
            const float4 rr = reinterpret_cast<const float4*>(rrv + cat * kFeatTile)[q];
            const uint32_t cc[4] = {c.x, c.y, c.z, c.w};
            const float tt[4] = {tf.x, tf.y, tf.z, tf.w};
            const float ri[4] = {rr.x, rr.y, rr.z, rr.w};
            float o[4];
#pragma unroll
            for (int e = 0; e < 4; ++e) {
                if (tt[e] > 0.f) {
                    const float cf =
                        (__int_as_float(0x4B000000u | (cc[e] & 0x7FFFFFu)) - 8388608.f) +
                        ((cc[e] & 0x800000u) ? 8388608.f : 0.f);
                    const float qq = __fmul_rn(cf, ri[e]);
                    o[e] = fmaf(fmaf(-qq, tt[e], cf), ri[e], qq);
                } else if (tt[e] == 0.f) {
                    o[e] = 0.f;
                } else {
                    o[e] = (float)((double)cc[e] / fma((double)-tt[e], 16777216.0, (double)ri[e]));
                }
            }
            *reinterpret_cast<float4*>(cp) = make_float4(o[0], o[1], o[2], o[3]);
        }
    }
    __syncthreads();
}

}  // namespace dso_b200
