// features.cu — feature stage (sm_100a): PTX count normalisation fused with
// the DCGM vector, and the DCGM per-metric mean.
//
// featurize (reference proj/src/ptx_features.cpp:311-329): per category
// (instr 101 | dtype 17 | memspace 8) v[i] = count[i] / total, all-zero when
// the category total is 0; as_vector (mlp.cpp:158-165) places the 8 DCGM
// ratios first.  The reference computes count/total in double and we emit
// float: for totals < 2^24 the correctly rounded FP32 quotient equals the
// double quotient rounded to float (no double-rounding case exists when both
// operands are exact in FP32 — see DESIGN.md §4.1), and the quotient is
// computed with one reciprocal per category plus the Markstein correction
//   q = c*r;  e = fma(-q, t, c);  q = fma(e, r, q)
// which is correctly rounded.  Totals >= 2^24 take an FP64 division
// (features_core.cuh).
//
// Memory-bound: 504 B of counts + 32 B of DCGM in, 536 B out per kernel
// (1,072 B); all accesses are 128-bit and row-contiguous over kernels.
#include <algorithm>

#include "common.cuh"
#include "features_core.cuh"

namespace dso_b200 {

namespace {

// One tile of 128 kernels per iteration: counts + DCGM staged and normalised in
// shared memory by tile_features (all loads of the tile in flight, 128-bit),
// then written out row-contiguous with 128-bit stores.  72.7 KB of shared
// memory per CTA -> 3 CTAs per SM, so one CTA's loads overlap another's math
// and stores.
__global__ void __launch_bounds__(256, 2) featurize_kernel(const uint32_t* __restrict__ counts,
                                                        const float* __restrict__ dcgm,
                                                        int64_t n, int64_t ld,
                                                        float* __restrict__ fused) {
    extern __shared__ __align__(16) float smem[];
    float* act = smem;
    float* scratch = smem + DSO_FUSED_ROWS * kFeatTile;
    const bool vec_ok = ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(counts) & 15) == 0) &&
                        ((reinterpret_cast<uintptr_t>(dcgm) & 15) == 0) &&
                        ((reinterpret_cast<uintptr_t>(fused) & 15) == 0);
    const int64_t tiles = (n + kFeatTile - 1) / kFeatTile;
    const int tid = threadIdx.x;
    auto full = [&](int64_t tile) { return vec_ok && tile * kFeatTile + kFeatTile <= n; };
    // the next tile's loads are issued before this tile's normalisation and
    // stores, so every CTA keeps a tile of reads in flight while it computes
    TileRegs R;
    int64_t tile = blockIdx.x;
    if (tile < tiles && full(tile)) tile_load(R, counts, dcgm, tile * kFeatTile, ld);
    for (; tile < tiles; tile += gridDim.x) {
        const int64_t t0 = tile * kFeatTile;
        if (full(tile))
            tile_store(act, R);
        else
            tile_load_scalar(act, counts, dcgm, t0, n, ld);
        __syncthreads();
        const int64_t next = tile + gridDim.x;
        if (next < tiles && full(next)) tile_load(R, counts, dcgm, next * kFeatTile, ld);
        tile_normalise(act, scratch);
        if (full(tile)) {
            const int q = tid & 31, rp = tid >> 5;
#pragma unroll
            for (int j = 0; j < 17; ++j) {
                const int r = rp + 8 * j;
                if (r < DSO_FUSED_ROWS)
                    __stcs(reinterpret_cast<float4*>(fused + (int64_t)r * ld + t0) + q,
                           reinterpret_cast<const float4*>(act + r * kFeatTile)[q]);
            }
        } else {
            const int m = tid & (kFeatTile - 1), h = tid >> 7;
            if (t0 + m < n)
                for (int r = h; r < DSO_FUSED_ROWS; r += 2)
                    fused[(int64_t)r * ld + t0 + m] = act[r * kFeatTile + m];
        }
        __syncthreads();
    }
}

// load_dcgm_samples mean (telemetry.cpp:73-89): double sum over rows in row
// order, divided by the row count, values checked against [0, 1].
__global__ void __launch_bounds__(256) dcgm_mean_kernel(const double* __restrict__ samples,
                                                        int64_t rows, int64_t n, int64_t ld,
                                                        float* __restrict__ out,
                                                        int64_t* __restrict__ bad_row,
                                                        int* __restrict__ any_bad) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        double sum[8] = {0, 0, 0, 0, 0, 0, 0, 0};
        int64_t bad = 0;
        for (int64_t r = 0; r < rows && !bad; ++r) {
#pragma unroll
            for (int m = 0; m < 8; ++m) {
                const double v = samples[(r * 8 + m) * ld + k];
                if (v < 0.0 || v > 1.0) bad = r + 1;
                sum[m] = __dadd_rn(sum[m], v);
            }
        }
        if (bad_row) bad_row[k] = bad;
        if (bad) {
            atomicOr(any_bad, 1);
            continue;
        }
#pragma unroll
        for (int m = 0; m < 8; ++m) out[m * ld + k] = (float)__ddiv_rn(sum[m], (double)rows);
    }
}

}  // namespace

cudaError_t launch_featurize(Ctx& cx, const uint32_t* counts, const float* dcgm, int64_t n,
                             int64_t ld, float* fused) {
    if (n <= 0) return cudaSuccess;
    const size_t smem = (size_t)(DSO_FUSED_ROWS * kFeatTile + 1024) * sizeof(float);
    {
        cudaError_t e = ensure_smem_attr((const void*)featurize_kernel, cx.device, (int)smem);
        if (e != cudaSuccess) return e;
    }
    const int64_t tiles = (n + kFeatTile - 1) / kFeatTile;
    const int grid = (int)std::min<int64_t>(tiles, (int64_t)cx.num_sms * 2);  // 2 CTAs per SM (registers)
    featurize_kernel<<<grid, 256, smem, cx.stream>>>(counts, dcgm, n, ld, fused);
    ++cx.launches;
    return cudaGetLastError();
}

cudaError_t launch_dcgm_mean(Ctx& cx, const double* samples, int64_t rows, int64_t n,
                             int64_t ld, float* out, int64_t* bad_row, int* any_bad_dev) {
    if (n <= 0) return cudaSuccess;
    dcgm_mean_kernel<<<grid_for(n, 256, cx.num_sms, 8), 256, 0, cx.stream>>>(
        samples, rows, n, ld, out, bad_row, any_bad_dev);
    ++cx.launches;
    return cudaGetLastError();
}

}  // namespace dso_b200
