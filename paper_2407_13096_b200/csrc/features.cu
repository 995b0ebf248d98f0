// features.cu — feature stage (sm_100a): PTX count normalisation fused with
// the DCGM vector, and the DCGM per-metric mean.
//
// featurize (reference proj/src/ptx_features.cpp:311-329): per category
// (instr 101 | dtype 17 | memspace 8) v[i] = count[i] / total, all-zero when
// the category total is 0; as_vector (mlp.cpp:307-314) places the 8 DCGM
// ratios first.  The reference computes count/total in double and we emit
// float: for totals < 2^24 the correctly rounded FP32 quotient equals the
// double quotient rounded to float (no double-rounding case exists when both
// operands are exact in FP32 — see DESIGN.md §4.1), and the quotient is
// computed with one reciprocal per category plus the Markstein correction
//   q = c*r;  e = fma(-q, t, c);  q = fma(e, r, q)
// which is correctly rounded.  Totals >= 2^24 take an FP64 division.
//
// Memory-bound: 504 B of counts + 32 B of DCGM in, 536 B out per kernel; all
// accesses are row-contiguous over kernels (SoA), i.e. fully coalesced.
#include "common.cuh"

namespace dso_b200 {

namespace {

__device__ __forceinline__ float u32_to_f32_exact(uint32_t v) {
    // exact for v < 2^24 (callers guarantee it); single I2F otherwise
    return __uint2float_rn(v);
}

// Correctly rounded c/t for c <= t < 2^24 given r = RN(1/t).
__device__ __forceinline__ float div_cr(float c, float t, float r) {
    const float q = __fmul_rn(c, r);
    const float e = fmaf(-q, t, c);
    return fmaf(e, r, q);
}

__device__ __forceinline__ float normalize_one(uint32_t count, uint64_t total, float tf,
                                               float r) {
    if (total == 0) return 0.f;
    if (total < (1u << 24)) return div_cr(u32_to_f32_exact(count), tf, r);
    return (float)((double)count / (double)total);
}

__global__ void __launch_bounds__(256) featurize_kernel(const uint32_t* __restrict__ counts,
                                                        const float* __restrict__ dcgm,
                                                        int64_t n, int64_t ld,
                                                        float* __restrict__ fused) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
#pragma unroll
        for (int m = 0; m < 8; ++m) fused[m * ld + k] = __ldg(dcgm + m * ld + k);
        const int base[3] = {0, DSO_INSTR_SLOTS, DSO_INSTR_SLOTS + DSO_DTYPE_SLOTS};
        const int len[3] = {DSO_INSTR_SLOTS, DSO_DTYPE_SLOTS, DSO_MEMSPACE_SLOTS};
#pragma unroll
        for (int cat = 0; cat < 3; ++cat) {
            uint64_t total = 0;
            for (int i = 0; i < len[cat]; ++i) total += __ldg(counts + (base[cat] + i) * ld + k);
            const float tf = (float)total;
            const float r = total ? __frcp_rn(tf) : 0.f;
            for (int i = 0; i < len[cat]; ++i) {
                const int row = base[cat] + i;
                fused[(8 + row) * ld + k] = normalize_one(__ldg(counts + row * ld + k), total, tf, r);
            }
        }
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
    featurize_kernel<<<grid_for(n, 256, cx.num_sms, 8), 256, 0, cx.stream>>>(counts, dcgm, n,
                                                                              ld, fused);
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
