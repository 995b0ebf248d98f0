// gen.cu — synthetic kernel generator on the device (sm_100a).
//
// Device restatement of gen_kernel / features_from (reference
// proj/src/sim_harness.cpp:17-144) with the splitmix64 Rng (rng.hpp:11-55),
// seeded like run_campaign's corpus (sim_harness.cpp:241-242):
//     kernel k  <-  gen_kernel(Rng(root).fork(salt_base + first + k).next_u64()).
// Compiled with --fmad=false: every double expression rounds exactly as the
// reference's x86-64 build (no FMA contraction), so truth parameters, DCGM
// values and the llround'ed PTX counts are bit-identical to the host's; the
// float outputs are those doubles rounded once.
//
// This is the synthetic-input source for the benchmark and for large parity
// runs (the host generator costs ~1 us per kernel; this one ~1 ns).
#include <math.h>

#include "common.cuh"

namespace dso_b200 {

namespace {

struct DevRng {
    uint64_t s;
    __device__ uint64_t next() {  // rng.hpp:18-23
        uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        return z ^ (z >> 31);
    }
    __device__ double uniform01() { return (double)(next() >> 11) * 0x1.0p-53; }  // rng.hpp:26
    __device__ double uniform(double lo, double hi) { return lo + (hi - lo) * uniform01(); }
    __device__ DevRng fork(uint64_t salt) const {  // rng.hpp:50-54
        DevRng c{s ^ (0xd1342543de82ef95ULL * (salt + 1))};
        c.next();
        return c;
    }
};

struct Range {
    double lo, hi, jitter;
};
// sim_harness.cpp:24-30
__device__ constexpr Range kAlpha{40.0, 400.0, 0.10};
__device__ constexpr Range kBeta{40.0, 400.0, 0.10};
__device__ constexpr Range kT0{0.04, 0.30, 0.05};
__device__ constexpr Range kGamma{0.004, 0.020, 0.10};
__device__ constexpr Range kC{0.002, 0.0055, 0.10};
__device__ constexpr Range kP0{40.0, 90.0, 0.05};
__device__ constexpr Range kKappa{5.0, 15.0, 0.05};

__device__ __forceinline__ double encode(const Range& r, double v) {  // :19-21
    const double floor_val = r.lo * (1.0 - r.jitter);
    const double span = r.hi * (1.0 + r.jitter) - floor_val;
    return (v - floor_val) / span;
}
__device__ __forceinline__ double jittered(const Range& r, double w, DevRng& rng) {  // :32-36
    return (r.lo + (r.hi - r.lo) * w) * (1.0 + r.jitter * rng.uniform(-1.0, 1.0));
}
__device__ __forceinline__ uint32_t slot(double w) {  // :67-69
    return (uint32_t)llround(w * 1e6);
}

// Count-row indices of the slots features_from fills (ptx_features.cpp:18-49).
enum : int {
    SL_ADD = 0, SL_MUL = 4, SL_FMA = 37, SL_SETP = 39, SL_MOV = 51, SL_LD = 54, SL_ST = 56,
    SL_CVT = 61, SL_BRA = 71, SL_RET = 74, SL_BAR = 76,
    DT = 101, MS = 118,
};

__global__ void __launch_bounds__(256) gen_kernel_dev(uint64_t root, uint64_t salt_base,
                                                      int64_t first, int64_t n, int64_t ld,
                                                      float* __restrict__ params,
                                                      uint32_t* __restrict__ counts,
                                                      float* __restrict__ dcgm) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n; k += stride) {
        DevRng r{root};
        const uint64_t seed = r.fork(salt_base + (uint64_t)(first + k)).next();
        // gen_kernel(seed): rho from Rng(seed), params from Rng(seed).fork(0x6e6b)
        DevRng rs{seed};
        const double rho = rs.uniform01();
        DevRng g = DevRng{seed}.fork(0x6e6b);
        const double alpha = jittered(kAlpha, 1.0 - rho, g);
        const double beta = jittered(kBeta, rho, g);
        const double t0 = jittered(kT0, g.uniform01(), g);
        const double gamma = jittered(kGamma, 1.0 - rho, g);
        const double c = jittered(kC, rho, g);
        const double p0 = jittered(kP0, g.uniform01(), g);
        const double kappa = jittered(kKappa, g.uniform01(), g);
        if (params) {
            params[k] = (float)p0;
            params[ld + k] = (float)kappa;
            params[2 * ld + k] = (float)gamma;
            params[3 * ld + k] = (float)c;
            params[4 * ld + k] = (float)t0;
            params[5 * ld + k] = (float)alpha;
            params[6 * ld + k] = (float)beta;
        }
        if (dcgm) {  // sim_harness.cpp:43-59
            const double za = encode(kAlpha, alpha), zb = encode(kBeta, beta),
                         zt = encode(kT0, t0), zg = encode(kGamma, gamma), zc = encode(kC, c),
                         zp = encode(kP0, p0), zk = encode(kKappa, kappa);
            dcgm[k] = (float)(0.30 + 0.65 * zt);
            dcgm[ld + k] = (float)(0.10 + 0.80 * zp);
            dcgm[2 * ld + k] = (float)(0.02 + 0.60 * zg);
            dcgm[3 * ld + k] = (float)(0.05 + 0.90 * za);
            dcgm[4 * ld + k] = (float)(0.02 + 0.70 * zk);
            dcgm[5 * ld + k] = (float)(0.05 + 0.90 * zb);
            dcgm[6 * ld + k] = (float)(0.02 + 0.90 * zc);
            dcgm[7 * ld + k] = (float)(0.05 + 0.45 * zb + 0.45 * zc);
        }
        if (counts) {  // sim_harness.cpp:61-95
            const double s = beta / (alpha + beta);
            const double arith = 0.70 * s;
            const double mem = 0.70 * (1.0 - s);
            uint32_t* col = counts + k;
            for (int row = 0; row < DSO_COUNT_ROWS; ++row) col[row * ld] = 0u;
            col[SL_ADD * ld] = slot(0.35 * arith);
            col[SL_MUL * ld] = slot(0.25 * arith);
            col[SL_FMA * ld] = slot(0.40 * arith);
            col[SL_LD * ld] = slot(0.60 * mem);
            col[SL_ST * ld] = slot(0.40 * mem);
            col[SL_MOV * ld] = slot(0.12);
            col[SL_SETP * ld] = slot(0.06);
            col[SL_BRA * ld] = slot(0.06);
            col[SL_CVT * ld] = slot(0.03);
            col[SL_BAR * ld] = slot(0.02);
            col[SL_RET * ld] = slot(0.01);
            col[(DT + 10) * ld] = slot(0.35 + 0.25 * s);  // .f32
            col[(DT + 2) * ld] = slot(0.30 - 0.15 * s);   // .s32
            col[(DT + 6) * ld] = slot(0.10);              // .u32
            col[(DT + 14) * ld] = slot(0.05);             // .b32
            col[(DT + 11) * ld] = slot(0.08 - 0.05 * s);  // .f64
            col[(DT + 7) * ld] = slot(0.07);              // .u64
            col[(DT + 15) * ld] = slot(0.05 - 0.05 * s);  // .b64
            col[(MS + 3) * ld] = slot(0.50 - 0.25 * s);   // .global
            col[(MS + 6) * ld] = slot(0.12 + 0.10 * s);   // .shared
            col[(MS + 5) * ld] = slot(0.08);              // .param
            col[(MS + 0) * ld] = slot(0.20 + 0.15 * s);   // .reg
            col[(MS + 4) * ld] = slot(0.05);              // .local
            col[(MS + 2) * ld] = slot(0.05);              // .const
        }
    }
}

// Sparse (CSR) variant: the same kernels as gen_kernel_dev, counts emitted as
// the 24 slots features_from fills (sim_harness.cpp:70-95), in slot order, as
// (count << 7) | slot; row_ptr[k] = 24 k (row_ptr[n] = 24 n).
__global__ void __launch_bounds__(256) gen_csr_dev(uint64_t root, uint64_t salt_base,
                                                   int64_t first, int64_t n,
                                                   uint64_t* __restrict__ row_ptr,
                                                   uint32_t* __restrict__ entries,
                                                   float* __restrict__ dcgm, int64_t ld) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k <= n; k += stride) {
        row_ptr[k] = 24u * (uint64_t)k;
        if (k == n) continue;
        DevRng r{root};
        const uint64_t seed = r.fork(salt_base + (uint64_t)(first + k)).next();
        DevRng rs{seed};
        const double rho = rs.uniform01();
        DevRng g = DevRng{seed}.fork(0x6e6b);
        const double alpha = jittered(kAlpha, 1.0 - rho, g);
        const double beta = jittered(kBeta, rho, g);
        const double t0 = jittered(kT0, g.uniform01(), g);
        const double gamma = jittered(kGamma, 1.0 - rho, g);
        const double c = jittered(kC, rho, g);
        const double p0 = jittered(kP0, g.uniform01(), g);
        const double kappa = jittered(kKappa, g.uniform01(), g);
        if (dcgm) {
            const double za = encode(kAlpha, alpha), zb = encode(kBeta, beta),
                         zt = encode(kT0, t0), zg = encode(kGamma, gamma), zc = encode(kC, c),
                         zp = encode(kP0, p0), zk = encode(kKappa, kappa);
            dcgm[k] = (float)(0.30 + 0.65 * zt);
            dcgm[ld + k] = (float)(0.10 + 0.80 * zp);
            dcgm[2 * ld + k] = (float)(0.02 + 0.60 * zg);
            dcgm[3 * ld + k] = (float)(0.05 + 0.90 * za);
            dcgm[4 * ld + k] = (float)(0.02 + 0.70 * zk);
            dcgm[5 * ld + k] = (float)(0.05 + 0.90 * zb);
            dcgm[6 * ld + k] = (float)(0.02 + 0.90 * zc);
            dcgm[7 * ld + k] = (float)(0.05 + 0.45 * zb + 0.45 * zc);
        }
        const double s = beta / (alpha + beta);
        const double arith = 0.70 * s;
        const double mem = 0.70 * (1.0 - s);
        const uint32_t cnt[24] = {
            slot(0.35 * arith), slot(0.25 * arith), slot(0.40 * arith), slot(0.06),
            slot(0.12),         slot(0.60 * mem),   slot(0.40 * mem),   slot(0.03),
            slot(0.06),         slot(0.01),         slot(0.02),
            slot(0.30 - 0.15 * s), slot(0.10), slot(0.07), slot(0.35 + 0.25 * s),
            slot(0.08 - 0.05 * s), slot(0.05), slot(0.05 - 0.05 * s),
            slot(0.20 + 0.15 * s), slot(0.05), slot(0.50 - 0.25 * s), slot(0.05), slot(0.08),
            slot(0.12 + 0.10 * s)};
        // slots in increasing order: add mul fma setp mov ld st cvt bra ret bar |
        // .s32 .u32 .u64 .f32 .f64 .b32 .b64 | .reg .const .global .local .param .shared
        const uint8_t sl[24] = {SL_ADD, SL_MUL, SL_FMA, SL_SETP, SL_MOV, SL_LD, SL_ST, SL_CVT,
                                SL_BRA, SL_RET, SL_BAR,
                                DT + 2, DT + 6, DT + 7, DT + 10, DT + 11, DT + 14, DT + 15,
                                MS + 0, MS + 2, MS + 3, MS + 4, MS + 5, MS + 6};
        uint32_t* e = entries + 24 * k;
#pragma unroll
        for (int i = 0; i < 24; ++i) e[i] = (cnt[i] << 7) | sl[i];
    }
}

}  // namespace

cudaError_t launch_gen_csr(Ctx& cx, uint64_t root, uint64_t salt_base, int64_t first, int64_t n,
                           uint64_t* row_ptr, uint32_t* entries, float* dcgm, int64_t ld) {
    if (n < 0) return cudaSuccess;
    const int grid = grid_for(n + 1, 256, cx.num_sms, 16);
    gen_csr_dev<<<grid, 256, 0, cx.stream>>>(root, salt_base, first, n, row_ptr, entries, dcgm,
                                             ld);
    ++cx.launches;
    return cudaGetLastError();
}

cudaError_t launch_gen(Ctx& cx, uint64_t root, uint64_t salt_base, int64_t first, int64_t n,
                       int64_t ld, float* params, uint32_t* counts, float* dcgm) {
    if (n <= 0) return cudaSuccess;
    const int grid = grid_for(n, 256, cx.num_sms, 16);
    gen_kernel_dev<<<grid, 256, 0, cx.stream>>>(root, salt_base, first, n, ld, params, counts,
                                                dcgm);
    ++cx.launches;
    return cudaGetLastError();
}

}  // namespace dso_b200
