// mlp.cu — predictor inference and the fused pipeline (sm_100a).
//
// Predictor: the reference MLP 134-100-50-25-7 (proj/src/mlp.cpp:326), sigmoid
// hidden layers, identity output (forward_trace mlp.cpp:171-181), output
// de-standardised (forward_raw mlp.cpp:381-384) and clamped (predict_params
// mlp.cpp:386-402, kBetaFloor mlp.cpp:15).
//
// Execution model (one persistent CTA per SM, 256 threads, ~165 KB smem):
//   * the whole model (19,825 weights + biases) is staged ONCE per CTA into
//     shared memory, transposed (k-major) and zero-padded per thread group;
//   * a tile of 128 kernels lives in one k-major activation buffer
//     act[134][128] (68.6 KB); every layer reads it, keeps its outputs in
//     registers, syncs, and writes them back in place — nothing between the
//     input load and the final result touches HBM;
//   * layers are register-tiled FP32 GEMMs on the FMA pipe using Blackwell's
//     packed FFMA2 (fma.rn.f32x2 — two FMAs per lane per instruction, with a
//     scalar-broadcast operand so no duplication MOVs are needed):
//       L1 134->100 : thread = 2 kernels x 26 neurons (pairs along n)
//       L2 100->50  : thread = 2 kernels x 13 neurons (pairs along m)
//       L3  50->25  : thread = 2 kernels x  7 neurons (pairs along m)
//       L4  25->7   : thread = 2 kernels x  2 neurons (pairs along m)
//     A warp shares its neuron group, so every weight load is a shared-memory
//     broadcast; activation loads are 256 B contiguous per warp.
//   Tensor cores are not used: TF32/BF16 cannot meet the 1e-5 relative
//   contract on the predicted parameters.
//
// The fused pipeline kernel adds the feature stage in front (raw PTX counts ->
// per-category fractions, fused with DCGM, straight into act) and the grid
// sweep + eta objective + argmin behind (2 threads per kernel, each half the
// core levels, merged with one shuffle), so a kernel's 536 input bytes become
// its 16 result bytes without any intermediate HBM traffic.
#include <math.h>

#include <vector>

#include "common.cuh"
#include "features_core.cuh"
#include "sweep_core.cuh"

namespace dso_b200 {

namespace {

constexpr int kTile = 128;     // kernels per CTA tile
constexpr int kThreads = 256;  // 8 warps

// Packed (transposed, padded) weight layout in floats.  See model_upload.
constexpr int kW1Stride = 112;  // 4 groups x 28 (26 used)
constexpr int kW2Stride = 64;   // 4 groups x 16 (13 used)
constexpr int kW3Stride = 32;   // 4 groups x 8  (7 used)
constexpr int kW4Stride = 8;    // 7 used
constexpr int kOffW1 = 0;
constexpr int kOffW2 = kOffW1 + 134 * kW1Stride;  // 15008
constexpr int kOffW3 = kOffW2 + 100 * kW2Stride;  // 21408
constexpr int kOffW4 = kOffW3 + 50 * kW3Stride;   // 23008
constexpr int kOffB1 = kOffW4 + 25 * kW4Stride;   // 23208
constexpr int kOffB2 = kOffB1 + 104;
constexpr int kOffB3 = kOffB2 + 52;
constexpr int kOffB4 = kOffB3 + 28;
constexpr int kModelFloats = kOffB4 + 8;          // 23400
constexpr int kOffAct = kModelFloats;              // act[134][128]
constexpr int kActFloats = 134 * kTile;
constexpr int kOffOut = kOffAct + kActFloats;      // out[8][128] + stats
constexpr int kOutFloats = 8 * kTile;
constexpr int kOffStats = kOffOut + kOutFloats;    // mean[8], std[8], eta, K
constexpr int kStatsFloats = 32;
constexpr int kOffTables = kOffStats + kStatsFloats;  // core4[nc], mem2[nm] (pipeline)
constexpr int kBaseFloats = kOffTables;

static_assert(kOffW2 % 4 == 0 && kOffW3 % 4 == 0 && kOffW4 % 4 == 0 && kOffB1 % 4 == 0 &&
                  kModelFloats % 4 == 0 && kOffOut % 4 == 0 && kOffTables % 4 == 0,
              "16-byte alignment of smem regions");

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// ---------------------------------------------------------------------------
// Stage the packed model into shared memory (once per CTA).
__device__ __forceinline__ void stage_model(float* smem, const float* __restrict__ packed) {
    const float4* src = reinterpret_cast<const float4*>(packed);
    float4* dst = reinterpret_cast<float4*>(smem);
    for (int i = threadIdx.x; i < kModelFloats / 4; i += kThreads) dst[i] = __ldg(src + i);
}

// ---------------------------------------------------------------------------
// The four layers on act[134][128] (k-major, kernels contiguous).
// Precondition: act rows 0..133 hold the tile's fused features; __syncthreads
// done.  Postcondition: out[n][m] (n < 7) holds forward_raw outputs
// (de-standardised, NOT clamped); __syncthreads done.
__device__ __forceinline__ void mlp_tile(float* smem) {
    const float* W = smem;
    float* act = smem + kOffAct;
    float2* act2 = reinterpret_cast<float2*>(act);  // [row][64] pairs of kernels
    const int tid = threadIdx.x;
    const int mp = tid & 63;  // kernel pair: kernels 2mp, 2mp+1
    const int g = tid >> 6;   // neuron group (uniform per warp)

    // Each layer's k-loop is software-pipelined over two register stages (A, B):
    // the operands of step k+1 are in flight while step k's FFMA2s issue, and
    // the stages alternate without register copies.  Only 2 warps share a
    // scheduler, so shared-memory latency is hidden by this ILP, not by TLP.
    // ---- L1: 134 -> 100 (neurons 26g .. 26g+25), pairs along n -------------
    {
        float2 acc0[13], acc1[13];
#pragma unroll
        for (int p = 0; p < 13; ++p) acc0[p] = acc1[p] = f2(0.f, 0.f);
        const float* wbase = W + kOffW1 + g * 28;
        struct Op {
            float2 a;
            float4 v[6];
            float2 l;
        };
        auto load = [&](Op& o, int k) {
            const float* w = wbase + k * kW1Stride;
            o.a = act2[k * 64 + mp];
#pragma unroll
            for (int q = 0; q < 6; ++q) o.v[q] = reinterpret_cast<const float4*>(w)[q];
            o.l = reinterpret_cast<const float2*>(w)[12];
        };
        auto math = [&](const Op& o) {
            float2 w[13];
#pragma unroll
            for (int q = 0; q < 6; ++q) {
                w[2 * q] = f2(o.v[q].x, o.v[q].y);
                w[2 * q + 1] = f2(o.v[q].z, o.v[q].w);
            }
            w[12] = o.l;
#pragma unroll
            for (int p = 0; p < 13; ++p) {
                acc0[p] = ffma2(f2(o.a.x, o.a.x), w[p], acc0[p]);
                acc1[p] = ffma2(f2(o.a.y, o.a.y), w[p], acc1[p]);
            }
        };
        Op A, B;
        load(A, 0);
#pragma unroll 1
        for (int k = 0; k < 134; k += 2) {
            load(B, k + 1);
            math(A);
            load(A, k + 2 < 134 ? k + 2 : 133);
            math(B);
        }
        __syncthreads();  // all reads of act done
        const float* b = W + kOffB1 + g * 26;
#pragma unroll
        for (int p = 0; p < 13; ++p) {
            const int n = g * 26 + 2 * p;
            const float b0 = b[2 * p], b1 = b[2 * p + 1];
            act2[n * 64 + mp] = f2(sigmoidf_fast(acc0[p].x + b0), sigmoidf_fast(acc1[p].x + b0));
            act2[(n + 1) * 64 + mp] =
                f2(sigmoidf_fast(acc0[p].y + b1), sigmoidf_fast(acc1[p].y + b1));
        }
        __syncthreads();
    }
    // ---- L2: 100 -> 50 (neurons 13g .. 13g+12), pairs along m ----------------
    {
        float2 acc[13];
#pragma unroll
        for (int t = 0; t < 13; ++t) acc[t] = f2(0.f, 0.f);
        const float* wbase = W + kOffW2 + g * 16;
        struct Op {
            float2 a;
            float4 v0, v1, v2;
            float v3;
        };
        auto load = [&](Op& o, int k) {
            const float* w = wbase + k * kW2Stride;
            o.a = act2[k * 64 + mp];
            o.v0 = reinterpret_cast<const float4*>(w)[0];
            o.v1 = reinterpret_cast<const float4*>(w)[1];
            o.v2 = reinterpret_cast<const float4*>(w)[2];
            o.v3 = w[12];
        };
        auto math = [&](const Op& o) {
            const float w[13] = {o.v0.x, o.v0.y, o.v0.z, o.v0.w, o.v1.x, o.v1.y, o.v1.z,
                                 o.v1.w, o.v2.x, o.v2.y, o.v2.z, o.v2.w, o.v3};
#pragma unroll
            for (int t = 0; t < 13; ++t) acc[t] = ffma2(o.a, f2(w[t], w[t]), acc[t]);
        };
        Op A, B;
        load(A, 0);
#pragma unroll 1
        for (int k = 0; k < 100; k += 2) {
            load(B, k + 1);
            math(A);
            load(A, k + 2 < 100 ? k + 2 : 99);
            math(B);
        }
        __syncthreads();
        const float* b = W + kOffB2 + g * 13;
#pragma unroll
        for (int t = 0; t < 13; ++t) {
            const float bb = b[t];
            act2[(g * 13 + t) * 64 + mp] =
                f2(sigmoidf_fast(acc[t].x + bb), sigmoidf_fast(acc[t].y + bb));
        }
        __syncthreads();
    }
    // ---- L3: 50 -> 25 (neurons 7g .. 7g+6), pairs along m ---------------------
    {
        float2 acc[7];
#pragma unroll
        for (int t = 0; t < 7; ++t) acc[t] = f2(0.f, 0.f);
        const float* wbase = W + kOffW3 + g * 8;
        struct Op {
            float2 a;
            float4 v0, v1;
        };
        auto load = [&](Op& o, int k) {
            const float* w = wbase + k * kW3Stride;
            o.a = act2[k * 64 + mp];
            o.v0 = reinterpret_cast<const float4*>(w)[0];
            o.v1 = reinterpret_cast<const float4*>(w)[1];
        };
        auto math = [&](const Op& o) {
            const float w[7] = {o.v0.x, o.v0.y, o.v0.z, o.v0.w, o.v1.x, o.v1.y, o.v1.z};
#pragma unroll
            for (int t = 0; t < 7; ++t) acc[t] = ffma2(o.a, f2(w[t], w[t]), acc[t]);
        };
        Op A, B;
        load(A, 0);
#pragma unroll 1
        for (int k = 0; k < 50; k += 2) {
            load(B, k + 1);
            math(A);
            load(A, k + 2 < 50 ? k + 2 : 49);
            math(B);
        }
        __syncthreads();
        const float* b = W + kOffB3 + g * 7;
#pragma unroll
        for (int t = 0; t < 7; ++t) {
            const float bb = b[t];
            act2[(g * 7 + t) * 64 + mp] =
                f2(sigmoidf_fast(acc[t].x + bb), sigmoidf_fast(acc[t].y + bb));
        }
        __syncthreads();
    }
    // ---- L4: 25 -> 7 (neurons 2g, 2g+1), identity, de-standardise -------------
    {
        float2 acc[2] = {f2(0.f, 0.f), f2(0.f, 0.f)};
        const float* wbase = W + kOffW4 + g * 2;
#pragma unroll 5
        for (int k = 0; k < 25; ++k) {
            const float2 a = act2[k * 64 + mp];
            const float2 w = *reinterpret_cast<const float2*>(wbase + k * kW4Stride);
            acc[0] = ffma2(a, f2(w.x, w.x), acc[0]);
            acc[1] = ffma2(a, f2(w.y, w.y), acc[1]);
        }
        const float* st = smem + kOffStats;  // mean[0..7], std[8..15]
        float2* out2 = reinterpret_cast<float2*>(smem + kOffOut);
#pragma unroll
        for (int t = 0; t < 2; ++t) {
            const int n = 2 * g + t;
            if (n < 7) {
                const float bb = W[kOffB4 + n];
                const float s = st[8 + n], mu = st[n];
                // forward_raw: (z * std) + mean, z = (W a) + b
                out2[n * 64 + mp] = f2(fmaf(acc[t].x + bb, s, mu), fmaf(acc[t].y + bb, s, mu));
            }
        }
        __syncthreads();
    }
}

// predict_params clamp (mlp.cpp:390-399) on out[.][m]; returns clamped flag.
__device__ __forceinline__ bool clamp_params(float p[7]) {
    bool cl = false;
#pragma unroll
    for (int i = 0; i < 7; ++i)
        if (p[i] < 0.f) {
            p[i] = 0.f;
            cl = true;
        }
    if (p[5] + p[6] <= 0.f) {
        p[6] = 1e-12f;
        cl = true;
    }
    return cl;
}

// Fused features already in HBM ([134][ld] float) -> act.  Full tiles: 17
// 128-bit loads per thread, all in flight; ragged / unaligned tiles: scalar.
__device__ __forceinline__ void load_features_fused(float* smem, const float* __restrict__ fused,
                                                    int64_t t0, int64_t n, int64_t ld,
                                                    bool vec_ok) {
    float* act = smem + kOffAct;
    const int tid = threadIdx.x;
    if (vec_ok && t0 + kTile <= n) {
        const int q = tid & 31, rp = tid >> 5;
        float4 v[17];
#pragma unroll
        for (int j = 0; j < 17; ++j) {
            const int r = rp + 8 * j;
            if (r < DSO_FUSED_ROWS)
                v[j] = __ldg(reinterpret_cast<const float4*>(fused + (int64_t)r * ld + t0) + q);
        }
#pragma unroll
        for (int j = 0; j < 17; ++j) {
            const int r = rp + 8 * j;
            if (r < DSO_FUSED_ROWS) reinterpret_cast<float4*>(act + r * kTile)[q] = v[j];
        }
    } else {
        const int m = tid & (kTile - 1);
        const int h = tid >> 7;
        const int64_t k = t0 + m;
        const bool live = k < n;
#pragma unroll 7
        for (int r = h; r < DSO_FUSED_ROWS; r += 2)
            act[r * kTile + m] = live ? __ldg(fused + (int64_t)r * ld + k) : 0.f;
    }
    __syncthreads();
}

__device__ __forceinline__ void stage_stats(float* smem, const float* mean, const float* std_) {
    if (threadIdx.x < 8) {
        smem[kOffStats + threadIdx.x] = mean[threadIdx.x];
        smem[kOffStats + 8 + threadIdx.x] = std_[threadIdx.x];
    }
}

struct Stats {
    float mean[8];
    float std_[8];
};

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kThreads, 1) predict_kernel(
    const float* __restrict__ packed, Stats stats, const float* __restrict__ fused, int64_t n,
    int64_t ld, float* __restrict__ params, uint8_t* __restrict__ clamped,
    float* __restrict__ raw) {
    extern __shared__ __align__(16) float smem[];
    stage_model(smem, packed);
    stage_stats(smem, stats.mean, stats.std_);
    __syncthreads();
    const bool vec_ok = ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(fused) & 15) == 0);
    const int64_t tiles = (n + kTile - 1) / kTile;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t t0 = tile * kTile;
        load_features_fused(smem, fused, t0, n, ld, vec_ok);
        mlp_tile(smem);
        if (threadIdx.x < kTile) {
            const int m = threadIdx.x;
            const int64_t k = t0 + m;
            if (k < n) {
                const float* out = smem + kOffOut;
                float p[7];
#pragma unroll
                for (int i = 0; i < 7; ++i) p[i] = out[i * kTile + m];
                if (raw)
#pragma unroll
                    for (int i = 0; i < 7; ++i) raw[i * ld + k] = p[i];
                const bool cl = clamp_params(p);
#pragma unroll
                for (int i = 0; i < 7; ++i) params[i * ld + k] = p[i];
                if (clamped) clamped[k] = cl ? 1 : 0;
            }
        }
        __syncthreads();
    }
}

// ---------------------------------------------------------------------------
// Fused pipeline: counts + DCGM -> features -> MLP -> clamp -> sweep -> argmin.
__global__ void __launch_bounds__(kThreads, 1) pipeline_kernel(
    const float* __restrict__ packed, Stats stats, const float4* __restrict__ core4, int nc,
    const float2* __restrict__ mem2, int nm, float eta, float K,
    const uint32_t* __restrict__ counts, const float* __restrict__ dcgm, int64_t n, int64_t ld,
    float* __restrict__ params_out, uint8_t* __restrict__ clamped_out,
    int32_t* __restrict__ idx_out, float* __restrict__ cost_out, float* __restrict__ energy_out,
    float* __restrict__ time_out, int64_t ld_out) {
    extern __shared__ __align__(16) float smem[];
    stage_model(smem, packed);
    stage_stats(smem, stats.mean, stats.std_);
    float4* s_core = reinterpret_cast<float4*>(smem + kOffTables);
    float2* s_mem = reinterpret_cast<float2*>(smem + kOffTables + 4 * nc);
    for (int i = threadIdx.x; i < nc; i += kThreads) s_core[i] = core4[i];
    for (int j = threadIdx.x; j < nm; j += kThreads) s_mem[j] = mem2[j];
    __syncthreads();

    const int64_t tiles = (n + kTile - 1) / kTile;
    const bool vec_ok = ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(counts) & 15) == 0) &&
                        ((reinterpret_cast<uintptr_t>(dcgm) & 15) == 0);
    const int tid = threadIdx.x;
    const int m = tid >> 1;    // kernel within tile (2 threads per kernel)
    const int half = tid & 1;  // which half of the core levels
    const int i_split = (nc + 1) >> 1;
    const int i_lo = half ? i_split : 0;
    const int i_hi = half ? nc : i_split;

    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t t0 = tile * kTile;
        tile_features(smem + kOffAct, smem + kOffOut, counts, dcgm, t0, n, ld, vec_ok);
        mlp_tile(smem);

        // ---- clamp + sweep + argmin: 2 threads per kernel --------------------
        const int64_t k = t0 + m;
        const float* out = smem + kOffOut;
        float pr[7];
#pragma unroll
        for (int i = 0; i < 7; ++i) pr[i] = out[i * kTile + m];
        const bool cl = clamp_params(pr);
        const KParams p{pr[0], pr[1], pr[2], pr[3], pr[4], pr[5], pr[6]};
        Best b{__int_as_float(0x7fc00000), __int_as_float(0x7fc00000), i_lo * nm};
        if (i_lo < i_hi) {
            if (nm == 4)
                b = sweep_levels<4>(p, s_core, s_mem, 4, i_lo, i_hi, eta, K);
            else if (nm == 1)
                b = sweep_levels<1>(p, s_core, s_mem, 1, i_lo, i_hi, eta, K);
            else if (nm == 3)
                b = sweep_levels<3>(p, s_core, s_mem, 3, i_lo, i_hi, eta, K);
            else
                b = sweep_levels<0>(p, s_core, s_mem, nm, i_lo, i_hi, eta, K);
        }
        // merge the two halves (the upper half holds the later pairs)
        Best o;
        o.c = __shfl_xor_sync(0xffffffffu, b.c, 1);
        o.e = __shfl_xor_sync(0xffffffffu, b.e, 1);
        o.i = __shfl_xor_sync(0xffffffffu, b.i, 1);
        if (half == 0 && k < n) {
            if (i_split < nc) merge_best(b, o);
            idx_out[k] = b.i;
            if (cost_out) cost_out[k] = b.c;
            if (energy_out) energy_out[k] = b.e;
            if (time_out) time_out[k] = time_at(p, s_core, s_mem, nm, b.i);
            if (params_out)
#pragma unroll
                for (int i = 0; i < 7; ++i) params_out[i * ld_out + k] = pr[i];
            if (clamped_out) clamped_out[k] = cl ? 1 : 0;
        }
        __syncthreads();  // out/act reused by the next tile
    }
}

}  // namespace

size_t mlp_smem_bytes() { return (size_t)kBaseFloats * sizeof(float); }

static size_t pipeline_smem_bytes(int nc, int nm) {
    return (size_t)(kBaseFloats + 4 * nc + 2 * nm) * sizeof(float);
}

// Pack the reference-layout model (W_l row-major [out][in], concatenated, in
// double) into the transposed zero-padded FP32 layout the kernels expect.
cudaError_t model_upload(Ctx& cx, const double* W, const double* b) {
    std::vector<float> pk(kModelFloats, 0.f);
    const double* W1 = W;
    const double* W2 = W1 + 100 * 134;
    const double* W3 = W2 + 50 * 100;
    const double* W4 = W3 + 25 * 50;
    for (int k = 0; k < 134; ++k)
        for (int g = 0; g < 4; ++g)
            for (int t = 0; t < 26; ++t) {
                const int nn = 26 * g + t;
                if (nn < 100) pk[kOffW1 + k * kW1Stride + g * 28 + t] = (float)W1[nn * 134 + k];
            }
    for (int k = 0; k < 100; ++k)
        for (int g = 0; g < 4; ++g)
            for (int t = 0; t < 13; ++t) {
                const int nn = 13 * g + t;
                if (nn < 50) pk[kOffW2 + k * kW2Stride + g * 16 + t] = (float)W2[nn * 100 + k];
            }
    for (int k = 0; k < 50; ++k)
        for (int g = 0; g < 4; ++g)
            for (int t = 0; t < 7; ++t) {
                const int nn = 7 * g + t;
                if (nn < 25) pk[kOffW3 + k * kW3Stride + g * 8 + t] = (float)W3[nn * 50 + k];
            }
    for (int k = 0; k < 25; ++k)
        for (int nn = 0; nn < 7; ++nn) pk[kOffW4 + k * kW4Stride + nn] = (float)W4[nn * 25 + k];
    const double* b1 = b;
    const double* b2 = b1 + 100;
    const double* b3 = b2 + 50;
    const double* b4 = b3 + 25;
    for (int i = 0; i < 100; ++i) pk[kOffB1 + i] = (float)b1[i];
    for (int i = 0; i < 50; ++i) pk[kOffB2 + i] = (float)b2[i];
    for (int i = 0; i < 25; ++i) pk[kOffB3 + i] = (float)b3[i];
    for (int i = 0; i < 7; ++i) pk[kOffB4 + i] = (float)b4[i];
    ModelDev& md = cx.model;
    if (!md.wt) {
        cudaError_t e = cudaMalloc(&md.wt, sizeof(float) * kModelFloats);
        if (e != cudaSuccess) return e;
    }
    md.wt_floats = kModelFloats;
    return cudaMemcpyAsync(md.wt, pk.data(), sizeof(float) * kModelFloats,
                           cudaMemcpyHostToDevice, cx.stream);
}

// Device-side repack of the master weights (reference layout, f32) into the
// packed inference layout, after a training update.  Padding stays zero.
__global__ void repack_kernel(const float* __restrict__ master, float* __restrict__ pk) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    constexpr int MW2 = 100 * 134, MW3 = MW2 + 50 * 100, MW4 = MW3 + 25 * 50;
    constexpr int MB1 = MW4 + 7 * 25, MB2 = MB1 + 100, MB3 = MB2 + 50, MB4 = MB3 + 25;
    if (e < MW2) {
        const int nn = e / 134, k = e - nn * 134;
        pk[kOffW1 + k * kW1Stride + (nn / 26) * 28 + nn % 26] = master[e];
    } else if (e < MW3) {
        const int f = e - MW2, nn = f / 100, k = f - nn * 100;
        pk[kOffW2 + k * kW2Stride + (nn / 13) * 16 + nn % 13] = master[e];
    } else if (e < MW4) {
        const int f = e - MW3, nn = f / 50, k = f - nn * 50;
        pk[kOffW3 + k * kW3Stride + (nn / 7) * 8 + nn % 7] = master[e];
    } else if (e < MB1) {
        const int f = e - MW4, nn = f / 25, k = f - nn * 25;
        pk[kOffW4 + k * kW4Stride + nn] = master[e];
    } else if (e < MB2) {
        pk[kOffB1 + e - MB1] = master[e];
    } else if (e < MB3) {
        pk[kOffB2 + e - MB2] = master[e];
    } else if (e < MB4) {
        pk[kOffB3 + e - MB3] = master[e];
    } else if (e < MB4 + 7) {
        pk[kOffB4 + e - MB4] = master[e];
    }
}

cudaError_t launch_repack(Ctx& cx) {
    const int total = 100 * 134 + 50 * 100 + 25 * 50 + 7 * 25 + 182;
    repack_kernel<<<(total + 255) / 256, 256, 0, cx.stream>>>(cx.model.w_master, cx.model.wt);
    ++cx.launches;
    return cudaGetLastError();
}

static Stats stats_of(const Ctx& cx) {
    Stats s;
    for (int i = 0; i < 8; ++i) {
        s.mean[i] = cx.model.mean[i];
        s.std_[i] = cx.model.std_[i];
    }
    return s;
}

cudaError_t launch_predict(Ctx& cx, const float* fused, int64_t n, int64_t ld, float* params,
                           uint8_t* clamped, float* raw) {
    if (n <= 0) return cudaSuccess;
    const size_t smem = mlp_smem_bytes();
    static bool attr_set = false;  // per process; same value for every device
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(predict_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(227 * 1024));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int64_t tiles = (n + kTile - 1) / kTile;
    const int grid = (int)(tiles < cx.num_sms ? tiles : cx.num_sms);
    predict_kernel<<<grid, kThreads, smem, cx.stream>>>(cx.model.wt, stats_of(cx), fused, n, ld,
                                                       params, clamped, raw);
    ++cx.launches;
    return cudaGetLastError();
}

cudaError_t launch_pipeline(Ctx& cx, const uint32_t* counts, const float* dcgm, int64_t n,
                            int64_t ld, float eta, float K, float* params, uint8_t* clamped,
                            int32_t* idx, float* cost, float* energy, float* time,
                            int64_t ld_out) {
    if (n <= 0) return cudaSuccess;
    const size_t smem = pipeline_smem_bytes(cx.dom.nc, cx.dom.nm);
    if (smem > 227 * 1024) return cudaErrorInvalidValue;
    static bool attr_set = false;
    if (!attr_set) {
        cudaError_t e = cudaFuncSetAttribute(pipeline_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)(227 * 1024));
        if (e != cudaSuccess) return e;
        attr_set = true;
    }
    const int64_t tiles = (n + kTile - 1) / kTile;
    const int grid = (int)(tiles < cx.num_sms ? tiles : cx.num_sms);
    pipeline_kernel<<<grid, kThreads, smem, cx.stream>>>(
        cx.model.wt, stats_of(cx), cx.dom.core4, cx.dom.nc, cx.dom.mem2, cx.dom.nm, eta, K,
        counts, dcgm, n, ld, params, clamped, idx, cost, energy, time, ld_out);
    ++cx.launches;
    return cudaGetLastError();
}

}  // namespace dso_b200
