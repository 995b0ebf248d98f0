// train.cu — predictor training on the device (sm_100a).
//
// One mini-batch step of the reference's SGD (reference proj/src/mlp.cpp):
//   forward_trace (:171-181) -> residual delta = out - y (:425-426, identity
//   output, MSE) -> backprop delta_l = (W_l^T delta_{l+1}) .* a(1-a) (:427-436)
//   -> gW_l = delta_{l+1} a_l^T, gb_l = sum_cols delta_{l+1} (:428-429)
//   -> W -= lr * g (:254-257).
// The reference scales delta by 1/(B*out) up front; here the kernel returns the
// UNSCALED sum over the batch and dso_train_apply applies lr/(B_global*out), so
// a data-parallel step is grad -> NCCL allreduce(sum) -> apply (identical
// update on every rank).
//
// train_grad_kernel: persistent, one CTA per SM, 256 threads, tiles of 64
// samples.  Per tile everything stays in shared memory (~195 KB): the model
// (packed per layer for the thread mappings below), the four activation
// layers, the deltas (written over the activations they no longer need), the
// targets.  Each thread owns fixed blocks of the gradient (gW1 4x14, gW2 2x10,
// gW3 1x5, gW4 1, one bias) and accumulates them in registers across all of
// its tiles; at the end every CTA writes its partial gradient once, and a
// second kernel sums the partials in a fixed order (deterministic, no atomics).
#include <math.h>

#include <algorithm>
#include <type_traits>

#include "common.cuh"
#include "tc.cuh"

namespace dso_b200 {

namespace {

constexpr int TM = 64;       // samples per tile
constexpr int RS = 64;       // row stride (floats) of activation buffers
constexpr int RS2 = RS / 2;  // in float2 units
constexpr int kThreads = 256;

// packed weights (floats): layer l stored [K][8 groups][TNP], neuron n = TN*g + t
constexpr int W1S = 0;                     // [134][16][8], layer 1: neuron n = 7*g + t
constexpr int W2S = W1S + 134 * 8 * 16;    // [100][8][8],  TN 7
constexpr int W3S = W2S + 100 * 8 * 8;     // [50][8][4],   TN 4
constexpr int W4S = W3S + 50 * 8 * 4;      // [25][8],      TN 1
constexpr int B1S = W4S + 25 * 8;          // [104]
constexpr int B2S = B1S + 104;             // [56]
constexpr int B3S = B2S + 56;              // [32]
constexpr int B4S = B3S + 32;              // [8]
// transposed copies for the delta recursion: [N_out][8 k-groups][TKP], k = TK*g + t
constexpr int T2S = B4S + 8;               // W2: [50][8][16], TK 13
constexpr int T3S = T2S + 50 * 8 * 16;     // W3: [25][8][8],  TK 7
constexpr int T4S = T3S + 25 * 8 * 8;      // W4: [7][8][4],   TK 4
constexpr int A0S = T4S + 7 * 8 * 4;       // [134][RS]
constexpr int A1S = A0S + 134 * RS;        // [104][RS]
constexpr int A2S = A1S + 104 * RS;        // [56][RS]
constexpr int A3S = A2S + 56 * RS;         // [32][RS]
constexpr int OS = A3S + 32 * RS;          // [8][RS]   output, then delta4
constexpr int YS = OS + 8 * RS;            // [8][RS]   targets
constexpr int kSmemFloats = YS + 8 * RS;
static_assert(kSmemFloats * 4 <= 227 * 1024, "shared memory");
static_assert(A0S % 4 == 0 && W2S % 4 == 0 && W3S % 4 == 0 && W4S % 4 == 0 && T2S % 4 == 0 &&
                  T3S % 4 == 0 && T4S % 4 == 0, "alignment");

// master (reference) layout offsets: W1 | W2 | W3 | W4 | b1 | b2 | b3 | b4
constexpr int MW1 = 0, MW2 = MW1 + 100 * 134, MW3 = MW2 + 50 * 100, MW4 = MW3 + 25 * 50;
constexpr int MB1 = MW4 + 7 * 25, MB2 = MB1 + 100, MB3 = MB2 + 50, MB4 = MB3 + 25;
constexpr int kMasterFloats = MB4 + 7;  // 20007

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

// loop unrolling of the forward / backward layers (build knobs)
#ifndef DSO_TRAIN_DENSE_UNROLL
#define DSO_TRAIN_DENSE_UNROLL 4
#endif
#ifndef DSO_TRAIN_L1_UNROLL
#define DSO_TRAIN_L1_UNROLL 4
#endif
#ifndef DSO_TRAIN_BACK_UNROLL
#define DSO_TRAIN_BACK_UNROLL 8
#endif
constexpr int kDenseUnroll = DSO_TRAIN_DENSE_UNROLL, kL1Unroll = DSO_TRAIN_L1_UNROLL,
              kBackUnroll = DSO_TRAIN_BACK_UNROLL;

// The weight image [0, A0S) of the training kernel's shared memory — forward
// packings per layer, transposed copies for the delta recursion, biases, zero
// padding — built from the master weights once per update (train_pack_kernel)
// and copied verbatim into every CTA's shared memory with 128-bit loads.
// (The image is zeroed by a memset first; the padding stays zero.)
__global__ void __launch_bounds__(kThreads) train_pack_kernel(const float* __restrict__ m,
                                                              float* __restrict__ img) {
    float* sm = img;

    for (int e = blockIdx.x * kThreads + threadIdx.x; e < 100 * 134; e += gridDim.x * kThreads) {
        const int n = e / 134, k = e - n * 134;
        sm[W1S + (k * 16 + n / 7) * 8 + n % 7] = m[MW1 + e];
    }
    for (int e = blockIdx.x * kThreads + threadIdx.x; e < 50 * 100; e += gridDim.x * kThreads) {
        const int n = e / 100, k = e - n * 100;
        sm[W2S + (k * 8 + n / 7) * 8 + n % 7] = m[MW2 + e];
    }
    for (int e = blockIdx.x * kThreads + threadIdx.x; e < 25 * 50; e += gridDim.x * kThreads) {
        const int n = e / 50, k = e - n * 50;
        sm[W3S + (k * 8 + n / 4) * 4 + n % 4] = m[MW3 + e];
    }
    for (int e = blockIdx.x * kThreads + threadIdx.x; e < 7 * 25; e += gridDim.x * kThreads) {
        const int n = e / 25, k = e - n * 25;
        sm[W4S + k * 8 + n] = m[MW4 + e];
    }
    for (int i = blockIdx.x * kThreads + threadIdx.x; i < 100; i += gridDim.x * kThreads) sm[B1S + i] = m[MB1 + i];
    for (int i = blockIdx.x * kThreads + threadIdx.x; i < 50; i += gridDim.x * kThreads) sm[B2S + i] = m[MB2 + i];
    for (int i = blockIdx.x * kThreads + threadIdx.x; i < 25; i += gridDim.x * kThreads) sm[B3S + i] = m[MB3 + i];
    for (int i = blockIdx.x * kThreads + threadIdx.x; i < 7; i += gridDim.x * kThreads) sm[B4S + i] = m[MB4 + i];
    for (int e = blockIdx.x * kThreads + threadIdx.x; e < 50 * 100; e += gridDim.x * kThreads) {
        const int n = e / 100, k = e - n * 100;
        sm[T2S + (n * 8 + k / 13) * 16 + k % 13] = m[MW2 + e];
    }
    for (int e = blockIdx.x * kThreads + threadIdx.x; e < 25 * 50; e += gridDim.x * kThreads) {
        const int n = e / 50, k = e - n * 50;
        sm[T3S + (n * 8 + k / 7) * 8 + k % 7] = m[MW3 + e];
    }
    for (int e = blockIdx.x * kThreads + threadIdx.x; e < 7 * 25; e += gridDim.x * kThreads) {
        const int n = e / 25, k = e - n * 25;
        sm[T4S + (n * 8 + k / 4) * 4 + k % 4] = m[MW4 + e];
    }
}

__device__ __forceinline__ void stage_weights(float* sm, const float* __restrict__ img) {
    static_assert(A0S % 4 == 0, "image is a whole number of float4");
    const float4* src = reinterpret_cast<const float4*>(img);
    float4* dst = reinterpret_cast<float4*>(sm);
    for (int i = threadIdx.x; i < A0S / 4; i += kThreads) dst[i] = __ldg(src + i);
}

// Dense layer on a 64-sample tile: out[TN*g+t][m] = act(sum_k W[k][g][t] in[k][m] + b).
// thread = (sample pair mp, neuron group g = warp); FFMA2 pairs along samples,
// scalar-broadcast weights; two-stage software pipeline over k.
template <int K, int TN, int TNP, bool SIGMOID>
__device__ __forceinline__ void dense(const float* sm, int woff, int boff, int in_off,
                                      int out_off) {
    const int mp = threadIdx.x & 31, g = threadIdx.x >> 5;
    const float2* in2 = reinterpret_cast<const float2*>(sm + in_off);
    float2 acc[TN];
#pragma unroll
    for (int t = 0; t < TN; ++t) acc[t] = f2(0.f, 0.f);
    struct Op {
        float2 a;
        float w[TNP];
    };
    auto load = [&](Op& o, int k) {
        o.a = in2[k * RS2 + mp];
        const float* w = sm + woff + (k * 8 + g) * TNP;
        if constexpr (TNP % 4 == 0) {
#pragma unroll
            for (int q = 0; q < TNP / 4; ++q) {
                const float4 v = reinterpret_cast<const float4*>(w)[q];
                o.w[4 * q] = v.x;
                o.w[4 * q + 1] = v.y;
                o.w[4 * q + 2] = v.z;
                o.w[4 * q + 3] = v.w;
            }
        } else {
#pragma unroll
            for (int q = 0; q < TNP; ++q) o.w[q] = w[q];
        }
    };
    auto math = [&](const Op& o) {
#pragma unroll
        for (int t = 0; t < TN; ++t) acc[t] = ffma2(o.a, f2(o.w[t], o.w[t]), acc[t]);
    };
    Op A, B;
    load(A, 0);
#pragma unroll kDenseUnroll
    for (int k = 0; k + 1 < K; k += 2) {
        load(B, k + 1);
        math(A);
        load(A, k + 2 < K ? k + 2 : K - 1);
        math(B);
    }
    if (K & 1) math(A);
    float2* out2 = reinterpret_cast<float2*>(const_cast<float*>(sm) + out_off);
#pragma unroll
    for (int t = 0; t < TN; ++t) {
        const float bb = sm[boff + TN * g + t];
        float2 z = f2(acc[t].x + bb, acc[t].y + bb);
        if (SIGMOID) z = f2(sigmoidf_fast(z.x), sigmoidf_fast(z.y));
        out2[(TN * g + t) * RS2 + mp] = z;
    }
}

// Layer 1 (134 -> 100, half of the forward/backward work): thread = 4 samples
// (a float4 of A0) x 7 neurons of group g (16 groups, 112 slots); a warp reads
// 16 sample quads (2 wavefronts) and the weights of 2 groups (2 LDS.128 of 8) per
// k for 14 FFMA2 — about 1.6x fewer shared-memory wavefronts per FFMA2 than the
// generic dense<> tile; two k per stage, operands of the next stage in flight.
__device__ __forceinline__ void dense_l1(float* sm) {
    const int lane = threadIdx.x & 31;
    const int sq = lane & 15, g = (threadIdx.x >> 5) * 2 + (lane >> 4);
    constexpr int RS4 = RS / 4;
    const float4* a4 = reinterpret_cast<const float4*>(sm + A0S) + sq;
    const float4* w4 = reinterpret_cast<const float4*>(sm + W1S) + g * 2;
    float2 acc0[7], acc1[7];
#pragma unroll
    for (int t = 0; t < 7; ++t) acc0[t] = acc1[t] = f2(0.f, 0.f);
    struct Op {
        float4 a[2], w0[2], w1[2];
    };
    auto load = [&](Op& o, int k) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            o.a[u] = a4[(k + u) * RS4];
            o.w0[u] = w4[(k + u) * 32];
            o.w1[u] = w4[(k + u) * 32 + 1];
        }
    };
    auto math = [&](const Op& o) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const float w[7] = {o.w0[u].x, o.w0[u].y, o.w0[u].z, o.w0[u].w,
                                o.w1[u].x, o.w1[u].y, o.w1[u].z};
            const float2 a01 = f2(o.a[u].x, o.a[u].y), a23 = f2(o.a[u].z, o.a[u].w);
#pragma unroll
            for (int t = 0; t < 7; ++t) {
                acc0[t] = ffma2(a01, f2(w[t], w[t]), acc0[t]);
                acc1[t] = ffma2(a23, f2(w[t], w[t]), acc1[t]);
            }
        }
    };
    Op A, B;
    load(A, 0);
#pragma unroll kL1Unroll
    for (int k = 0; k < 132; k += 4) {  // 134 = 33 double stages + one trailing pair
        load(B, k + 2);
        math(A);
        load(A, k + 4);
        math(B);
    }
    math(A);  // k = 132, 133
    float4* out4 = reinterpret_cast<float4*>(sm + A1S) + sq;
#pragma unroll
    for (int t = 0; t < 7; ++t) {
        const int n = 7 * g + t;
        if (n < 100) {
            const float bb = sm[B1S + n];
            out4[n * RS4] = make_float4(sigmoidf_fast(acc0[t].x + bb), sigmoidf_fast(acc0[t].y + bb),
                                        sigmoidf_fast(acc1[t].x + bb), sigmoidf_fast(acc1[t].y + bb));
        }
    }
}

// Layer 2 (100 -> 50) with layer 1's register tile (4 samples x 7 neurons per
// thread, a quarter of the shared-memory loads per FFMA2 of dense<>): eight groups
// of 7 neurons x 16 sample quads cover 128 threads, so the two halves of the CTA
// each take half of K; the upper half leaves its partial sums in the output rows,
// the lower half adds them, the bias and the sigmoid.
__device__ __forceinline__ void dense_l2_split(float* sm) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sq = lane & 15, g = (warp & 3) * 2 + (lane >> 4), half = warp >> 2;
    constexpr int RS4 = RS / 4;
    const int k0 = half * 50;
    const float4* a4 = reinterpret_cast<const float4*>(sm + A1S) + sq;
    const float4* w4 = reinterpret_cast<const float4*>(sm + W2S) + g * 2;  // 16 float4 per k
    float2 acc0[7], acc1[7];
#pragma unroll
    for (int t = 0; t < 7; ++t) acc0[t] = acc1[t] = f2(0.f, 0.f);
    struct Op {
        float4 a[2], w0[2], w1[2];
    };
    auto load = [&](Op& o, int k) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            o.a[u] = a4[(k + u) * RS4];
            o.w0[u] = w4[(k + u) * 16];
            o.w1[u] = w4[(k + u) * 16 + 1];
        }
    };
    auto math = [&](const Op& o) {
#pragma unroll
        for (int u = 0; u < 2; ++u) {
            const float w[7] = {o.w0[u].x, o.w0[u].y, o.w0[u].z, o.w0[u].w,
                                o.w1[u].x, o.w1[u].y, o.w1[u].z};
            const float2 a01 = f2(o.a[u].x, o.a[u].y), a23 = f2(o.a[u].z, o.a[u].w);
#pragma unroll
            for (int t = 0; t < 7; ++t) {
                acc0[t] = ffma2(a01, f2(w[t], w[t]), acc0[t]);
                acc1[t] = ffma2(a23, f2(w[t], w[t]), acc1[t]);
            }
        }
    };
    Op A, B;
    load(A, k0);
#pragma unroll kL1Unroll
    for (int k = k0; k < k0 + 48; k += 4) {  // 50 = 12 double stages + one trailing pair
        load(B, k + 2);
        math(A);
        load(A, k + 4);
        math(B);
    }
    math(A);  // k0 + 48, k0 + 49
    float4* out4 = reinterpret_cast<float4*>(sm + A2S) + sq;
    if (half == 1) {
#pragma unroll
        for (int t = 0; t < 7; ++t)
            if (7 * g + t < 50)
                out4[(7 * g + t) * RS4] = make_float4(acc0[t].x, acc0[t].y, acc1[t].x, acc1[t].y);
    }
    __syncthreads();
    if (half == 0) {
#pragma unroll
        for (int t = 0; t < 7; ++t) {
            const int n = 7 * g + t;
            if (n < 50) {
                const float4 q = out4[n * RS4];
                const float bb = sm[B2S + n];
                out4[n * RS4] = make_float4(sigmoidf_fast(acc0[t].x + q.x + bb),
                                            sigmoidf_fast(acc0[t].y + q.y + bb),
                                            sigmoidf_fast(acc1[t].x + q.z + bb),
                                            sigmoidf_fast(acc1[t].y + q.w + bb));
            }
        }
    }
}

// delta_l[k][m] = (sum_n W[n][k] delta_{l+1}[n][m]) * a_l[k][m] (1 - a_l[k][m]),
// thread = (sample pair, group of TK consecutive k); weights read as scalar
// broadcasts from the packed [K][8][TNP] layout of layer l.  Returns values in
// registers (the caller writes them over a_l after a barrier).
template <int KOUT, int TK, int NIN, int TKP>
__device__ __forceinline__ void backprop(const float* sm, int toff, int din_off, int a_off,
                                         float2 (&res)[TK]) {
    const int mp = threadIdx.x & 31, kg = threadIdx.x >> 5;
    const float2* d2 = reinterpret_cast<const float2*>(sm + din_off);
    const float2* a2 = reinterpret_cast<const float2*>(sm + a_off);
#pragma unroll
    for (int t = 0; t < TK; ++t) res[t] = f2(0.f, 0.f);
    // weights W[n][TK*kg + t] are contiguous in the transposed copy (warp-uniform
    // broadcast loads, TKP/4 LDS.128 per n)
#pragma unroll kBackUnroll
    for (int n = 0; n < NIN; ++n) {
        const float2 d = d2[n * RS2 + mp];
        const float4* w4 = reinterpret_cast<const float4*>(sm + toff + (n * 8 + kg) * TKP);
        float w[TKP];
#pragma unroll
        for (int q = 0; q < TKP / 4; ++q) {
            const float4 v = w4[q];
            w[4 * q] = v.x;
            w[4 * q + 1] = v.y;
            w[4 * q + 2] = v.z;
            w[4 * q + 3] = v.w;
        }
#pragma unroll
        for (int t = 0; t < TK; ++t) res[t] = ffma2(d, f2(w[t], w[t]), res[t]);
    }
#pragma unroll
    for (int t = 0; t < TK; ++t) {
        const int k = kg * TK + t;
        if (k < KOUT) {
            const float2 a = a2[k * RS2 + mp];
            res[t] = f2(res[t].x * a.x * (1.f - a.x), res[t].y * a.y * (1.f - a.y));
        }
    }
}

template <int KOUT, int TK>
__device__ __forceinline__ void store_delta(float* sm, int a_off, const float2 (&res)[TK]) {
    const int mp = threadIdx.x & 31, kg = threadIdx.x >> 5;
    float2* a2 = reinterpret_cast<float2*>(sm + a_off);
#pragma unroll
    for (int t = 0; t < TK; ++t) {
        const int k = kg * TK + t;
        if (k < KOUT) a2[k * RS2 + mp] = res[t];
    }
}

// Rows of one 64-sample tile, smem [R][RS] (feature-major) -> global rows
// [R][lds] at column t0 (lds % 4 == 0, t0 % 64 == 0: float4 stores).
__device__ __forceinline__ void write_rows(const float* sm, int off, int R, float* __restrict__ g,
                                           int64_t lds, int64_t t0) {
    for (int e = threadIdx.x; e < R * (TM / 4); e += kThreads) {
        const int r = e / (TM / 4), q = e % (TM / 4);
        const float4 v = reinterpret_cast<const float4*>(sm + off + r * RS)[q];
        reinterpret_cast<float4*>(g + (int64_t)r * lds + t0)[q] = v;
    }
}

// Scratch rows written by train_fb_kernel (feature-major [row][lds]):
// deltas D1 | D2 | D3 | D4 then activations A1 | A2 | A3.
constexpr int SD1 = 0, SD2 = 100, SD3 = 150, SD4 = 175, SA1 = 182, SA2 = 282, SA3 = 332;
constexpr int kScratchRows = 357;
constexpr int kScratchAlloc = 504;  // floats per sample: the stage images
static_assert(kScratchAlloc >= kScratchRows, "the scratch holds either layout");

// Stage images for the tensor-core weight gradient (train_tc): per 16-sample
// stage one contiguous block holding that stage's operands exactly as
// train_wgrad_tc_kernel's shared memory holds them (SWIZZLE_NONE K-major core
// matrices, 8 rows x 4 samples per 128 bytes).  Layers 2-4 share one MMA chain:
// their deltas are stacked into one A operand (rows d2 0-49 | d3 50-74 | d4 75-81)
// and their inputs into one B operand (rows a1 0-99 | a2 100-149 | a3 150-174 |
// ones 175), so D = A B^T holds the three weight gradients as diagonal blocks and
// the bias gradients in the ones column (the off-diagonal blocks are not used).
// Segments: 0 = d1 (A of layer 1, 104 rows), 1 = stacked deltas (88 rows),
// 2 = x + ones row (136 rows), 3 = stacked inputs + ones row (176 rows).
// The kernel moves a stage with one bulk copy.
namespace wimg {
constexpr int KS = 16;
__host__ __device__ constexpr int ROWS(int s) {
    return s == 0 ? 104 : s == 1 ? 88 : s == 2 ? 136 : 176;
}
// (closed form, not recursive: it must fold to a constant in device code)
__host__ __device__ constexpr int OFF(int s) {
    return KS * (s <= 0 ? 0 : s == 1 ? 104 : s == 2 ? 192 : s == 3 ? 328 : 504);
}
constexpr int FLOATS = OFF(4);  // 8064 floats = 32,256 bytes per stage
static_assert(OFF(4) == OFF(3) + ROWS(3) * KS && OFF(3) == OFF(2) + ROWS(2) * KS &&
                  OFF(2) == OFF(1) + ROWS(1) * KS, "image size");
}  // namespace wimg

// Rows [lo, hi) of segment `seg` in the four stage images of one 64-sample tile:
// row r takes smem row r - lo of [..][RS] at `off` (off < 0: the constant `fill`).
// A warp writes one 512-byte block (8 rows x 4 sample quads of one stage) at a time;
// lane -> (row r & 7, quad (lane / 8 + r) & 3), so a quarter-warp's reads hit 4
// distinct bank groups (2-way at most with the 256-byte row stride).
__device__ __forceinline__ void write_img(const float* sm, int off, int lo, int hi, float fill,
                                          int seg, float* __restrict__ img, int64_t tile) {
    const int g0 = lo >> 3, G = ((hi + 7) >> 3) - g0;
    float* base = img + tile * 4 * wimg::FLOATS + wimg::OFF(seg);
    const int lane = threadIdx.x & 31, rl = lane & 7, k4 = ((lane >> 3) + rl) & 3;
    for (int wi = threadIdx.x >> 5; wi < 4 * G; wi += kThreads / 32) {
        const int st = wi / G, g = g0 + wi - st * G, r = g * 8 + rl;
        if (r < lo || r >= hi) continue;
        const float4 v = off >= 0
                             ? *reinterpret_cast<const float4*>(sm + off + (r - lo) * RS + st * 16 + 4 * k4)
                             : make_float4(fill, fill, fill, fill);
        reinterpret_cast<float4*>(base + st * wimg::FLOATS)[(g * 4 + k4) * 8 + rl] = v;
    }
}

// Forward (forward_trace) and the backward deltas (analytic_gradients' delta
// recursion) of 64-sample tiles; activations and deltas go to the scratch rows
// for train_wgrad_kernel, the per-CTA loss sum to loss_partial.
template <bool IMG>
__global__ void __launch_bounds__(kThreads, 1)
    train_fb_kernel(const float* __restrict__ master, const float* __restrict__ x,
                    const float* __restrict__ y, int64_t n, int64_t ld,
                    float* __restrict__ scr, int64_t lds, double* __restrict__ loss_partial) {
    extern __shared__ __align__(16) float sm[];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent launch
    stage_weights(sm, master);
    __syncthreads();
    const int tid = threadIdx.x;
    double loss = 0.0;

    const int64_t tiles = (n + TM - 1) / TM;
    const bool xvec = (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    auto full_tile = [&](int64_t tile) { return tile * TM + TM <= n; };
    // x of a full, aligned tile -> A0 with 16-byte cp.async (no registers); it is
    // issued for the NEXT tile as soon as layer 1 has consumed A0, so the loads
    // fly during layers 2..4 and the backward pass
    auto prefetch_x = [&](int64_t tile) {
        const int64_t t0 = tile * TM;
        for (int e = tid; e < 134 * (TM / 4); e += kThreads) {
            const int r = e / (TM / 4), q = e % (TM / 4);
            const uint32_t dst = (uint32_t)__cvta_generic_to_shared(sm + A0S + r * RS + 4 * q);
            asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst),
                         "l"(x + (int64_t)r * ld + t0 + 4 * q)
                         : "memory");
        }
        asm volatile("cp.async.commit_group;" ::: "memory");
    };
    bool prefetched = false;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t t0 = tile * TM;
        const int valid = (int)(n - t0 < TM ? n - t0 : TM);
        // ---- stage inputs (zeros for dead samples) ------------------------------
        if (prefetched) {
            asm volatile("cp.async.wait_all;" ::: "memory");
        } else if (valid == TM && xvec) {
            for (int e = tid; e < 134 * (TM / 4); e += kThreads) {
                const int r = e / (TM / 4), q = e % (TM / 4);
                reinterpret_cast<float4*>(sm + A0S + r * RS)[q] =
                    __ldg(reinterpret_cast<const float4*>(x + (int64_t)r * ld + t0) + q);
            }
        } else {
            for (int e = tid; e < 134 * TM; e += kThreads) {
                const int r = e / TM, m = e - r * TM;
                sm[A0S + r * RS + m] = m < valid ? __ldg(x + (int64_t)r * ld + t0 + m) : 0.f;
            }
        }
        if (valid == TM && (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(y) & 15) == 0) {
            for (int e = tid; e < 8 * (TM / 4); e += kThreads) {
                const int r = e / (TM / 4), q = e % (TM / 4);
                reinterpret_cast<float4*>(sm + YS + r * RS)[q] =
                    r < 7 ? __ldg(reinterpret_cast<const float4*>(y + (int64_t)r * ld + t0) + q)
                          : make_float4(0.f, 0.f, 0.f, 0.f);
            }
        } else {
            for (int e = tid; e < 8 * TM; e += kThreads) {
                const int r = e / TM, m = e - r * TM;
                sm[YS + r * RS + m] = (r < 7 && m < valid) ? __ldg(y + (int64_t)r * ld + t0 + m) : 0.f;
            }
        }
        __syncthreads();
        // ---- forward (forward_trace) -------------------------------------------------
        dense_l1(sm);
        if constexpr (IMG) {  // x + ones row + zero row, before the prefetch overwrites A0
            write_img(sm, A0S, 0, 134, 0.f, 2, scr, tile);
            write_img(sm, -1, 134, 135, 1.f, 2, scr, tile);
            write_img(sm, -1, 135, 136, 0.f, 2, scr, tile);
        }
        __syncthreads();
        const int64_t next = tile + gridDim.x;
        prefetched = next < tiles && xvec && full_tile(next);
        if (prefetched) prefetch_x(next);
#ifndef DSO_TRAIN_L2_DENSE
        dense_l2_split(sm);
#else
        dense<100, 7, 8, true>(sm, W2S, B2S, A1S, A2S);
#endif
        __syncthreads();
        dense<50, 4, 4, true>(sm, W3S, B3S, A2S, A3S);
        __syncthreads();
        dense<25, 1, 1, false>(sm, W4S, B4S, A3S, OS);
        __syncthreads();
        if constexpr (IMG) {
            write_img(sm, A1S, 0, 100, 0.f, 3, scr, tile);
            write_img(sm, A2S, 100, 150, 0.f, 3, scr, tile);
            write_img(sm, A3S, 150, 175, 0.f, 3, scr, tile);
            write_img(sm, -1, 175, 176, 1.f, 3, scr, tile);
        } else {
            write_rows(sm, A1S, 100, scr + SA1 * lds, lds, t0);
            write_rows(sm, A2S, 50, scr + SA2 * lds, lds, t0);
            write_rows(sm, A3S, 25, scr + SA3 * lds, lds, t0);
        }
        // ---- residual and loss: delta4 = out - y (dead samples 0) -----------------
        if (tid < TM) {
            float l = 0.f;
            for (int r = 0; r < 7; ++r) {
                const float d = tid < valid ? sm[OS + r * RS + tid] - sm[YS + r * RS + tid] : 0.f;
                sm[OS + r * RS + tid] = d;
                l = fmaf(d, d, l);
            }
            sm[OS + 7 * RS + tid] = 0.f;
            loss += 0.5 * (double)l;
        }
        __syncthreads();
        if constexpr (IMG) { write_img(sm, OS, 75, 82, 0.f, 1, scr, tile); write_img(sm, -1, 82, 88, 0.f, 1, scr, tile); } else write_rows(sm, OS, 7, scr + SD4 * lds, lds, t0);
        // ---- d3 = (W4^T d4) .* a3(1-a3), d2, d1 likewise ------------------------------
        float2 r3[4];
        backprop<25, 4, 7, 4>(sm, T4S, OS, A3S, r3);
        __syncthreads();
        store_delta<25, 4>(sm, A3S, r3);
        __syncthreads();
        if constexpr (IMG) write_img(sm, A3S, 50, 75, 0.f, 1, scr, tile); else write_rows(sm, A3S, 25, scr + SD3 * lds, lds, t0);
        float2 r2[7];
        backprop<50, 7, 25, 8>(sm, T3S, A3S, A2S, r2);
        __syncthreads();
        store_delta<50, 7>(sm, A2S, r2);
        __syncthreads();
        if constexpr (IMG) write_img(sm, A2S, 0, 50, 0.f, 1, scr, tile); else write_rows(sm, A2S, 50, scr + SD2 * lds, lds, t0);
        float2 r1[13];
        backprop<100, 13, 50, 16>(sm, T2S, A2S, A1S, r1);
        __syncthreads();
        store_delta<100, 13>(sm, A1S, r1);
        __syncthreads();
        if constexpr (IMG) { write_img(sm, A1S, 0, 100, 0.f, 0, scr, tile); write_img(sm, -1, 100, 104, 0.f, 0, scr, tile); } else write_rows(sm, A1S, 100, scr + SD1 * lds, lds, t0);
        __syncthreads();
    }
    // loss: block reduce of the 64 per-sample-thread partials
    __shared__ double red[kThreads / 32];
    double v = loss;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if ((tid & 31) == 0) red[tid >> 5] = v;
    __syncthreads();
    if (tid == 0) {
        double s = 0.0;
        for (int w = 0; w < kThreads / 32; ++w) s += red[w];
        loss_partial[blockIdx.x] = s;
    }
}

// ---------------------------------------------------------------------------
// Weight gradients gW_l = D_l A_{l-1}^T and bias gradients sum_m D_l, summed
// over a contiguous sample range per CTA (split-K; partials reduced in CTA order
// by reduce_partials).  Chunks of 32 samples are staged TRANSPOSED into shared
// memory (sample-major: one 532-float record per sample holding D1 | A0 | D2 |
// A1 | D3 | A2 | D4 | A3), so a thread's 8x8 output tile accumulates with packed
// FFMA2 over k pairs: {g[n][k], g[n][k+1]} += d[m][n] * {a[m][k], a[m][k+1]}
// (4 LDS.128 per 32 FFMA2).  The next chunk's global loads are issued before
// the current chunk's math (register double-buffering).
constexpr int WG_THREADS = 384;
constexpr int WG_CHUNK = 32;
// Record layout: every operand row block of 8 (one thread tile's n or k block)
// is stored with a 12-float stride, so the 16-byte chunks of consecutive blocks
// fall in different bank groups (a warp's 17 k blocks read in 3 wavefronts).
constexpr int WG_BLK = 12;
constexpr int blk_off(int r) { return (r / 8) * WG_BLK + r % 8; }
// segment starts (in floats): D1 13 blocks | A0 17 | D2 7 | A1 13 | D3 4 | A2 7 | D4 1 | A3 4
constexpr int RD1 = 0, RA0 = RD1 + 13 * WG_BLK, RD2 = RA0 + 17 * WG_BLK, RA1 = RD2 + 7 * WG_BLK,
              RD3 = RA1 + 13 * WG_BLK, RA2 = RD3 + 4 * WG_BLK, RD4 = RA2 + 7 * WG_BLK,
              RA3 = RD4 + 1 * WG_BLK;
constexpr int WG_REC = RA3 + 4 * WG_BLK + 4;  // floats per sample record (16-byte multiple)
static_assert(WG_REC % 4 == 0 && 2 * WG_CHUNK * WG_REC * 4 <= 227 * 1024, "wgrad smem");
constexpr int WG_ROWS = 491;  // rows staged per sample (valid rows only)
constexpr int WG_TILES = 221 + 91 + 28 + 4;
constexpr int WG_F4 = WG_ROWS * (WG_CHUNK / 4);  // float4 loads per chunk
constexpr int WG_LOADS = (WG_F4 + WG_THREADS - 1) / WG_THREADS;

// staged row r (0..490) -> (record offset, global source row, from x?)
__device__ __forceinline__ void wg_row(int r, int& off, int& src, bool& from_x) {
    from_x = false;
    if (r < 100) { off = RD1 + blk_off(r); src = SD1 + r; return; }
    r -= 100;
    if (r < 134) { off = RA0 + blk_off(r); src = r; from_x = true; return; }
    r -= 134;
    if (r < 50) { off = RD2 + blk_off(r); src = SD2 + r; return; }
    r -= 50;
    if (r < 100) { off = RA1 + blk_off(r); src = SA1 + r; return; }
    r -= 100;
    if (r < 25) { off = RD3 + blk_off(r); src = SD3 + r; return; }
    r -= 25;
    if (r < 50) { off = RA2 + blk_off(r); src = SA2 + r; return; }
    r -= 50;
    if (r < 7) { off = RD4 + blk_off(r); src = SD4 + r; return; }
    r -= 7;
    off = RA3 + blk_off(r);
    src = SA3 + r;
}

__global__ void __launch_bounds__(WG_THREADS, 1)
    train_wgrad_kernel(const float* __restrict__ x, int64_t ld, const float* __restrict__ scr,
                       int64_t lds, int64_t n, int64_t per_cta, float* __restrict__ partial) {
    extern __shared__ __align__(16) float sm[];  // [2][WG_CHUNK][WG_REC]
    const int tid = threadIdx.x;
    const int64_t s_lo = (int64_t)blockIdx.x * per_cta;
    const int64_t s_hi = s_lo + per_cta < n ? s_lo + per_cta : n;
    for (int i = tid; i < 2 * WG_CHUNK * WG_REC; i += WG_THREADS) sm[i] = 0.f;  // padding
    // this thread's output tile
    int dOff = 0, aOff = 0, n0 = 0, k0 = 0, layer = -1;
    if (tid < 221) { layer = 0; n0 = 8 * (tid / 17); k0 = 8 * (tid % 17); dOff = RD1; aOff = RA0; }
    else if (tid < 312) { const int u = tid - 221; layer = 1; n0 = 8 * (u / 13); k0 = 8 * (u % 13); dOff = RD2; aOff = RA1; }
    else if (tid < 340) { const int u = tid - 312; layer = 2; n0 = 8 * (u / 7); k0 = 8 * (u % 7); dOff = RD3; aOff = RA2; }
    else if (tid < 344) { const int u = tid - 340; layer = 3; n0 = 0; k0 = 8 * u; dOff = RD4; aOff = RA3; }
    float2 acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = make_float2(0.f, 0.f);
    float bsum[5] = {0.f, 0.f, 0.f, 0.f, 0.f};  // bias threads: rows bt, bt+40, ...
    const int bt = tid - WG_TILES;
    const bool xvec = (ld & 3) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
    float4 st[WG_LOADS];
    auto load = [&](int64_t c0) {
#pragma unroll
        for (int u = 0; u < WG_LOADS; ++u) {
            const int e = tid + u * WG_THREADS;
            float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
            if (e < WG_F4) {
                const int r = e / (WG_CHUNK / 4), q = e % (WG_CHUNK / 4);
                int off, src;
                bool fx;
                wg_row(r, off, src, fx);
                const int64_t m0 = c0 + 4 * q;
                const float* base = fx ? x + (int64_t)src * ld : scr + (int64_t)src * lds;
                if (m0 + 4 <= s_hi && (!fx || xvec)) {
                    v = __ldg(reinterpret_cast<const float4*>(base + m0));
                } else {
                    if (m0 < s_hi) v.x = __ldg(base + m0);
                    if (m0 + 1 < s_hi) v.y = __ldg(base + m0 + 1);
                    if (m0 + 2 < s_hi) v.z = __ldg(base + m0 + 2);
                    if (m0 + 3 < s_hi) v.w = __ldg(base + m0 + 3);
                }
            }
            st[u] = v;
        }
    };
    auto store = [&](float* buf) {
#pragma unroll
        for (int u = 0; u < WG_LOADS; ++u) {
            const int e = tid + u * WG_THREADS;
            if (e < WG_F4) {
                const int r = e / (WG_CHUNK / 4), q = e % (WG_CHUNK / 4);
                int off, src;
                bool fx;
                wg_row(r, off, src, fx);
                float* d = buf + (4 * q) * WG_REC + off;
                d[0] = st[u].x;
                d[WG_REC] = st[u].y;
                d[2 * WG_REC] = st[u].z;
                d[3 * WG_REC] = st[u].w;
            }
        }
    };
    __syncthreads();
    int cur = 0;
    if (s_lo < s_hi) {
        load(s_lo);
        store(sm);
    }
    __syncthreads();
    for (int64_t c0 = s_lo; c0 < s_hi; c0 += WG_CHUNK) {
        const bool more = c0 + WG_CHUNK < s_hi;
        if (more) load(c0 + WG_CHUNK);  // in flight during the math below
        const float* buf = sm + cur * WG_CHUNK * WG_REC;
        if (layer >= 0) {
            // two register stages: sample m+1's operands load while m's FFMA2s issue
            struct Op {
                float4 d0, d1, a0, a1;
            };
            const int dB = dOff + (n0 / 8) * WG_BLK, aB = aOff + (k0 / 8) * WG_BLK;
            auto ld = [&](Op& o, int m) {
                const float* rec = buf + m * WG_REC;
                o.d0 = *reinterpret_cast<const float4*>(rec + dB);
                o.d1 = *reinterpret_cast<const float4*>(rec + dB + 4);
                o.a0 = *reinterpret_cast<const float4*>(rec + aB);
                o.a1 = *reinterpret_cast<const float4*>(rec + aB + 4);
            };
            auto fma = [&](const Op& o) {
                const float dv[8] = {o.d0.x, o.d0.y, o.d0.z, o.d0.w,
                                     o.d1.x, o.d1.y, o.d1.z, o.d1.w};
                const float2 av[4] = {make_float2(o.a0.x, o.a0.y), make_float2(o.a0.z, o.a0.w),
                                      make_float2(o.a1.x, o.a1.y), make_float2(o.a1.z, o.a1.w)};
#pragma unroll
                for (int i = 0; i < 8; ++i)
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        acc[i][j] = ffma2(make_float2(dv[i], dv[i]), av[j], acc[i][j]);
            };
            Op A, B;
            ld(A, 0);
#pragma unroll 1
            for (int m = 0; m < WG_CHUNK; m += 2) {
                ld(B, m + 1);
                fma(A);
                if (m + 2 < WG_CHUNK) ld(A, m + 2);
                fma(B);
            }
        } else if (bt >= 0) {
            // bias gradients: rows of D1 (100) | D2 (50) | D3 (25) | D4 (7) = 182
#pragma unroll
            for (int u = 0; u < 5; ++u) {
                const int r = bt + 40 * u;
                if (r < 182) {
                    const int off = r < 100 ? RD1 + blk_off(r)
                                  : r < 150 ? RD2 + blk_off(r - 100)
                                  : r < 175 ? RD3 + blk_off(r - 150)
                                            : RD4 + blk_off(r - 175);
                    float sacc = 0.f;
                    for (int m = 0; m < WG_CHUNK; ++m) sacc += buf[m * WG_REC + off];
                    bsum[u] += sacc;
                }
            }
        }
        if (more) store(sm + (cur ^ 1) * WG_CHUNK * WG_REC);
        __syncthreads();
        cur ^= 1;
    }
    // ---- this CTA's partial gradient, master layout ------------------------------------
    float* P = partial + (int64_t)blockIdx.x * kMasterFloats;
    if (layer >= 0) {
        const int NO[4] = {100, 50, 25, 7}, KI[4] = {134, 100, 50, 25};
        const int WO[4] = {MW1, MW2, MW3, MW4};
        const int no = NO[layer], ki = KI[layer], wo = WO[layer];
#pragma unroll
        for (int i = 0; i < 8; ++i)
#pragma unroll
            for (int j = 0; j < 4; ++j) {
                const int nn = n0 + i, k = k0 + 2 * j;
                if (nn < no && k < ki) P[wo + nn * ki + k] = acc[i][j].x;
                if (nn < no && k + 1 < ki) P[wo + nn * ki + k + 1] = acc[i][j].y;
            }
    } else if (bt >= 0) {
#pragma unroll
        for (int u = 0; u < 5; ++u) {
            const int r = bt + 40 * u;
            if (r < 182) P[MB1 + r] = bsum[u];
        }
    }
}

// Sum the per-CTA partials in CTA order (deterministic), in double.
// ---------------------------------------------------------------------------
// Weight gradients on the 5th-generation tensor cores (train_wgrad_tc_kernel).
// Per CTA a contiguous range of samples (split-K, partials reduced by
// reduce_partials as for train_wgrad_kernel).  For layer l the contraction over
// samples  gW_l[n][k] = sum_s delta_l[n][s] a_{l-1}[k][s]  is one MMA chain
// D_l[M=128 x N_l] += A[128 x 16] . B[N_l x 16]^T per stage of 16 samples, with
// A = the deltas (rows = output neurons, zero-padded to 128) and B = the layer's
// inputs (rows = input features, zero-padded to N_l = 144 / 112 / 64 / 32, plus
// one row of ones whose column gives the bias gradient sum_s delta_l[n][s]).
// 3xTF32 (hi.hi + hi.lo + lo.hi, FP32 accumulation in TMEM: 352 columns) keeps
// the FP32 result.  A copy warp moves a stage's image (written by
// train_fb_kernel<true> already in the SWIZZLE_NONE K-major core-matrix layout)
// into the stage's hi buffer with eight bulk copies; sixteen loader warps split
// it in place into hi and lo (two stage buffers), one thread issues the MMAs, and
// four warps read the accumulators out at the end.
namespace twg {
constexpr int KS = 16;                      // samples per stage
constexpr int kLoadWarps = 16, kThreadsWG = (kLoadWarps + 2) * 32;  // + MMA warp + copy warp
// two MMA chains: c = 0 is layer 1 (A = d1, B = x + ones), c = 1 the stacked
// layers 2-4 (A = d2|d3|d4, B = a1|a2|a3 + ones); N (multiple of 16, ones row
// included) and D's TMEM column per chain
__host__ __device__ constexpr int NPADC(int c) { return c == 0 ? 144 : 176; }
__host__ __device__ constexpr int TCOLC(int c) { return c == 0 ? 0 : 144; }
// stage layout (floats): A_c [128][KS] at 2048 c, then B_0, B_1; hi part, then lo part
constexpr int BOFF = 2 * 128 * KS;
__host__ __device__ constexpr int AOFFC(int c) { return c * 128 * KS; }
__host__ __device__ constexpr int BREG(int c) { return BOFF + TCOLC(c) * KS; }
// shared-memory base of image segment s (wimg: d1, stacked deltas, x, stacked inputs)
__host__ __device__ constexpr int SEGBASE(int s) { return s < 2 ? AOFFC(s) : BREG(s - 2); }
constexpr int HALF = BOFF + 320 * KS;         // floats of one hi (or lo) part
constexpr int STAGE = 2 * HALF;               // hi + lo
constexpr int NRAW = 3;                       // raw landing buffers (stage images)
constexpr int RAW = STAGE;                    // float offset of raw buffer 0
constexpr int MBF = RAW + NRAW * wimg::FLOATS;  // barriers
constexpr int SMEM_FLOATS = MBF + 32;         // one hi/lo stage + 3 raw images + barriers
constexpr int ITEMS = wimg::FLOATS / 4;       // float4 items per stage image
static_assert(KS == wimg::KS, "stage image and MMA stage agree");
constexpr int PER_T = (ITEMS + kLoadWarps * 32 - 1) / (kLoadWarps * 32);

__device__ __forceinline__ void mb_init(uint64_t* b, int count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(tc::smem_addr(b)), "r"(count)
                 : "memory");
}
__device__ __forceinline__ void mb_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(tc::smem_addr(b))
                 : "memory");
}
__device__ __forceinline__ void mb_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(tc::smem_addr(b)), "r"(parity), "r"(100000u)
            : "memory");
}
// the same without a suspend-time hint (the bulk-copy barriers: polled)
__device__ __forceinline__ void mb_wait_spin(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    while (!done)
        asm volatile(
            "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
            : "=r"(done)
            : "r"(tc::smem_addr(b)), "r"(parity)
            : "memory");
}
}  // namespace twg

__global__ void __launch_bounds__(twg::kThreadsWG, 1)
    train_wgrad_tc_kernel(const float* __restrict__ img, int64_t n, int64_t per,
                          float* __restrict__ partial) {
    using namespace twg;
    extern __shared__ __align__(16) float sm[];
    // barriers: FULL, EMPTY (MMA commit), DONE, LOADED[3] (bulk copies), RFREE[3]
    uint64_t* mb = reinterpret_cast<uint64_t*>(sm + MBF);
    uint32_t* tslot = reinterpret_cast<uint32_t*>(sm + MBF + 20);
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const int64_t s_lo = (int64_t)blockIdx.x * per, s_hi = min(n, s_lo + per);
    const int stages = s_hi > s_lo ? (int)((s_hi - s_lo + KS - 1) / KS) : 0;
    // zero the hi/lo stage (padding rows stay zero; the images carry the ones rows)
    for (int i = tid; i < STAGE / 4; i += kThreadsWG)
        reinterpret_cast<float4*>(sm)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
    if (tid == 0) {
        mb_init(mb + 0, kLoadWarps);  // FULL
        mb_init(mb + 1, 1);           // EMPTY
        mb_init(mb + 2, 1);           // DONE
        for (int i = 0; i < NRAW; ++i) {
            mb_init(mb + 3 + i, 1);            // LOADED[i] (expect_tx)
            mb_init(mb + 6 + i, kLoadWarps);   // RFREE[i]
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (warp == kLoadWarps) tc::tmem_alloc<512>(tslot);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tbase = *tslot;
    // launched as a programmatic dependent of the forward kernel: the prologue above
    // overlaps its tail; the stage images are read only after it has completed
    asm volatile("griddepcontrol.wait;" ::: "memory");

    if (warp < kLoadWarps) {
        // ---- loaders: raw stage image -> the hi/lo stage (once the MMAs of the
        // previous stage are done with it), then the raw buffer is free again ------
        int soff[PER_T];
#pragma unroll
        for (int i = 0; i < PER_T; ++i) {
            const int j = tid + i * kLoadWarps * 32;  // float4 of the stage image
            soff[i] = -1;
            if (j < wimg::FLOATS / 4) {
                int sg = 0;
#pragma unroll
                for (int t = 1; t < 4; ++t) sg = 4 * j >= wimg::OFF(t) ? t : sg;
                soff[i] = SEGBASE(sg) + 4 * j - wimg::OFF(sg);
            }
        }
        float* hi = sm;
        float* lo = sm + HALF;
        for (int it = 0; it < stages; ++it) {
            const int rb = it % NRAW;
            mb_wait_spin(mb + 3 + rb, (uint32_t)((it / NRAW) & 1));
            const float* raw = sm + RAW + rb * wimg::FLOATS;
            float4 v[PER_T];
#pragma unroll
            for (int i = 0; i < PER_T; ++i)
                if (soff[i] >= 0)
                    v[i] = reinterpret_cast<const float4*>(raw)[tid + i * kLoadWarps * 32];
            __syncwarp();
            if (lane == 0) mb_arrive(mb + 6 + rb);  // raw buffer consumed
            if (it > 0) mb_wait_spin(mb + 1, (uint32_t)((it - 1) & 1));  // MMAs of it-1 done
#pragma unroll
            for (int i = 0; i < PER_T; ++i) {
                if (soff[i] < 0) continue;
                const float4 h = make_float4(tc::tf32_hi_finite(v[i].x), tc::tf32_hi_finite(v[i].y),
                                             tc::tf32_hi_finite(v[i].z), tc::tf32_hi_finite(v[i].w));
                *reinterpret_cast<float4*>(hi + soff[i]) = h;
                *reinterpret_cast<float4*>(lo + soff[i]) =
                    make_float4(v[i].x - h.x, v[i].y - h.y, v[i].z - h.z, v[i].w - h.w);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) mb_arrive(mb + 0);
        }
        // every loader's stage writes are ordered before the read-out below reuses the
        // stage memory as its transpose buffer
        asm volatile("bar.sync 2, %0;" ::"n"(kLoadWarps * 32) : "memory");
    } else if (warp == kLoadWarps + 1) {
        // ---- copy warp: stage images into the raw buffers, NRAW stages ahead ------
        if (lane == 0) {
            const int64_t st0 = s_lo / KS;
            for (int it = 0; it < stages; ++it) {
                const int rb = it % NRAW;
                if (it >= NRAW) mb_wait_spin(mb + 6 + rb, (uint32_t)(((it / NRAW) - 1) & 1));
                const uint32_t bar = tc::smem_addr(mb + 3 + rb);
                asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar),
                             "r"((uint32_t)(wimg::FLOATS * 4))
                             : "memory");
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        tc::smem_addr(sm + RAW + rb * wimg::FLOATS)),
                    "l"(img + (st0 + it) * wimg::FLOATS), "r"((uint32_t)(wimg::FLOATS * 4)), "r"(bar)
                    : "memory");
            }
        }
    } else if (lane == 0) {
        // ---- MMA issuer ----------------------------------------------------------
        const uint32_t s0 = tc::smem_addr(sm);
        // the hi/lo stage is fixed: every operand descriptor is a base descriptor plus a
        // compile-time offset in its 16-byte address field (no carry: smem < 256 KB)
        const uint64_t dh = tc::sdesc(s0, 128, (KS / 4) * 128),
                       dl = tc::sdesc(s0 + HALF * 4, 128, (KS / 4) * 128);
        for (int it = 0; it < stages; ++it) {
            mb_wait_spin(mb + 0, (uint32_t)(it & 1));
            tc::fence_after();
#pragma unroll
            for (int l = 0; l < 2; ++l) {
                const uint32_t id = tc::idesc_tf32(128, NPADC(l));
                const uint32_t d = tbase + (uint32_t)TCOLC(l);
#pragma unroll
                for (int kk = 0; kk < KS / 8; ++kk) {
                    const uint64_t ao = (uint64_t)((AOFFC(l) * 4 + kk * 256) >> 4),
                                   bo = (uint64_t)((BREG(l) * 4 + kk * 256) >> 4);
                    const uint64_t ah = dh + ao, al = dl + ao, bh = dh + bo, bl = dl + bo;
                    tc::mma_tf32_ss(d, ah, bh, id, (it > 0 || kk > 0) ? 1u : 0u);
                    tc::mma_tf32_ss(d, ah, bl, id, 1u);
                    tc::mma_tf32_ss(d, al, bh, id, 1u);
                }
            }
            tc::commit(mb + 1);  // EMPTY: the hi/lo stage may be rewritten
        }
        tc::commit(mb + 2);      // DONE
    }
    __syncwarp();
    // ---- accumulators -> this CTA's partial gradient (master layout) ------------
    // per layer: TMEM (lane = output neuron) -> a [128][NPAD + 1] transpose buffer in the
    // now idle stage memory -> global in master order (row-major W[n][k], then the
    // biases), consecutive threads on consecutive addresses
    if (warp < 4) {
        float* out = partial + (int64_t)blockIdx.x * kMasterFloats;
        const int row = 32 * warp + lane;  // output neuron
        if (stages > 0) {
            mb_wait(mb + 2, 0);
            tc::fence_after();
        }
        float* tr = sm;  // the stage and raw buffers are idle now
        // chain c: TMEM columns -> tr[128][NPADC + 1] -> the diagonal blocks in master order
        auto chain = [&](auto cc) {
            constexpr int c = decltype(cc)::value;
            constexpr int P = NPADC(c) + 1;
            for (int c0 = 0; c0 < NPADC(c); c0 += 8) {
                float v[8];
                if (stages > 0) {
                    tc::ld8(tbase + ((uint32_t)(32 * warp) << 16) + (uint32_t)(TCOLC(c) + c0), v);
                    tc::wait_ld();
                } else {
#pragma unroll
                    for (int j = 0; j < 8; ++j) v[j] = 0.f;
                }
#pragma unroll
                for (int j = 0; j < 8; ++j) tr[row * P + c0 + j] = v[j];
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
            // block (rows r0.., columns k0..) of NO x NI, bias in column `bc`
            auto block = [&](int mw, int mb, int NO, int NI, int r0, int k0, int bc) {
                for (int j = row; j < NO * NI; j += 128) out[mw + j] = tr[(r0 + j / NI) * P + k0 + j % NI];
                for (int m = row; m < NO; m += 128) out[mb + m] = tr[(r0 + m) * P + bc];
            };
            if constexpr (c == 0) {
                block(MW1, MB1, 100, 134, 0, 0, 134);
            } else {
                block(MW2, MB2, 50, 100, 0, 0, 175);
                block(MW3, MB3, 25, 50, 50, 100, 175);
                block(MW4, MB4, 7, 25, 75, 150, 175);
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
        };
        chain(std::integral_constant<int, 0>{});
        chain(std::integral_constant<int, 1>{});
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == kLoadWarps) tc::tmem_dealloc<512>(tbase);
}

__global__ void __launch_bounds__(256) reduce_partials(const float* __restrict__ partial, int parts,
                                                    const double* __restrict__ loss_partial,
                                                    int loss_parts, float* __restrict__ grad,
                                                    double* __restrict__ loss_sum) {
    // block = 32 consecutive outputs x 8 slices (warp j sums parts j, j+8, ... in
    // order; lanes read 128 contiguous bytes per part), then a fixed combination
    // ((s0+s4)+(s2+s6)) + ((s1+s5)+(s3+s7)) — deterministic
    __shared__ double red[8][32];
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent launch
    const int lane = threadIdx.x & 31, j = threadIdx.x >> 5;
    const int e = blockIdx.x * 32 + lane;
    double s = 0.0;
    if (e < kMasterFloats) {
#pragma unroll 4
        for (int c = j; c < parts; c += 8) s += partial[(int64_t)c * kMasterFloats + e];
    }
    red[j][lane] = s;
    __syncthreads();
    if (j == 0 && e < kMasterFloats) {
        const double a = (red[0][lane] + red[4][lane]) + (red[2][lane] + red[6][lane]);
        const double b = (red[1][lane] + red[5][lane]) + (red[3][lane] + red[7][lane]);
        grad[e] = (float)(a + b);
    }
    if (blockIdx.x == 0 && j == 0) {  // loss: lane l sums parts l, l+32, ..., fixed butterfly
        double l = 0.0;
        for (int c = lane; c < loss_parts; c += 32) l += loss_partial[c];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        if (lane == 0) *loss_sum = l;
    }
}

__global__ void sgd_apply(float* __restrict__ master, const float* __restrict__ grad, float s) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent launch
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < kMasterFloats) master[e] = fmaf(-s, grad[e], master[e]);
}

// sgd_apply that also writes the updated weight into the training kernel's
// image (the positions train_pack_kernel uses), so the next gradient needs no
// repack; the image's zero padding is never touched.
__global__ void sgd_apply_pack(float* __restrict__ master, const float* __restrict__ grad,
                               float s, float* __restrict__ img) {
    asm volatile("griddepcontrol.wait;" ::: "memory");  // programmatic dependent launch
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e >= kMasterFloats) return;
    const float w = fmaf(-s, grad[e], master[e]);
    master[e] = w;
    if (e < MW2) {
        const int n = e / 134, k = e - n * 134;
        img[W1S + (k * 16 + n / 7) * 8 + n % 7] = w;
    } else if (e < MW3) {
        const int i = e - MW2, n = i / 100, k = i - n * 100;
        img[W2S + (k * 8 + n / 7) * 8 + n % 7] = w;
        img[T2S + (n * 8 + k / 13) * 16 + k % 13] = w;
    } else if (e < MW4) {
        const int i = e - MW3, n = i / 50, k = i - n * 50;
        img[W3S + (k * 8 + n / 4) * 4 + n % 4] = w;
        img[T3S + (n * 8 + k / 7) * 8 + k % 7] = w;
    } else if (e < MB1) {
        const int i = e - MW4, n = i / 25, k = i - n * 25;
        img[W4S + k * 8 + n] = w;
        img[T4S + (n * 8 + k / 4) * 4 + k % 4] = w;
    } else if (e < MB2) {
        img[B1S + (e - MB1)] = w;
    } else if (e < MB3) {
        img[B2S + (e - MB2)] = w;
    } else if (e < MB4) {
        img[B3S + (e - MB3)] = w;
    } else {
        img[B4S + (e - MB4)] = w;
    }
}

}  // namespace

cudaError_t train_prepare(Ctx& cx, int64_t n) {
    if (cx.model.generic) {  // sized by launch_gen_grad's first call: reserve it here
        const GenNet g = gen_net_of(cx.model);
        const int64_t parts = std::max<int64_t>(1, std::min<int64_t>((n + 63) / 64, 2 * cx.num_sms));
        const size_t need = (size_t)parts * (g.nw + g.nb) * sizeof(float) + (size_t)parts * 8 + 256;
        if (cx.train_scratch_bytes < need) {
            cudaFree(cx.train_scratch);
            cx.train_scratch = nullptr;
            cx.train_scratch_bytes = 0;
            cudaError_t e = cudaMalloc(&cx.train_scratch, need);
            if (e != cudaSuccess) return e;
            cx.train_scratch_bytes = need;
        }
        return cudaSuccess;
    }
    const int parts = cx.num_sms;
    const int64_t lds = ((n + TM - 1) / TM) * TM;
    const size_t need = (size_t)parts * kMasterFloats * sizeof(float) + (size_t)parts * sizeof(double) +
                        (size_t)kScratchAlloc * (size_t)(lds > 0 ? lds : TM) * sizeof(float) + 256;
    if (cx.train_scratch_bytes < need) {
        cudaFree(cx.train_scratch);
        cx.train_scratch = nullptr;
        cx.train_scratch_bytes = 0;
        cudaError_t e = cudaMalloc(&cx.train_scratch, need);
        if (e != cudaSuccess) return e;
        cx.train_scratch_bytes = need;
    }
    if (!cx.model.w_train) {
        cudaError_t e = cudaMalloc(&cx.model.w_train, sizeof(float) * A0S);
        if (e != cudaSuccess) return e;
        cx.model.train_dirty = true;
    }
    cudaError_t e = ensure_smem_attr((const void*)train_fb_kernel<false>, cx.device,
                                     (int)((size_t)kSmemFloats * sizeof(float)));
    if (e != cudaSuccess) return e;
    e = ensure_smem_attr((const void*)train_fb_kernel<true>, cx.device,
                         (int)((size_t)kSmemFloats * sizeof(float)));
    if (e != cudaSuccess) return e;
    return ensure_smem_attr((const void*)train_wgrad_kernel, cx.device,
                            (int)((size_t)2 * WG_CHUNK * WG_REC * sizeof(float)));
}

// Launch as a programmatic dependent of the previous kernel in the stream: its CTAs
// may start while the previous grid drains; the kernel calls griddepcontrol.wait
// before it reads that grid's outputs.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    return cudaLaunchKernelEx(&cfg, kernel, ((KArgs)args)...);
}

cudaError_t launch_train_grad(Ctx& cx, const float* x, const float* y, int64_t n, int64_t ld,
                              float* grad, double* loss_sum_dev) {
    if (cx.model.generic) return launch_gen_grad(cx, x, y, n, ld, grad, loss_sum_dev);
    const int parts = cx.num_sms;
    const int64_t lds = ((n + TM - 1) / TM) * TM;  // scratch row length (whole tiles)
    const size_t part_b = (size_t)parts * kMasterFloats * sizeof(float);
    const size_t loss_b = (size_t)parts * sizeof(double);
    // row scratch [357][lds] (FMA-pipe weight gradient) or the stage images (tcgen05)
    const size_t act_b = (size_t)kScratchAlloc * (size_t)(lds > 0 ? lds : TM) * sizeof(float);
    const size_t need = part_b + loss_b + act_b + 256;
    if (cx.train_scratch_bytes < need) {
        cudaFree(cx.train_scratch);
        cx.train_scratch = nullptr;
        cx.train_scratch_bytes = 0;
        cudaError_t e = cudaMalloc(&cx.train_scratch, need);
        if (e != cudaSuccess) return e;
        cx.train_scratch_bytes = need;
    }
    float* partial = (float*)cx.train_scratch;
    double* lp = (double*)(partial + (size_t)parts * kMasterFloats);
    float* act = (float*)(((uintptr_t)(lp + parts) + 255) & ~(uintptr_t)255);
    const size_t smem = (size_t)kSmemFloats * sizeof(float);
    const size_t smem_wg = (size_t)2 * WG_CHUNK * WG_REC * sizeof(float);
    {
        cudaError_t e = ensure_smem_attr(cx.train_tc ? (const void*)train_fb_kernel<true>
                                                     : (const void*)train_fb_kernel<false>,
                                         cx.device, (int)smem);
        if (e != cudaSuccess) return e;
        e = ensure_smem_attr((const void*)train_wgrad_kernel, cx.device, (int)smem_wg);
        if (e != cudaSuccess) return e;
    }
    // grids sized to the batch (small batches launch few CTAs); every launched CTA
    // writes its partial, and the reduction reads exactly those
    const int64_t tiles = (n + TM - 1) / TM;
    const int fb_parts = (int)std::max<int64_t>(1, std::min<int64_t>(parts, tiles));
    if (!cx.model.w_train) {
        cudaError_t e = cudaMalloc(&cx.model.w_train, sizeof(float) * A0S);
        if (e != cudaSuccess) return e;
        cx.model.train_dirty = true;
    }
    if (cx.model.train_dirty) {  // the image is 100 KB: memset + scatter
        cudaError_t e = cudaMemsetAsync(cx.model.w_train, 0, sizeof(float) * A0S, cx.stream);
        if (e != cudaSuccess) return e;
        train_pack_kernel<<<64, kThreads, 0, cx.stream>>>(cx.model.w_master, cx.model.w_train);
        ++cx.launches;
        cx.model.train_dirty = false;
    }
    {
        cudaError_t e = launch_pdl(cx.train_tc ? train_fb_kernel<true> : train_fb_kernel<false>,
                                   dim3(fb_parts), dim3(kThreads), smem, cx.stream,
                                   (const float*)cx.model.w_train, x, y, n, ld, act, lds, lp);
        if (e != cudaSuccess) return e;
    }
    const int64_t chunks = (n + WG_CHUNK - 1) / WG_CHUNK;
    const int wg_parts = (int)std::max<int64_t>(1, std::min<int64_t>(parts, chunks));
    int64_t per = (n + wg_parts - 1) / wg_parts;
    per = ((per + WG_CHUNK - 1) / WG_CHUNK) * WG_CHUNK;
    if (per == 0) per = WG_CHUNK;
    if (cx.train_tc) {
        const size_t smem_tc = (size_t)twg::SMEM_FLOATS * sizeof(float);
        cudaError_t e = ensure_smem_attr((const void*)train_wgrad_tc_kernel, cx.device, (int)smem_tc);
        if (e != cudaSuccess) return e;
        e = launch_pdl(train_wgrad_tc_kernel, dim3(wg_parts), dim3(twg::kThreadsWG), smem_tc,
                       cx.stream, (const float*)act, n, per, partial);
        if (e != cudaSuccess) return e;
    } else {
        train_wgrad_kernel<<<wg_parts, WG_THREADS, smem_wg, cx.stream>>>(x, ld, act, lds, n, per,
                                                                         partial);
    }
    {
        cudaError_t e = launch_pdl(reduce_partials, dim3((kMasterFloats + 31) / 32), dim3(256), 0,
                                   cx.stream, (const float*)partial, wg_parts, (const double*)lp,
                                   fb_parts, grad, loss_sum_dev);
        if (e != cudaSuccess) return e;
    }
    cx.launches += 3;
    return cudaGetLastError();
}

cudaError_t launch_train_apply(Ctx& cx, const float* grad, float lr_scale, bool repack) {
    if (cx.model.generic) return launch_gen_apply(cx, grad, lr_scale);
    if (cx.model.w_train && !cx.model.train_dirty) {
        // update master and the training image together (no repack before the
        // next gradient)
        cudaError_t e = launch_pdl(sgd_apply_pack, dim3((kMasterFloats + 255) / 256), dim3(256), 0,
                                   cx.stream, cx.model.w_master, grad, lr_scale, cx.model.w_train);
        if (e != cudaSuccess) return e;
    } else {
        cx.model.train_dirty = true;
        cudaError_t e = launch_pdl(sgd_apply, dim3((kMasterFloats + 255) / 256), dim3(256), 0,
                                   cx.stream, cx.model.w_master, grad, lr_scale);
        if (e != cudaSuccess) return e;
    }
    ++cx.launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess || !repack) return e;
    cx.model.infer_dirty = true;  // the next inference launch repacks (launch_ws)
    return cudaSuccess;
}

}  // namespace dso_b200
