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

#include "common.cuh"

namespace dso_b200 {

namespace {

constexpr int TM = 64;       // samples per tile
constexpr int RS = 68;       // row stride (floats) of activation buffers (bank padding)
constexpr int RS2 = RS / 2;  // in float2 units
constexpr int kThreads = 256;

// packed weights (floats): layer l stored [K][8 groups][TNP], neuron n = TN*g + t
constexpr int W1S = 0;                     // [134][8][16], TN 13
constexpr int W2S = W1S + 134 * 8 * 16;    // [100][8][8],  TN 7
constexpr int W3S = W2S + 100 * 8 * 8;     // [50][8][4],   TN 4
constexpr int W4S = W3S + 50 * 8 * 4;      // [25][8],      TN 1
constexpr int B1S = W4S + 25 * 8;          // [104]
constexpr int B2S = B1S + 104;             // [56]
constexpr int B3S = B2S + 56;              // [32]
constexpr int B4S = B3S + 32;              // [8]
constexpr int A0S = B4S + 8;               // [140][RS]  (rows 134..139 zero)
constexpr int A1S = A0S + 140 * RS;        // [104][RS]
constexpr int A2S = A1S + 104 * RS;        // [56][RS]
constexpr int A3S = A2S + 56 * RS;         // [32][RS]
constexpr int OS = A3S + 32 * RS;          // [8][RS]   output, then delta4
constexpr int YS = OS + 8 * RS;            // [8][RS]   targets
constexpr int kSmemFloats = YS + 8 * RS;
static_assert(A0S % 4 == 0 && W2S % 4 == 0 && W3S % 4 == 0 && W4S % 4 == 0, "alignment");

// master (reference) layout offsets: W1 | W2 | W3 | W4 | b1 | b2 | b3 | b4
constexpr int MW1 = 0, MW2 = MW1 + 100 * 134, MW3 = MW2 + 50 * 100, MW4 = MW3 + 25 * 50;
constexpr int MB1 = MW4 + 7 * 25, MB2 = MB1 + 100, MB3 = MB2 + 50, MB4 = MB3 + 25;
constexpr int kMasterFloats = MB4 + 7;  // 20007

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }

__device__ void stage_weights(float* sm, const float* __restrict__ m) {
    for (int i = threadIdx.x; i < A0S; i += kThreads) sm[i] = 0.f;
    __syncthreads();
    for (int e = threadIdx.x; e < 100 * 134; e += kThreads) {
        const int n = e / 134, k = e - n * 134;
        sm[W1S + (k * 8 + n / 13) * 16 + n % 13] = m[MW1 + e];
    }
    for (int e = threadIdx.x; e < 50 * 100; e += kThreads) {
        const int n = e / 100, k = e - n * 100;
        sm[W2S + (k * 8 + n / 7) * 8 + n % 7] = m[MW2 + e];
    }
    for (int e = threadIdx.x; e < 25 * 50; e += kThreads) {
        const int n = e / 50, k = e - n * 50;
        sm[W3S + (k * 8 + n / 4) * 4 + n % 4] = m[MW3 + e];
    }
    for (int e = threadIdx.x; e < 7 * 25; e += kThreads) {
        const int n = e / 25, k = e - n * 25;
        sm[W4S + k * 8 + n] = m[MW4 + e];
    }
    for (int i = threadIdx.x; i < 100; i += kThreads) sm[B1S + i] = m[MB1 + i];
    for (int i = threadIdx.x; i < 50; i += kThreads) sm[B2S + i] = m[MB2 + i];
    for (int i = threadIdx.x; i < 25; i += kThreads) sm[B3S + i] = m[MB3 + i];
    for (int i = threadIdx.x; i < 7; i += kThreads) sm[B4S + i] = m[MB4 + i];
    // zero padding rows of A0 (k = 134..139 feed gW1's 14-wide k blocks)
    for (int i = threadIdx.x; i < 6 * RS; i += kThreads) sm[A0S + 134 * RS + i] = 0.f;
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
#pragma unroll 1
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

// delta_l[k][m] = (sum_n W[n][k] delta_{l+1}[n][m]) * a_l[k][m] (1 - a_l[k][m]),
// thread = (sample pair, group of TK consecutive k); weights read as scalar
// broadcasts from the packed [K][8][TNP] layout of layer l.  Returns values in
// registers (the caller writes them over a_l after a barrier).
template <int KOUT, int TK, int NIN, int TN, int TNP>
__device__ __forceinline__ void backprop(const float* sm, int woff, int din_off, int a_off,
                                         float2 (&res)[TK]) {
    const int mp = threadIdx.x & 31, kg = threadIdx.x >> 5;
    const float2* d2 = reinterpret_cast<const float2*>(sm + din_off);
    const float2* a2 = reinterpret_cast<const float2*>(sm + a_off);
#pragma unroll
    for (int t = 0; t < TK; ++t) res[t] = f2(0.f, 0.f);
#pragma unroll 2
    for (int n = 0; n < NIN; ++n) {
        const float2 d = d2[n * RS2 + mp];
        const int gofs = (n / TN) * TNP + n % TN;
#pragma unroll
        for (int t = 0; t < TK; ++t) {
            const int k = kg * TK + t;
            if (k < KOUT) {
                const float w = sm[woff + k * 8 * TNP + gofs];
                res[t] = ffma2(d, f2(w, w), res[t]);
            }
        }
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

// acc[i][j] += sum_m D[n0+i][m] * A[k0+j][m] over the 64 samples of the tile.
template <int TNB, int TKB>
__device__ __forceinline__ void outer_acc(const float* sm, int d_off, int a_off, int n0, int k0,
                                          float (&acc)[TNB][TKB]) {
#pragma unroll 2
    for (int mq = 0; mq < TM / 4; ++mq) {
        float4 d[TNB], a[TKB];
#pragma unroll
        for (int i = 0; i < TNB; ++i)
            d[i] = reinterpret_cast<const float4*>(sm + d_off + (n0 + i) * RS)[mq];
#pragma unroll
        for (int j = 0; j < TKB; ++j)
            a[j] = reinterpret_cast<const float4*>(sm + a_off + (k0 + j) * RS)[mq];
#pragma unroll
        for (int i = 0; i < TNB; ++i)
#pragma unroll
            for (int j = 0; j < TKB; ++j) {
                acc[i][j] = fmaf(d[i].x, a[j].x, acc[i][j]);
                acc[i][j] = fmaf(d[i].y, a[j].y, acc[i][j]);
                acc[i][j] = fmaf(d[i].z, a[j].z, acc[i][j]);
                acc[i][j] = fmaf(d[i].w, a[j].w, acc[i][j]);
            }
    }
}

__device__ __forceinline__ float row_sum(const float* sm, int off) {
    float s = 0.f;
#pragma unroll
    for (int mq = 0; mq < TM / 4; ++mq) {
        const float4 v = reinterpret_cast<const float4*>(sm + off)[mq];
        s += (v.x + v.y) + (v.z + v.w);
    }
    return s;
}

__global__ void __launch_bounds__(kThreads, 1)
    train_grad_kernel(const float* __restrict__ master, const float* __restrict__ x,
                      const float* __restrict__ y, int64_t n, int64_t ld,
                      float* __restrict__ partial, double* __restrict__ loss_partial) {
    extern __shared__ __align__(16) float sm[];
    stage_weights(sm, master);
    __syncthreads();
    const int tid = threadIdx.x;
    // owned gradient blocks (threads 0..249; 250..255 own only a bias slot)
    const bool own = tid < 250;
    const int nb = tid / 10, kb = tid % 10;
    float g1[4][14], g2[2][10], g3[1][5], g4[1][1], gb = 0.f;
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 14; ++j) g1[i][j] = 0.f;
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
        for (int j = 0; j < 10; ++j) g2[i][j] = 0.f;
#pragma unroll
    for (int j = 0; j < 5; ++j) g3[0][j] = 0.f;
    g4[0][0] = 0.f;
    double loss = 0.0;

    const int64_t tiles = (n + TM - 1) / TM;
    for (int64_t tile = blockIdx.x; tile < tiles; tile += gridDim.x) {
        const int64_t t0 = tile * TM;
        const int valid = (int)(n - t0 < TM ? n - t0 : TM);
        // ---- stage inputs (zeros for dead samples) ------------------------------
        for (int e = tid; e < 134 * TM; e += kThreads) {
            const int r = e / TM, m = e - r * TM;
            sm[A0S + r * RS + m] = m < valid ? __ldg(x + (int64_t)r * ld + t0 + m) : 0.f;
        }
        for (int e = tid; e < 8 * TM; e += kThreads) {
            const int r = e / TM, m = e - r * TM;
            sm[YS + r * RS + m] = (r < 7 && m < valid) ? __ldg(y + (int64_t)r * ld + t0 + m) : 0.f;
        }
        __syncthreads();
        // ---- forward (forward_trace) -------------------------------------------------
        dense<134, 13, 16, true>(sm, W1S, B1S, A0S, A1S);
        __syncthreads();
        dense<100, 7, 8, true>(sm, W2S, B2S, A1S, A2S);
        __syncthreads();
        dense<50, 4, 4, true>(sm, W3S, B3S, A2S, A3S);
        __syncthreads();
        dense<25, 1, 1, false>(sm, W4S, B4S, A3S, OS);
        __syncthreads();
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
        // ---- layer 4: gW4 += d4 a3^T; d3 = (W4^T d4) .* a3(1-a3) ---------------------
        if (tid < 175) {
            float a4[1][1] = {{0.f}};
            outer_acc<1, 1>(sm, OS, A3S, tid / 25, tid % 25, a4);
            g4[0][0] += a4[0][0];
        }
        float2 r3[4];
        backprop<25, 4, 7, 1, 1>(sm, W4S, OS, A3S, r3);
        __syncthreads();
        store_delta<25, 4>(sm, A3S, r3);
        __syncthreads();
        // ---- layer 3: gW3 += d3 a2^T; d2 = (W3^T d3) .* a2(1-a2) ---------------------
        if (own) outer_acc<1, 5>(sm, A3S, A2S, nb, kb * 5, g3);
        float2 r2[7];
        backprop<50, 7, 25, 4, 4>(sm, W3S, A3S, A2S, r2);
        __syncthreads();
        store_delta<50, 7>(sm, A2S, r2);
        __syncthreads();
        // ---- layer 2: gW2 += d2 a1^T; d1 = (W2^T d2) .* a1(1-a1) ---------------------
        if (own) outer_acc<2, 10>(sm, A2S, A1S, nb * 2, kb * 10, g2);
        float2 r1[13];
        backprop<100, 13, 50, 7, 8>(sm, W2S, A2S, A1S, r1);
        __syncthreads();
        store_delta<100, 13>(sm, A1S, r1);
        __syncthreads();
        // ---- layer 1: gW1 += d1 a0^T; biases -------------------------------------------
        if (own) outer_acc<4, 14>(sm, A1S, A0S, nb * 4, kb * 14, g1);
        if (tid < 100)
            gb += row_sum(sm, A1S + tid * RS);
        else if (tid < 150)
            gb += row_sum(sm, A2S + (tid - 100) * RS);
        else if (tid < 175)
            gb += row_sum(sm, A3S + (tid - 150) * RS);
        else if (tid < 182)
            gb += row_sum(sm, OS + (tid - 175) * RS);
        __syncthreads();
    }
    // ---- write this CTA's partial gradient (master layout) ----------------------------
    float* P = partial + (int64_t)blockIdx.x * kMasterFloats;
    if (own) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
#pragma unroll
            for (int j = 0; j < 14; ++j) {
                const int nn = nb * 4 + i, k = kb * 14 + j;
                if (k < 134) P[MW1 + nn * 134 + k] = g1[i][j];
            }
#pragma unroll
        for (int i = 0; i < 2; ++i)
#pragma unroll
            for (int j = 0; j < 10; ++j) P[MW2 + (nb * 2 + i) * 100 + kb * 10 + j] = g2[i][j];
#pragma unroll
        for (int j = 0; j < 5; ++j) P[MW3 + nb * 50 + kb * 5 + j] = g3[0][j];
    }
    if (tid < 175) P[MW4 + (tid / 25) * 25 + tid % 25] = g4[0][0];
    if (tid < 182) P[MB1 + tid] = gb;
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

// Sum the per-CTA partials in CTA order (deterministic), in double.
__global__ void reduce_partials(const float* __restrict__ partial, int parts,
                                const double* __restrict__ loss_partial, float* __restrict__ grad,
                                double* __restrict__ loss_sum) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < kMasterFloats) {
        double s = 0.0;
        for (int c = 0; c < parts; ++c) s += partial[(int64_t)c * kMasterFloats + e];
        grad[e] = (float)s;
    }
    if (e == 0) {
        double s = 0.0;
        for (int c = 0; c < parts; ++c) s += loss_partial[c];
        *loss_sum = s;
    }
}

__global__ void sgd_apply(float* __restrict__ master, const float* __restrict__ grad, float s) {
    const int e = blockIdx.x * blockDim.x + threadIdx.x;
    if (e < kMasterFloats) master[e] = fmaf(-s, grad[e], master[e]);
}

}  // namespace

cudaError_t launch_train_grad(Ctx& cx, const float* x, const float* y, int64_t n, int64_t ld,
                              float* grad, double* loss_sum_dev) {
    const int parts = cx.num_sms;
    const size_t need = (size_t)parts * kMasterFloats * sizeof(float) + parts * sizeof(double);
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
    static bool attr = false;
    const size_t smem = (size_t)kSmemFloats * sizeof(float);
    if (!attr) {
        cudaError_t e = cudaFuncSetAttribute(train_grad_kernel,
                                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        if (e != cudaSuccess) return e;
        attr = true;
    }
    // CTAs with no tile still write zero partials, so every slot is defined
    train_grad_kernel<<<parts, kThreads, smem, cx.stream>>>(cx.model.w_master, x, y, n, ld,
                                                            partial, lp);
    reduce_partials<<<(kMasterFloats + 255) / 256, 256, 0, cx.stream>>>(partial, parts, lp, grad,
                                                                        loss_sum_dev);
    cx.launches += 2;
    return cudaGetLastError();
}

cudaError_t launch_train_apply(Ctx& cx, const float* grad, float lr_scale) {
    sgd_apply<<<(kMasterFloats + 255) / 256, 256, 0, cx.stream>>>(cx.model.w_master, grad,
                                                                  lr_scale);
    ++cx.launches;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return launch_repack(cx);  // inference kernels see the updated weights
}

}  // namespace dso_b200
