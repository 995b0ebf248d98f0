// Microbenchmark: FFMA vs FFMA2 (pair and scalar-broadcast forms) at 1, 2, 8
// warps per SM sub-partition.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 ffma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
    unsigned long long A = *reinterpret_cast<unsigned long long*>(&a);
    unsigned long long B = *reinterpret_cast<unsigned long long*>(&b);
    unsigned long long Cc = *reinterpret_cast<unsigned long long*>(&c), D;
    asm volatile("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(D) : "l"(A), "l"(B), "l"(Cc));
    return *reinterpret_cast<float2*>(&D);
}

template <int MODE, int CH>
__global__ void probe(float* out, int iters, float s) {
    float2 a[CH];
    for (int i = 0; i < CH; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    float2 w[4];
    for (int i = 0; i < 4; ++i) w[i] = make_float2(s + i * 1e-3f, s * 0.999f - i * 1e-3f);
    float x = s * 1.0001f;
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 4; ++u) {
#pragma unroll
            for (int i = 0; i < CH; ++i) {
                if (MODE == 0) {  // scalar FFMA, 3 distinct regs
                    a[i].x = fmaf(a[i].x, w[u].x, w[(u + 1) & 3].y);
                    a[i].y = fmaf(a[i].y, w[u].y, w[(u + 2) & 3].x);
                } else if (MODE == 1) {  // FFMA2 pair x pair
                    a[i] = ffma2(w[u], w[(u + 1) & 3], a[i]);
                } else {  // FFMA2 scalar-broadcast x pair (the MLP form)
                    a[i] = ffma2(make_float2(x, x), w[u], a[i]);
                }
            }
        }
        x += 1e-7f;
    }
    float acc = 0.f;
    for (int i = 0; i < CH; ++i) acc += a[i].x + a[i].y;
    if (acc == 1234.5f) out[0] = acc;
}

template <int MODE, int CH>
void run(const char* name, int blocks, int threads) {
    float* out;
    cudaMalloc(&out, 4);
    int iters = 2048;
    probe<MODE, CH><<<blocks, threads>>>(out, iters, 0.9999f);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) probe<MODE, CH><<<blocks, threads>>>(out, iters, 0.9999f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double flops = 5.0 * blocks * threads * iters * 4.0 * CH * 2 * 2;
    printf("%-28s blocks %4d threads %4d  %.1f TFLOP/s\n", name, blocks, threads, flops / (ms * 1e-3) / 1e12);
    cudaFree(out);
}

int main() {
    int sms;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int wps : {1, 2, 8}) {
        int threads = 128 * wps;
        run<0, 8>("FFMA scalar", sms, threads);
        run<1, 8>("FFMA2 pair", sms, threads);
        run<2, 8>("FFMA2 bcast", sms, threads);
        run<2, 26>("FFMA2 bcast ILP26", sms, threads);
    }
    return 0;
}
