// probe.cu — FP32 FMA-pipe peak probe (roofline denominator).
//
// MEASURED_PEAKS.json carries HBM bandwidth and cuBLAS bf16 throughput only;
// the hot path here is bound by the FP32 pipe, so the library measures that
// peak itself on the same device, same clocks, right before the benchmark:
// a grid of 148 x 4 CTAs x 256 threads runs 8 independent FMA chains per
// thread (enough ILP to cover the 4-cycle latency at any occupancy).
//   mode 0: scalar FFMA with three distinct register operands
//   mode 1: packed FFMA2 (fma.rn.f32x2)
// Reported as flops (2 per FMA lane-op) / CUDA-event time.
#include "common.cuh"

namespace dso_b200 {

namespace {

template <int MODE>
__global__ void __launch_bounds__(256) fma_probe(float* out, int iters, float s) {
    float2 a[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = make_float2(threadIdx.x * 1e-3f + i, i * 0.5f);
    const float2 m = make_float2(s, s * 0.999f);
    const float2 c = make_float2(1e-7f, -1e-7f);
    for (int it = 0; it < iters; ++it) {
#pragma unroll
        for (int u = 0; u < 16; ++u) {
#pragma unroll
            for (int i = 0; i < 8; ++i) {
                if (MODE == 1) {
                    a[i] = ffma2(a[i], m, c);
                } else {
                    a[i].x = fmaf(a[i].x, m.x, c.x);
                    a[i].y = fmaf(a[i].y, m.y, c.y);
                }
            }
        }
    }
    float acc = 0.f;
#pragma unroll
    for (int i = 0; i < 8; ++i) acc += a[i].x + a[i].y;
    if (acc == 1234.5f) out[0] = acc;  // keep the chains alive
}

}  // namespace

}  // namespace dso_b200

using namespace dso_b200;

extern "C" int32_t dso_probe_fp32_peak(dso_ctx* ctx, int32_t mode, double* tflops) {
    if (!ctx || !tflops) return kInvalidArgument;
    Ctx& c = ctx->c;
    if (cudaSetDevice(c.device) != cudaSuccess) return kCuda;
    float* out = nullptr;
    if (cudaMalloc(&out, 4) != cudaSuccess) return kCuda;
    const int blocks = c.num_sms * 4, threads = 256, iters = 4096;
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto launch = [&]() {
        if (mode == 1)
            fma_probe<1><<<blocks, threads, 0, c.stream>>>(out, iters, 0.9999f);
        else
            fma_probe<0><<<blocks, threads, 0, c.stream>>>(out, iters, 0.9999f);
        ++c.launches;
    };
    launch();  // warm-up (clocks, I-cache)
    launch();
    cudaEventRecord(e0, c.stream);
    const int reps = 5;
    for (int r = 0; r < reps; ++r) launch();
    cudaEventRecord(e1, c.stream);
    cudaError_t err = cudaEventSynchronize(e1);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    cudaFree(out);
    if (err != cudaSuccess) return kCuda;
    // lane-FMAs: blocks*threads*iters*16*8 pairs, 2 lanes each, 2 flops each
    const double flops = (double)reps * blocks * threads * iters * 16.0 * 8.0 * 2.0 * 2.0;
    *tflops = flops / (ms * 1e-3) / 1e12;
    return kOk;
}
