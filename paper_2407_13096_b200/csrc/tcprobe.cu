// tcprobe.cu — bring-up probe for the tcgen05 building blocks in tc.cuh.
//
// One CTA computes D[128][N] = A[128][K] . B[N][K]^T on the 5th-generation
// tensor core (kind::tf32, A staged in TMEM by tcgen05.st, B in shared memory
// in the SWIZZLE_NONE K-major core-matrix layout), either as a single TF32
// pass or as 3xTF32 (hi.hi + hi.lo + lo.hi), and reports the clock64 cycles of
// `reps` back-to-back MMA chains.  Test/measurement only (not on the product
// path): tests/test_gpu_tc.py checks it against numpy.
#include "common.cuh"
#include "tc.cuh"

namespace dso_b200 {
namespace {

__device__ __forceinline__ void probe_mbar_wait(uint64_t* mbar, uint32_t parity) {
    const uint32_t bar = tc::smem_addr(mbar);
    asm volatile(
        "{\n\t.reg .pred P;\n\tWAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n\t"
        "@!P bra WAIT_%=;\n\t}" ::"r"(bar),
        "r"(parity)
        : "memory");
}

__global__ void __launch_bounds__(128, 1)
    tc_gemm_probe(const float* __restrict__ A, const float* __restrict__ B, float* __restrict__ D,
                  int K, int N, int passes, int reps, long long* cycles) {
    extern __shared__ __align__(128) float sm[];
    float* bh = sm;
    float* bl = sm + N * K;
    uint64_t* mbar = reinterpret_cast<uint64_t*>(sm + 2 * N * K);
    uint32_t* slot = reinterpret_cast<uint32_t*>(mbar + 1);
    const int tid = threadIdx.x, warp = tid >> 5;
    for (int e = tid; e < N * K; e += 128) {
        const int n = e / K, k = e % K;
        const float x = B[e], h = tc::tf32_hi(x);
        const int off = ((n >> 3) * (K >> 2) + (k >> 2)) * 32 + (n & 7) * 4 + (k & 3);
        bh[off] = h;
        bl[off] = x - h;
    }
    if (warp == 0) tc::tmem_alloc<512>(slot);
    if (tid == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(tc::smem_addr(mbar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const uint32_t tb = *slot;
    const int AH = 128, AL = 128 + K;
    for (int c0 = 0; c0 < K; c0 += 8) {
        float h[8], l[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
            const float x = A[tid * K + c0 + i];
            h[i] = tc::tf32_hi(x);
            l[i] = x - h[i];
        }
        tc::st8(tc::taddr(tb, warp * 32, AH + c0), h);
        tc::st8(tc::taddr(tb, warp * 32, AL + c0), l);
    }
    tc::wait_st();
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B (generic) -> tensor core
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    const long long t0 = clock64();
    if (tid == 0) {
        const uint32_t id = tc::idesc_tf32(128, N);
        const uint32_t sh = tc::smem_addr(bh), sl = tc::smem_addr(bl);
        const uint32_t lbo = 128, sbo = (uint32_t)(K >> 2) * 128;
        for (int r = 0; r < reps; ++r)
            for (int kk = 0; kk < K / 8; ++kk) {
                const uint64_t dh = tc::sdesc(sh + kk * 256, lbo, sbo);
                tc::mma_tf32_ts(tb, tb + AH + kk * 8, dh, id, kk > 0 ? 1u : 0u);
                if (passes == 3) {
                    const uint64_t dl = tc::sdesc(sl + kk * 256, lbo, sbo);
                    tc::mma_tf32_ts(tb, tb + AH + kk * 8, dl, id, 1u);
                    tc::mma_tf32_ts(tb, tb + AL + kk * 8, dh, id, 1u);
                }
            }
        tc::commit(mbar);
    }
    __syncwarp();
    probe_mbar_wait(mbar, 0);
    tc::fence_after();
    const long long t1 = clock64();
    for (int c0 = 0; c0 < N; c0 += 8) {
        float v[8];
        tc::ld8(tc::taddr(tb, warp * 32, c0), v);
        tc::wait_ld();
#pragma unroll
        for (int i = 0; i < 8; ++i) D[tid * N + c0 + i] = v[i];
    }
    if (tid == 0 && cycles) cycles[0] = t1 - t0;
    tc::fence_before();
    __syncthreads();
    tc::fence_after();
    if (warp == 0) tc::tmem_dealloc<512>(tb);
}

}  // namespace
}  // namespace dso_b200

using namespace dso_b200;

// Device pointers: A [128][K], B [N][K], D [128][N]; K % 8 == 0, K <= 192,
// N % 16 == 0, 16 <= N <= 128.  cycles (device, optional) gets the MMA time.
extern "C" int32_t dso_debug_tc_gemm(const float* A, const float* B, float* D, int32_t K,
                                     int32_t N, int32_t passes, int32_t reps, long long* cycles) {
    if (K <= 0 || K % 8 || K > 192 || N < 16 || N > 128 || N % 16 || reps < 1) return kInvalidArgument;
    const size_t smem = (size_t)2 * N * K * sizeof(float) + 16;
    if (cudaFuncSetAttribute(tc_gemm_probe, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)smem) != cudaSuccess)
        return kCuda;
    tc_gemm_probe<<<1, 128, smem>>>(A, B, D, K, N, passes, reps, cycles);
    if (cudaGetLastError() != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) return kCuda;
    return 0;
}
