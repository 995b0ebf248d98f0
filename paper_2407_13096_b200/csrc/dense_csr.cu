// dense_csr.cu — dense [126][ld] PTX counts -> slot-sorted CSR rows on the device, so
// dso_pipeline's dense input runs on the tensor-core CSR pipeline (mlp_tc.cuh)
// instead of the FMA-pipe kernel: one pass counts each kernel's non-zero slots,
// a device scan turns the counts into row_ptr, a second pass writes the entries
// ((count << 7) | slot, increasing slot).  Both passes read the counts coalesced
// (thread = kernel, a row of 32 consecutive kernels per warp load).
#include <cub/device/device_scan.cuh>

#include "common.cuh"

namespace dso_b200 {
namespace {

constexpr int kBlk = 256;

__global__ void __launch_bounds__(kBlk) dense_nnz_kernel(const uint32_t* __restrict__ counts,
                                                         int64_t n, int64_t ld,
                                                         uint64_t* __restrict__ nnz,
                                                         int* __restrict__ wide) {
    const int64_t k = (int64_t)blockIdx.x * kBlk + threadIdx.x;
    if (k > n) return;
    if (k == n) {  // the scan's last element: row_ptr[n] = total
        nnz[n] = 0;
        return;
    }
    uint32_t c = 0, big = 0;
#pragma unroll 14
    for (int r = 0; r < DSO_COUNT_ROWS; ++r) {
        const uint32_t v = __ldg(counts + (int64_t)r * ld + k);
        c += v != 0u;
        big |= v >> 25;
    }
    nnz[k] = c;
    if (big) *wide = 1;
}

// Entries of a block of 256 kernels are contiguous in the output: they are
// gathered in shared memory (thread = kernel, at its row's offset) and written out
// coalesced — direct per-kernel writes would leave 4-byte pieces of 32 kernels'
// rows per store instruction (partial sectors).  A block with more than kStage
// entries writes directly.
constexpr int kStage = 8192;
__global__ void __launch_bounds__(kBlk) dense_fill_kernel(const uint32_t* __restrict__ counts,
                                                          int64_t n, int64_t ld,
                                                          const uint64_t* __restrict__ row_ptr,
                                                          uint32_t* __restrict__ entries) {
    __shared__ uint32_t s_ent[kStage];
    const int64_t k0 = (int64_t)blockIdx.x * kBlk, k = k0 + threadIdx.x;
    const int64_t k1 = k0 + kBlk < n ? k0 + kBlk : n;
    const uint64_t b0 = row_ptr[k0], b1 = row_ptr[k1];
    const bool staged = b1 - b0 <= (uint64_t)kStage;
    if (k < n) {
        const uint64_t p0 = row_ptr[k];
        uint32_t* dst = staged ? s_ent : entries + p0;
        int p = staged ? (int)(p0 - b0) : 0;
#pragma unroll 14
        for (int r = 0; r < DSO_COUNT_ROWS; ++r) {
            const uint32_t v = __ldg(counts + (int64_t)r * ld + k);
            if (v) dst[p++] = (v << 7) | (uint32_t)r;
        }
    }
    if (staged) {
        __syncthreads();
        const int tot = (int)(b1 - b0);
        for (int i = threadIdx.x; i < tot; i += kBlk) entries[b0 + i] = s_ent[i];
    }
}

}  // namespace

cudaError_t launch_pipeline_dense_via_csr(Ctx& cx, const uint32_t* counts, const float* dcgm,
                                          int64_t n, int64_t ld, float eta, float K,
                                          float* params, uint8_t* clamped, int32_t* idx,
                                          float* cost, float* energy, float* time, bool* done) {
    *done = false;
    if (n <= 0) {
        *done = true;
        return cudaSuccess;
    }
    size_t scan_b = 0;
    cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, scan_b, (uint64_t*)nullptr,
                                                  (uint64_t*)nullptr, (int64_t)(n + 1), cx.stream);
    if (e != cudaSuccess) return e;
    // [nnz (n+1) | row_ptr (n+1) | wide flag | scan temp | entries (grown after the scan)]
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t o_rp = al((size_t)(n + 1) * 8), o_flag = o_rp + al((size_t)(n + 1) * 8),
                 o_tmp = o_flag + 256, o_ent = o_tmp + al(scan_b);
    bool moved = false;  // set when grow() replaced the allocation
    auto grow = [&](size_t need) -> cudaError_t {
        if (cx.dcsr_bytes >= need) return cudaSuccess;
        moved = true;
        cudaError_t r = cudaStreamSynchronize(cx.stream);
        if (r != cudaSuccess) return r;
        cudaFree(cx.dcsr_scratch);
        cx.dcsr_scratch = nullptr;
        cx.dcsr_bytes = 0;
        r = cudaMalloc(&cx.dcsr_scratch, need);
        if (r != cudaSuccess) return r;
        cx.dcsr_bytes = need;
        return cudaSuccess;
    };
    if ((e = grow(o_ent + (size_t)n * 4 * 32)) != cudaSuccess) return e;  // room for ~32 per kernel
    char* base = (char*)cx.dcsr_scratch;
    uint64_t* nnz = (uint64_t*)base;
    uint64_t* rp = (uint64_t*)(base + o_rp);
    int* wide = (int*)(base + o_flag);
    if ((e = cudaMemsetAsync(wide, 0, sizeof(int), cx.stream)) != cudaSuccess) return e;
    const unsigned blocks = (unsigned)((n + 1 + kBlk - 1) / kBlk);
    dense_nnz_kernel<<<blocks, kBlk, 0, cx.stream>>>(counts, n, ld, nnz, wide);
    ++cx.launches;
    if ((e = cub::DeviceScan::ExclusiveSum(base + o_tmp, scan_b, nnz, rp, (int64_t)(n + 1),
                                           cx.stream)) != cudaSuccess)
        return e;
    ++cx.launches;
    // the total (row_ptr[n]) and the field check decide the entry buffer / the path
    struct {
        uint64_t total;
        int wide;
    } h{};
    if ((e = cudaMemcpyAsync(&h.total, rp + n, 8, cudaMemcpyDeviceToHost, cx.stream)) != cudaSuccess ||
        (e = cudaMemcpyAsync(&h.wide, wide, 4, cudaMemcpyDeviceToHost, cx.stream)) != cudaSuccess ||
        (e = cudaStreamSynchronize(cx.stream)) != cudaSuccess)
        return e;
    if (h.wide) return cudaSuccess;  // a count >= 2^25: the caller runs the dense kernels
    moved = false;
    if ((e = grow(o_ent + (size_t)(h.total + 4) * 4)) != cudaSuccess) return e;
    base = (char*)cx.dcsr_scratch;
    nnz = (uint64_t*)base;
    rp = (uint64_t*)(base + o_rp);
    wide = (int*)(base + o_flag);
    if (moved) {
        // the buffer was regrown: row_ptr lived in the old allocation, recompute it
        if ((e = cudaMemsetAsync(wide, 0, sizeof(int), cx.stream)) != cudaSuccess) return e;
        dense_nnz_kernel<<<blocks, kBlk, 0, cx.stream>>>(counts, n, ld, nnz, wide);
        if ((e = cub::DeviceScan::ExclusiveSum(base + o_tmp, scan_b, nnz, rp, (int64_t)(n + 1),
                                               cx.stream)) != cudaSuccess)
            return e;
        cx.launches += 2;
    }
    uint32_t* ent = (uint32_t*)(base + o_ent);
    dense_fill_kernel<<<(unsigned)((n + kBlk - 1) / kBlk), kBlk, 0, cx.stream>>>(counts, n, ld, rp,
                                                                                 ent);
    ++cx.launches;
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
    *done = true;
    return launch_pipeline_csr(cx, rp, ent, 0, dcgm, n, ld, eta, K, params, clamped, idx, cost,
                               energy, time, ld);
}

}  // namespace dso_b200
