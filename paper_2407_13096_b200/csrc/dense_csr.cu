// dense_csr.cu — dense [126][ld] PTX counts -> slot-sorted CSR rows on the device, so
// dso_pipeline's dense input runs on the tensor-core CSR pipeline (mlp_tc.cuh)
// instead of the FMA-pipe kernel.  One pass over the counts (thread = kernel, a row
// of 32 consecutive kernels per warp load): per block of 256 kernels a block scan
// of the non-zero counts plus a decoupled look-back gives row_ptr, and the entries
// ((count << 7) | slot, increasing slot) are gathered in shared memory and written
// out coalesced.
#include <cub/block/block_scan.cuh>

#include "common.cuh"

namespace dso_b200 {
namespace {

#ifndef DSO_DCSR_BLK
#define DSO_DCSR_BLK 256
#endif
constexpr int kBlk = DSO_DCSR_BLK;

#ifndef DSO_DCSR_MINB
#define DSO_DCSR_MINB 6
#endif
constexpr int kStage = 32 * kBlk;  // entries of a block gathered in shared memory

// One pass (the default): per block of 256 kernels the counts are read once; each
// kernel's first kPer entries wait in shared memory while a block scan and a
// decoupled look-back over the preceding blocks (dynamic block order, so every
// predecessor is running or done) give the block's offset; then row_ptr and the
// entries are written (a kernel with more than kPer non-zeros re-reads its
// column).  status[b]: bits 62-63 = 1 (block aggregate) or 2 (inclusive prefix).
constexpr int kPer = 24;
__device__ __forceinline__ uint64_t ld_acquire(const unsigned long long* p) {
    unsigned long long v;
    asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
    return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, uint64_t v) {
    asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"((unsigned long long)v) : "memory");
}
constexpr uint64_t kAgg = 1ull << 62, kPre = 2ull << 62, kVal = (1ull << 62) - 1;
__global__ void __launch_bounds__(kBlk, DSO_DCSR_MINB) dense_csr_fused_kernel(
    const uint32_t* __restrict__ counts, int64_t n, int64_t ld, uint64_t* __restrict__ row_ptr,
    uint32_t* __restrict__ entries, uint64_t cap, unsigned long long* __restrict__ status,
    unsigned int* __restrict__ ticket, int* __restrict__ flags) {
    using Scan = cub::BlockScan<uint32_t, kBlk>;
    __shared__ typename Scan::TempStorage s_scan;
    // s_tmp[j][thread] (pass A) and the block's gathered entries share one buffer
    __shared__ uint32_t s_buf[kStage];
    static_assert(kPer * kBlk <= kStage, "staging");
    auto s_tmp = reinterpret_cast<uint32_t(*)[kBlk]>(s_buf);
    __shared__ uint64_t s_prefix;
    __shared__ unsigned int s_bid;
    const int tid = threadIdx.x;
    if (tid == 0) s_bid = atomicAdd(ticket, 1u);
    __syncthreads();
    const unsigned int bid = s_bid;
    const int64_t k = (int64_t)bid * kBlk + tid;
    uint32_t c = 0, big = 0;
    if (k < n) {
#pragma unroll 14
        for (int r = 0; r < DSO_COUNT_ROWS; ++r) {
            const uint32_t v = __ldg(counts + (int64_t)r * ld + k);
            if (v) {
                if (c < kPer) s_tmp[c][tid] = (v << 7) | (uint32_t)r;
                ++c;
            }
            big |= v >> 25;
        }
    }
    uint32_t excl, agg;
    Scan(s_scan).ExclusiveSum(c, excl, agg);
    const int any_big = __syncthreads_or(big != 0u);
    if (tid < 32) {
        // decoupled look-back, one warp: lane l inspects block bid - 1 - l; a step
        // covers 32 predecessors (the nearest inclusive prefix plus the aggregates
        // of the blocks after it)
        const int lane = tid;
        if (lane == 0) {
            if (any_big) atomicOr(flags, 1);
            st_release(status + bid, (bid == 0 ? kPre : kAgg) | agg);
        }
        uint64_t prefix = 0;
        if (bid > 0) {
            for (int64_t j = (int64_t)bid - 1 - lane;; j -= 32) {
                uint64_t st = j >= 0 ? ld_acquire(status + j) : kPre;
                while (__any_sync(0xffffffffu, (st >> 62) == 0))
                    if ((st >> 62) == 0) st = ld_acquire(status + j);
                const uint32_t pre = __ballot_sync(0xffffffffu, (st >> 62) == 2);
                const int first = pre ? __ffs(pre) - 1 : 31;
                uint64_t v = lane <= first ? (st & kVal) : 0;
#pragma unroll
                for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
                prefix += v;
                if (pre) break;
            }
            if (lane == 0) st_release(status + bid, kPre | (prefix + agg));
        }
        if (lane == 0) s_prefix = prefix;
    }
    __syncthreads();
    const uint64_t base = s_prefix;
    if (k < n) row_ptr[k] = base + excl;
    if (k == n - 1) row_ptr[n] = base + excl + c;
    if (any_big) return;  // the caller runs the dense kernels
    if (base + agg > cap) {  // the entry buffer is too small: the caller regrows and reruns
        if (tid == 0) atomicOr(flags, 2);
        return;
    }
    const bool staged = agg <= (uint32_t)kStage;  // block-uniform
    uint32_t e[kPer];
#pragma unroll
    for (int j = 0; j < kPer; ++j) e[j] = (uint32_t)j < c ? s_tmp[j][tid] : 0u;
    __syncthreads();  // s_tmp is overwritten by the gathered entries below
    if (k < n) {
        uint32_t* dst = staged ? s_buf + excl : entries + base + excl;
        if (c <= (uint32_t)kPer) {
#pragma unroll
            for (int j = 0; j < kPer; ++j)
                if ((uint32_t)j < c) dst[j] = e[j];
        } else {
            uint32_t p = 0;
            for (int r = 0; r < DSO_COUNT_ROWS; ++r) {
                const uint32_t v = __ldg(counts + (int64_t)r * ld + k);
                if (v) dst[p++] = (v << 7) | (uint32_t)r;
            }
        }
    }
    if (staged) {
        __syncthreads();
        for (uint32_t i = tid; i < agg; i += kBlk) entries[base + i] = s_buf[i];
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
    const int64_t nb = (n + kBlk - 1) / kBlk;
    // [row_ptr (n+1) | status (nb) | ticket, flags | entries]
    auto al = [](size_t b) { return (b + 255) & ~(size_t)255; };
    const size_t o_st = al((size_t)(n + 1) * 8), o_fl = o_st + al((size_t)nb * 8),
                 o_ent = o_fl + 256;
    auto grow = [&](size_t need) -> cudaError_t {
        if (cx.dcsr_bytes >= need) return cudaSuccess;
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
    cudaError_t e = grow(o_ent + (size_t)n * 4 * 32);  // room for ~32 entries per kernel
    if (e != cudaSuccess) return e;
    for (int attempt = 0; attempt < 2; ++attempt) {
        char* base = (char*)cx.dcsr_scratch;
        uint64_t* rp = (uint64_t*)base;
        unsigned long long* status = (unsigned long long*)(base + o_st);
        unsigned int* ticket = (unsigned int*)(base + o_fl);
        int* flags = (int*)(base + o_fl + 16);
        uint32_t* ent = (uint32_t*)(base + o_ent);
        const uint64_t cap = (uint64_t)((cx.dcsr_bytes - o_ent) / 4);
        if ((e = cudaMemsetAsync(base + o_st, 0, o_ent - o_st, cx.stream)) != cudaSuccess) return e;
        dense_csr_fused_kernel<<<(unsigned)nb, kBlk, 0, cx.stream>>>(counts, n, ld, rp, ent, cap,
                                                                       status, ticket, flags);
        ++cx.launches;
        // the field check and the entry count decide the path / the buffer
        struct {
            uint64_t total;
            int flags;
        } h{};
        if ((e = cudaMemcpyAsync(&h.total, rp + n, 8, cudaMemcpyDeviceToHost, cx.stream)) != cudaSuccess ||
            (e = cudaMemcpyAsync(&h.flags, flags, 4, cudaMemcpyDeviceToHost, cx.stream)) != cudaSuccess ||
            (e = cudaStreamSynchronize(cx.stream)) != cudaSuccess)
            return e;
        if (h.flags & 1) return cudaSuccess;  // a count >= 2^25: the caller runs the dense kernels
        if (h.flags & 2) {                    // more entries than the buffer holds: regrow, rerun
            if ((e = grow(o_ent + (size_t)(h.total + 4) * 4)) != cudaSuccess) return e;
            continue;
        }
        *done = true;
        return launch_pipeline_csr(cx, rp, ent, 0, dcgm, n, ld, eta, K, params, clamped, idx,
                                   cost, energy, time, ld);
    }
    return cudaErrorUnknown;  // unreachable: the second pass has room for every entry
}

}  // namespace dso_b200
