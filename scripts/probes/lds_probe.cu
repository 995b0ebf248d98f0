// lds_probe.cu — shared-memory wavefront cost of the load patterns the MLP and
// sweep loops can use (run under ncu, metric
// l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum, one kernel per pattern).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o lds_probe lds_probe.cu
// Each kernel: 1 warp per CTA, 1 CTA, 64 loads of the pattern; wavefronts/load
// = metric / (64 * loads-per-iteration).  Address patterns (16-byte units u):
//   P0 uniform                       all lanes u = 0
//   P1 two halves                    u = lane / 16           (2 distinct)
//   P2 two interleaved               u = lane & 1
//   P3 16 distinct, halves duplicate u = lane % 16
//   P4 16 distinct, pairs duplicate  u = lane / 2
//   P5 4 distinct (quarters)         u = lane / 8
//   P6 4 distinct interleaved        u = lane & 3
//   P7 per-lane contiguous           u = lane
//   P8 4 distinct, 512 B apart       u = (lane & 3) * 32   (bank-conflicting)
//   P9 8 distinct interleaved        u = lane & 7
#include <cstdio>

template <int P>
__device__ __forceinline__ int unit_of(int lane) {
    switch (P) {
        case 0: return 0;
        case 1: return lane / 16;
        case 2: return lane & 1;
        case 3: return lane % 16;
        case 4: return lane / 2;
        case 5: return lane / 8;
        case 6: return lane & 3;
        case 7: return lane;
        case 8: return (lane & 3) * 32;
        default: return lane & 7;
    }
}

template <int P, int W>  // W = vector width in floats (1, 2, 4)
__global__ void probe(float* out, int salt) {
    __shared__ __align__(16) float s[4096];
    for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = (float)(i ^ salt);
    __syncthreads();
    const int lane = threadIdx.x & 31;
    // byte offset: 16-byte unit for W=4, 8-byte unit for W=2, 4-byte unit for W=1
    const int off = unit_of<P>(lane) * W;
    float acc = 0.f;
#pragma unroll 1
    for (int it = 0; it < 64; ++it) {
        const int base = (it & 7) * 512 + off;  // stays in range, same bank phase
        if (W == 4) {
            float4 v = *reinterpret_cast<const float4*>(s + base);
            acc += v.x + v.y + v.z + v.w;
        } else if (W == 2) {
            float2 v = *reinterpret_cast<const float2*>(s + base);
            acc += v.x + v.y;
        } else {
            acc += s[base];
        }
        __syncwarp();
    }
    out[threadIdx.x] = acc;
}

template <int P>
void run_p(float* d) {
    probe<P, 4><<<1, 32>>>(d, P);
    probe<P, 2><<<1, 32>>>(d, P);
    probe<P, 1><<<1, 32>>>(d, P);
}

int main() {
    float* d;
    cudaMalloc(&d, 4096);
    run_p<0>(d); run_p<1>(d); run_p<2>(d); run_p<3>(d); run_p<4>(d);
    run_p<5>(d); run_p<6>(d); run_p<7>(d); run_p<8>(d); run_p<9>(d);
    cudaDeviceSynchronize();
    printf("done %s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
