// mlp_gen.cu — the predictor for ANY layer chain (TrainConfig.layer_sizes,
// mlp.hpp:87-89; init_mlp / validate accept any chain, mlp.cpp:184-226), and the
// 64-bit-count feature stage.
//
// The fused engines (mlp.cu ws_kernel, mlp_tc.cuh tc_kernel, train.cu) are
// specialised to the default topology 134-100-50-25-7 (mlp.cpp:177).  Every
// other chain runs here, on the same device model (w_master, the reference
// layout: row-major W_l concatenated, then the biases):
//   * gen_forward_kernel — forward_trace / forward_raw / predict_params
//     (mlp.cpp:17-32,228-253): thread = sample, activations in shared memory
//     ([width][64] double-buffered), weights read as warp-uniform __ldg
//     broadcasts, FP32 with the reference's order (z = W a, then + b; sigmoid
//     1 / (1 + exp(-z)) on hidden layers, identity on the output);
//   * gen_grad_kernel — analytic_gradients + mse_loss (mlp.cpp:259-289): the
//     forward keeps every layer's activations of the block's 64 samples in
//     shared memory, backprop overwrites them with the deltas in place, and the
//     weight / bias gradient sums over the block's samples go into the block's
//     private partial row; gen_reduce sums the rows in block order
//     (deterministic);
//   * featurize_u64_kernel — featurize + as_vector (ptx_features.cpp:311-329,
//     mlp.cpp:158-165) on uint64 counts (KernelInstructionCounts,
//     ptx_features.hpp:31-37): exact integer category totals, one FP64 division
//     per count, rounded once to float;
//   * csr_to_dense_kernel — CSR entries scattered into dense [126][ld] counts
//     for the staged pipeline of a non-default model.
// Limits of the generic engine: <= 8 layers, widths <= 256, sum of widths
// <= 700 (dso_set_model rejects larger chains with InvalidModel).
#include <algorithm>
#include <cmath>

#include "common.cuh"

namespace dso_b200 {

namespace {

constexpr int GT = 64;  // samples per block

__device__ __forceinline__ float sigmoid_ref(float z) { return 1.f / (1.f + expf(-z)); }

__global__ void __launch_bounds__(GT) gen_forward_kernel(const float* __restrict__ w, GenNet net,
                                                         const float* __restrict__ stats,
                                                         const float* __restrict__ x, int64_t n,
                                                         int64_t ld, float* __restrict__ raw,
                                                         float* __restrict__ params,
                                                         uint8_t* __restrict__ clamped,
                                                         int64_t ld_out) {
    extern __shared__ float act[];  // [2][maxw][GT]
    const int t = threadIdx.x;
    const int L = net.layers, out_dim = net.sizes[L];
    for (int64_t base = (int64_t)blockIdx.x * GT; base < n; base += (int64_t)gridDim.x * GT) {
        const int64_t k = base + t;
        const bool live = k < n;
        float* a = act;
        float* b = act + net.maxw * GT;
        for (int i = 0; i < net.sizes[0]; ++i) a[i * GT + t] = live ? x[(int64_t)i * ld + k] : 0.f;
        for (int l = 0; l < L; ++l) {
            const int in = net.sizes[l], out = net.sizes[l + 1];
            const float* W = w + net.woff[l];
            const float* B = w + net.nw + net.boff[l];
            for (int o = 0; o < out; ++o) {
                float z = 0.f;
                for (int i = 0; i < in; ++i) z = fmaf(__ldg(W + o * in + i), a[i * GT + t], z);
                z += __ldg(B + o);
                b[o * GT + t] = l + 1 < L ? sigmoid_ref(z) : z;
            }
            float* s = a;
            a = b;
            b = s;
        }
        if (!live) continue;
        // forward_raw: out * std + mean; predict_params' clamp (mlp.cpp:237-253)
        bool cl = false;
        for (int o = 0; o < out_dim; ++o) {
            const float r = fmaf(a[o * GT + t], stats[out_dim + o], stats[o]);
            if (raw) raw[(int64_t)o * ld_out + k] = r;
            a[o * GT + t] = r;
        }
        if (params && out_dim == DSO_PARAM_ROWS) {
            float p[DSO_PARAM_ROWS];
            for (int o = 0; o < DSO_PARAM_ROWS; ++o) {
                p[o] = a[o * GT + t];
                if (p[o] < 0.f) {
                    p[o] = 0.f;
                    cl = true;
                }
            }
            if (p[5] + p[6] <= 0.f) {
                p[6] = 1e-12f;  // kBetaFloor, mlp.cpp:15
                cl = true;
            }
            for (int o = 0; o < DSO_PARAM_ROWS; ++o) params[(int64_t)o * ld_out + k] = p[o];
            if (clamped) clamped[k] = cl ? 1 : 0;
        }
    }
}

// Batch-sum gradient of 0.5*||out - y||^2 over the block's samples into the
// block's partial row (weights then biases, the master layout), loss into
// loss_part[block].
__global__ void __launch_bounds__(GT) gen_grad_kernel(const float* __restrict__ w, GenNet net,
                                                      const float* __restrict__ x,
                                                      const float* __restrict__ y, int64_t n,
                                                      int64_t ld, float* __restrict__ partial,
                                                      double* __restrict__ loss_part) {
    extern __shared__ float act[];  // layer l at act[aoff[l] * GT], [width][GT]
    const int t = threadIdx.x;
    const int L = net.layers;
    const int64_t np = net.nw + net.nb;
    float* P = partial + (int64_t)blockIdx.x * np;
    for (int64_t e = t; e < np; e += GT) P[e] = 0.f;
    double loss = 0.0;
    for (int64_t base = (int64_t)blockIdx.x * GT; base < n; base += (int64_t)gridDim.x * GT) {
        const int64_t k = base + t;
        const bool live = k < n;
        __syncthreads();  // the previous tile's gradient sums have read act
        for (int i = 0; i < net.sizes[0]; ++i)
            act[i * GT + t] = live ? x[(int64_t)i * ld + k] : 0.f;
        for (int l = 0; l < L; ++l) {
            const int in = net.sizes[l], out = net.sizes[l + 1];
            const float* W = w + net.woff[l];
            const float* B = w + net.nw + net.boff[l];
            const float* a = act + net.aoff[l] * GT;
            float* b = act + net.aoff[l + 1] * GT;
            for (int o = 0; o < out; ++o) {
                float z = 0.f;
                for (int i = 0; i < in; ++i) z = fmaf(__ldg(W + o * in + i), a[i * GT + t], z);
                z += __ldg(B + o);
                b[o * GT + t] = l + 1 < L ? sigmoid_ref(z) : z;
            }
        }
        // output delta (out - y), zero for padding samples; loss
        {
            float* d = act + net.aoff[L] * GT;
            for (int o = 0; o < net.sizes[L]; ++o) {
                const float diff = live ? d[o * GT + t] - y[(int64_t)o * ld + k] : 0.f;
                loss += 0.5 * (double)diff * (double)diff;
                d[o * GT + t] = diff;
            }
        }
        for (int l = L - 1; l >= 0; --l) {
            const int in = net.sizes[l], out = net.sizes[l + 1];
            const float* a = act + net.aoff[l] * GT;
            const float* d = act + net.aoff[l + 1] * GT;
            __syncthreads();  // deltas of layer l+1 complete
            // gW[o][i] += sum_t d[o][t] a[i][t]; gb[o] += sum_t d[o][t]
            for (int p = t; p < out * (in + 1); p += GT) {
                const int o = p / (in + 1), i = p - o * (in + 1);
                float s = 0.f;
                if (i < in) {
                    for (int u = 0; u < GT; ++u) s = fmaf(d[o * GT + u], a[i * GT + u], s);
                    P[net.woff[l] + o * in + i] += s;
                } else {
                    for (int u = 0; u < GT; ++u) s += d[o * GT + u];
                    P[net.nw + net.boff[l] + o] += s;
                }
            }
            if (l == 0) break;
            __syncthreads();  // a_l fully read by the sums above
            // d_l = (W_l^T d_{l+1}) * a_l (1 - a_l), in place over a_l (own column)
            const float* W = w + net.woff[l];
            float* al = act + net.aoff[l] * GT;
            for (int i = 0; i < in; ++i) {
                float s = 0.f;
                for (int o = 0; o < out; ++o) s = fmaf(__ldg(W + o * in + i), d[o * GT + t], s);
                const float av = al[i * GT + t];
                al[i * GT + t] = s * (av * (1.f - av));
            }
        }
    }
    // block loss: fixed-order tree over the block's threads
    __shared__ double red[GT];
    __syncthreads();
    red[t] = loss;
    __syncthreads();
    for (int s = GT / 2; s > 0; s >>= 1) {
        if (t < s) red[t] += red[t + s];
        __syncthreads();
    }
    if (t == 0) loss_part[blockIdx.x] = red[0];
}

__global__ void gen_reduce(const float* __restrict__ partial, int parts, int64_t np,
                           const double* __restrict__ loss_part, float* __restrict__ grad,
                           double* __restrict__ loss_sum) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < np) {
        double s = 0.0;
        for (int c = 0; c < parts; ++c) s += partial[(int64_t)c * np + e];
        grad[e] = (float)s;
    }
    if (e == 0) {
        double l = 0.0;
        for (int c = 0; c < parts; ++c) l += loss_part[c];
        *loss_sum = l;
    }
}

__global__ void gen_apply(float* __restrict__ master, const float* __restrict__ grad, int64_t np,
                          float s) {
    const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (e < np) master[e] = fmaf(-s, grad[e], master[e]);
}

// featurize on uint64 counts [126][ld] (+ DCGM [8][ld]) -> fused [134][ld]
__global__ void featurize_u64_kernel(const uint64_t* __restrict__ counts,
                                     const float* __restrict__ dcgm, int64_t n, int64_t ld,
                                     float* __restrict__ fused) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        unsigned long long tot[3] = {0, 0, 0};
        for (int r = 0; r < DSO_COUNT_ROWS; ++r) {
            const int cat = r < DSO_INSTR_SLOTS ? 0 : (r < DSO_INSTR_SLOTS + DSO_DTYPE_SLOTS ? 1 : 2);
            tot[cat] += counts[(int64_t)r * ld + k];
        }
        for (int j = 0; j < 8; ++j) fused[(int64_t)j * ld + k] = dcgm[(int64_t)j * ld + k];
        for (int r = 0; r < DSO_COUNT_ROWS; ++r) {
            const int cat = r < DSO_INSTR_SLOTS ? 0 : (r < DSO_INSTR_SLOTS + DSO_DTYPE_SLOTS ? 1 : 2);
            const uint64_t c = counts[(int64_t)r * ld + k];
            const double v = tot[cat] ? __ddiv_rn((double)c, (double)tot[cat]) : 0.0;
            fused[(int64_t)(8 + r) * ld + k] = (float)v;
        }
    }
}

// CSR entries ((count << 7) | slot, duplicates add) -> dense uint32 [126][ld]
__global__ void csr_to_dense_kernel(const uint64_t* __restrict__ row_ptr,
                                    const uint32_t* __restrict__ entries, uint64_t ent_base,
                                    int64_t n, int64_t ld, uint32_t* __restrict__ counts) {
    for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < n;
         k += (int64_t)gridDim.x * blockDim.x) {
        for (int r = 0; r < DSO_COUNT_ROWS; ++r) counts[(int64_t)r * ld + k] = 0u;
        for (uint64_t e = row_ptr[k]; e < row_ptr[k + 1]; ++e) {
            const uint32_t v = entries[e - ent_base];
            const int slot = (int)(v & 127u);
            if (slot < DSO_COUNT_ROWS) counts[(int64_t)slot * ld + k] += v >> 7;
        }
    }
}

int grid_of(int64_t n, int block, int sms, int per_sm) {
    const int64_t g = (n + block - 1) / block;
    return (int)std::max<int64_t>(1, std::min<int64_t>(g, (int64_t)sms * per_sm));
}

}  // namespace

GenNet gen_net_of(const ModelDev& md) {
    GenNet g{};
    g.layers = md.n_layers - 1;
    int64_t wo = 0, bo = 0, ao = 0;
    g.maxw = 0;
    for (int l = 0; l <= g.layers; ++l) {
        g.sizes[l] = md.sizes[l];
        g.maxw = std::max(g.maxw, md.sizes[l]);
        g.aoff[l] = (int)ao;
        ao += md.sizes[l];
        if (l < g.layers) {
            g.woff[l] = (int)wo;
            g.boff[l] = (int)bo;
            wo += (int64_t)md.sizes[l] * md.sizes[l + 1];
            bo += md.sizes[l + 1];
        }
    }
    g.sum_widths = (int)ao;
    g.nw = wo;
    g.nb = bo;
    return g;
}

cudaError_t launch_gen_forward(Ctx& cx, const float* x, int64_t n, int64_t ld, float* raw,
                               float* params, uint8_t* clamped, int64_t ld_out) {
    if (n <= 0) return cudaSuccess;
    const GenNet g = gen_net_of(cx.model);
    const int smem = 2 * g.maxw * GT * (int)sizeof(float);
    cudaError_t e = ensure_smem_attr((const void*)gen_forward_kernel, cx.device, 2 * kGenMaxWidth * GT * 4);
    if (e != cudaSuccess) return e;
    gen_forward_kernel<<<grid_of(n, GT, cx.num_sms, 8), GT, smem, cx.stream>>>(
        cx.model.w_master, g, cx.model.gstats, x, n, ld, raw, params, clamped, ld_out);
    ++cx.launches;
    return cudaGetLastError();
}

cudaError_t launch_gen_grad(Ctx& cx, const float* x, const float* y, int64_t n, int64_t ld,
                            float* grad, double* loss_sum_dev) {
    const GenNet g = gen_net_of(cx.model);
    const int64_t np = g.nw + g.nb;
    const int parts = grid_of(std::max<int64_t>(n, 1), GT, cx.num_sms, 2);
    const size_t need = (size_t)parts * np * sizeof(float) + (size_t)parts * sizeof(double) + 256;
    if (cx.train_scratch_bytes < need) {
        cudaFree(cx.train_scratch);
        cx.train_scratch = nullptr;
        cx.train_scratch_bytes = 0;
        cudaError_t e = cudaMalloc(&cx.train_scratch, need);
        if (e != cudaSuccess) return e;
        cx.train_scratch_bytes = need;
    }
    float* partial = (float*)cx.train_scratch;
    double* lp = (double*)(((uintptr_t)(partial + (size_t)parts * np) + 15) & ~(uintptr_t)15);
    const int smem = g.sum_widths * GT * (int)sizeof(float);
    cudaError_t e = ensure_smem_attr((const void*)gen_grad_kernel, cx.device, kGenMaxSumWidths * GT * 4);
    if (e != cudaSuccess) return e;
    gen_grad_kernel<<<parts, GT, smem, cx.stream>>>(cx.model.w_master, g, x, y, n, ld, partial, lp);
    gen_reduce<<<(unsigned)((np + 255) / 256), 256, 0, cx.stream>>>(partial, parts, np, lp, grad,
                                                                 loss_sum_dev);
    cx.launches += 2;
    return cudaGetLastError();
}

cudaError_t launch_gen_apply(Ctx& cx, const float* grad, float lr_scale) {
    const int64_t np = cx.model.n_weights + cx.model.n_biases;
    gen_apply<<<(unsigned)((np + 255) / 256), 256, 0, cx.stream>>>(cx.model.w_master, grad, np,
                                                                lr_scale);
    ++cx.launches;
    return cudaGetLastError();
}

cudaError_t launch_featurize_u64(Ctx& cx, const uint64_t* counts, const float* dcgm, int64_t n,
                                 int64_t ld, float* fused) {
    if (n <= 0) return cudaSuccess;
    featurize_u64_kernel<<<grid_of(n, 128, cx.num_sms, 8), 128, 0, cx.stream>>>(counts, dcgm, n,
                                                                               ld, fused);
    ++cx.launches;
    return cudaGetLastError();
}

cudaError_t launch_csr_to_dense(Ctx& cx, const uint64_t* row_ptr, const uint32_t* entries,
                                uint64_t ent_base, int64_t n, int64_t ld, uint32_t* counts) {
    if (n <= 0) return cudaSuccess;
    csr_to_dense_kernel<<<grid_of(n, 128, cx.num_sms, 8), 128, 0, cx.stream>>>(
        row_ptr, entries, ent_base, n, ld, counts);
    ++cx.launches;
    return cudaGetLastError();
}

// The pipeline of a non-default chain (134 inputs, 7 outputs): staged through
// device scratch — [CSR ->] dense counts -> featurize -> generic forward + clamp ->
// the FP32 sweep — with the fused pipeline's outputs and semantics.
cudaError_t launch_gen_pipeline(Ctx& cx, const uint32_t* counts, const uint64_t* row_ptr,
                                const uint32_t* entries, uint64_t ent_base, const float* dcgm,
                                int64_t n, int64_t ld, float eta, float K, float* params,
                                uint8_t* clamped, int32_t* idx, float* cost, float* energy,
                                float* time, int64_t ld_out) {
    if (n <= 0) return cudaSuccess;
    const size_t cnt_b = row_ptr ? (size_t)DSO_COUNT_ROWS * n * 4 : 0;
    const size_t need = cnt_b + (size_t)DSO_FUSED_ROWS * n * 4 + (size_t)DSO_PARAM_ROWS * n * 4 +
                        (size_t)n * 4 + (size_t)n + 1024;
    if (cx.gen_scratch_bytes < need) {
        cudaFree(cx.gen_scratch);
        cx.gen_scratch = nullptr;
        cx.gen_scratch_bytes = 0;
        cudaError_t e = cudaMalloc(&cx.gen_scratch, need);
        if (e != cudaSuccess) return e;
        cx.gen_scratch_bytes = need;
    }
    char* p = (char*)cx.gen_scratch;
    auto take = [&](size_t b) {
        char* r = p;
        p += (b + 255) & ~(size_t)255;
        return r;
    };
    uint32_t* dc = row_ptr ? (uint32_t*)take(cnt_b) : nullptr;
    float* fused = (float*)take((size_t)DSO_FUSED_ROWS * n * 4);
    float* pr = (float*)take((size_t)DSO_PARAM_ROWS * n * 4);
    int32_t* ks = (int32_t*)take((size_t)n * 4);
    int64_t cld = ld;
    if (row_ptr) {
        cudaError_t e = launch_csr_to_dense(cx, row_ptr, entries, ent_base, n, n, dc);
        if (e != cudaSuccess) return e;
        counts = dc;
        cld = n;
    }
    // featurize reads counts and DCGM with one leading dimension: stage DCGM alongside
    const float* dg = dcgm;
    if (cld != ld) {
        float* d2 = (float*)take((size_t)8 * n * 4);
        cudaError_t e = cudaMemcpy2DAsync(d2, (size_t)n * 4, dcgm, (size_t)ld * 4, (size_t)n * 4, 8,
                                          cudaMemcpyDeviceToDevice, cx.stream);
        if (e != cudaSuccess) return e;
        dg = d2;
    }
    cudaError_t e = launch_featurize(cx, counts, dg, n, cld, fused);
    if (e != cudaSuccess) return e;
    e = launch_gen_forward(cx, fused, n, cld, nullptr, pr, clamped, n);
    if (e != cudaSuccess) return e;
    e = launch_sweep_f32(cx, pr, n, n, eta, K, idx, cost, energy, time, ks);
    if (e != cudaSuccess) return e;
    if (params)
        e = cudaMemcpy2DAsync(params, (size_t)ld_out * 4, pr, (size_t)n * 4, (size_t)n * 4,
                              DSO_PARAM_ROWS, cudaMemcpyDeviceToDevice, cx.stream);
    return e;
}

}  // namespace dso_b200
