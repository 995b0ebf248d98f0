// dp.cu — predictor training behind the C-ABI: one data-parallel SGD step
// (gradient -> NCCL allreduce -> update) and the reference's fit_model epoch
// loop (mlp.cpp:84-130) on the device, with NCCL reached through dlopen.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2", preferring a copy that is
// already mapped into the process — e.g. the one torch.distributed uses), so
// libdso_b200.so has no link-time NCCL dependency and never mixes two NCCL
// builds in one process.  Communicators are plain ncclComm_t handles: the host
// may create them here (dso_nccl_comm_init from a dso_nccl_unique_id broadcast
// over any channel) or pass one made by its own NCCL.
#include <dlfcn.h>
#include <math.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <functional>
#include <limits>
#include <mutex>
#include <string>
#include <vector>

#include "common.cuh"

using namespace dso_b200;

namespace {

struct NcclApi {
    bool ok = false;
    std::string why;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t,
                              ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.why = std::string("libnccl.so.2 not found: ") + (e ? e : "");
            return;
        }
        auto sym = [&](const char* name) { return dlsym(h, name); };
        api.GetUniqueId = (decltype(api.GetUniqueId))sym("ncclGetUniqueId");
        api.CommInitRank = (decltype(api.CommInitRank))sym("ncclCommInitRank");
        api.CommDestroy = (decltype(api.CommDestroy))sym("ncclCommDestroy");
        api.AllReduce = (decltype(api.AllReduce))sym("ncclAllReduce");
        api.GroupStart = (decltype(api.GroupStart))sym("ncclGroupStart");
        api.GroupEnd = (decltype(api.GroupEnd))sym("ncclGroupEnd");
        api.GetVersion = (decltype(api.GetVersion))sym("ncclGetVersion");
        api.GetErrorString = (decltype(api.GetErrorString))sym("ncclGetErrorString");
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllReduce &&
                 api.GroupStart && api.GroupEnd;
        if (!api.ok) api.why = "libnccl.so.2 lacks the collective entry points";
    });
    return api;
}

int32_t fail(dso_ctx* ctx, int32_t st, const std::string& msg) {
    if (ctx) ctx->c.last_error = msg;
    return st;
}

#define DSO_CUDA(ctx, expr)                                                          \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess)                                                       \
            return fail(ctx, kCuda, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    } while (0)

#define DSO_NCCL(ctx, expr)                                                                   \
    do {                                                                                      \
        ncclResult_t _r = (expr);                                                             \
        if (_r != ncclSuccess)                                                                \
            return fail(ctx, kCuda, std::string(#expr) + ": " +                               \
                                        (nccl().GetErrorString ? nccl().GetErrorString(_r)    \
                                                               : "nccl error"));              \
    } while (0)

// splitmix64 (rng.hpp:11-46): fork and the Lemire shuffle, as in abi.cu
uint64_t rng_next(uint64_t& s) {
    uint64_t z = (s += 0x9e3779b97f4a7c15ULL);
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}
uint64_t rng_fork(uint64_t seed, uint64_t salt) {  // Rng(seed).fork(salt), rng.hpp:50-54
    uint64_t s = seed ^ (0xd1342543de82ef95ULL * (salt + 1));
    rng_next(s);
    return s;
}
uint64_t rng_below(uint64_t& s, uint64_t n) {
    uint64_t x = rng_next(s);
    __uint128_t m = (__uint128_t)x * n;
    uint64_t l = (uint64_t)m;
    if (l < n) {
        const uint64_t t = (0ULL - n) % n;
        while (l < t) {
            x = rng_next(s);
            m = (__uint128_t)x * n;
            l = (uint64_t)m;
        }
    }
    return (uint64_t)(m >> 64);
}
void shuffle_into(uint64_t n, uint64_t& s, int64_t* out) {  // shuffled_indices, rng.hpp:58-64
    for (uint64_t i = 0; i < n; ++i) out[i] = (int64_t)i;
    for (uint64_t i = n; i > 1; --i) std::swap(out[i - 1], out[rng_below(s, i)]);
}

// dst[r][k] = src[r][idx[k]] for rows r < rows, k < n (dataset columns in epoch order)
__global__ void gather_columns(const float* __restrict__ src, int64_t ld_src, int rows,
                               const int64_t* __restrict__ idx, int64_t n,
                               float* __restrict__ dst, int64_t ld_dst) {
    const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int64_t j = idx[k];
    for (int r = blockIdx.y; r < rows; r += gridDim.y) dst[r * ld_dst + k] = src[r * ld_src + j];
}

// epoch loss bookkeeping (sgd_epoch, mlp.cpp:101-103): acc += loss_sum / (b * out)
__global__ void acc_loss(double* __restrict__ acc, const double* __restrict__ loss_sum, double inv) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *acc += *loss_sum * inv;
}
__global__ void zero_d(double* p) {
    if (threadIdx.x == 0 && blockIdx.x == 0) *p = 0.0;
}

struct TrainBufs {
    float* grad;
    double* dbl;  // [0] loss_sum, [1] epoch accumulator
};

// The context's training buffers (Ctx::dp_grad / dp_dbl, freed by dso_ctx_destroy).
cudaError_t bufs_for(dso_ctx* ctx, TrainBufs& out) {
    Ctx& c = ctx->c;
    const int64_t np = c.model.n_weights + c.model.n_biases;
    if (c.dp_np < np) {
        cudaFree(c.dp_grad);
        c.dp_grad = nullptr;
        c.dp_np = 0;
        cudaError_t r = cudaMalloc(&c.dp_grad, sizeof(float) * np);
        if (r != cudaSuccess) return r;
        c.dp_np = np;
    }
    if (!c.dp_dbl) {
        cudaError_t r = cudaMalloc(&c.dp_dbl, sizeof(double) * 4);
        if (r != cudaSuccess) return r;
    }
    out = TrainBufs{c.dp_grad, c.dp_dbl};
    return cudaSuccess;
}

int32_t check(dso_ctx* ctx) {
    if (!ctx) return kInvalidArgument;
    if (!ctx->c.has_model) return fail(ctx, kInvalidModel, "no model set (dso_set_model)");
    cudaError_t e = cudaSetDevice(ctx->c.device);
    if (e != cudaSuccess) return fail(ctx, kCuda, cudaGetErrorString(e));
    return kOk;
}

// grad -> [allreduce] -> apply on the context stream; loss_sum stays on the device
int32_t step_on_stream(dso_ctx* ctx, TrainBufs* tb, const float* x, const float* y, int64_t n,
                       int64_t ld, double lr, int64_t global_batch, ncclComm_t comm,
                       bool repack) {
    Ctx& c = ctx->c;
    const int64_t np = c.model.n_weights + c.model.n_biases;
    const int out = c.model.sizes[c.model.n_layers - 1];
    DSO_CUDA(ctx, launch_train_grad(c, x, y, n, ld, tb->grad, tb->dbl));
    if (comm) {
        const NcclApi& api = nccl();
        if (!api.ok) return fail(ctx, kIoError, api.why);
        DSO_NCCL(ctx, api.GroupStart());
        DSO_NCCL(ctx, api.AllReduce(tb->grad, tb->grad, (size_t)np, ncclFloat32, ncclSum, comm, c.stream));
        DSO_NCCL(ctx, api.AllReduce(tb->dbl, tb->dbl, 1, ncclFloat64, ncclSum, comm, c.stream));
        DSO_NCCL(ctx, api.GroupEnd());
    }
    const double scale = 1.0 / ((double)global_batch * out);
    DSO_CUDA(ctx, launch_train_apply(c, tb->grad, (float)(lr * scale), repack));
    return kOk;
}

}  // namespace

extern "C" {

int32_t dso_nccl_version(int32_t* version) {
    const NcclApi& api = nccl();
    if (!api.ok || !version) return kIoError;
    int v = 0;
    if (api.GetVersion) api.GetVersion(&v);
    *version = v;
    return kOk;
}

int32_t dso_nccl_unique_id(uint8_t* id) {
    const NcclApi& api = nccl();
    if (!id) return kInvalidArgument;
    if (!api.ok) return kIoError;
    ncclUniqueId u;
    if (api.GetUniqueId(&u) != ncclSuccess) return kCuda;
    static_assert(sizeof(ncclUniqueId) == DSO_NCCL_ID_BYTES, "ncclUniqueId size");
    memcpy(id, &u, sizeof(u));
    return kOk;
}

int32_t dso_nccl_comm_init(int32_t nranks, const uint8_t* id, int32_t rank, int32_t device,
                           void** comm) {
    const NcclApi& api = nccl();
    if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) return kInvalidArgument;
    if (!api.ok) return kIoError;
    if (cudaSetDevice(device) != cudaSuccess) return kCuda;
    ncclUniqueId u;
    memcpy(&u, id, sizeof(u));
    ncclComm_t c = nullptr;
    if (api.CommInitRank(&c, nranks, u, rank) != ncclSuccess) return kCuda;
    *comm = c;
    return kOk;
}

int32_t dso_nccl_comm_destroy(void* comm) {
    const NcclApi& api = nccl();
    if (!comm) return kOk;
    if (!api.ok) return kIoError;
    return api.CommDestroy((ncclComm_t)comm) == ncclSuccess ? kOk : kCuda;
}

int32_t dso_train_step(dso_ctx* ctx, const float* x, const float* y_std, int64_t n, int64_t ld,
                       double lr, int64_t global_batch, void* comm, double* loss) {
    int32_t st = check(ctx);
    if (st) return st;
    if (n < 0 || ld < n) return fail(ctx, kInvalidArgument, "batch requires 0 <= n <= ld");
    if (global_batch < 1) return fail(ctx, kInvalidArgument, "global_batch must be positive");
    if (!(lr >= 0.0)) return fail(ctx, kInvalidArgument, "learning rate must be >= 0");
    TrainBufs tbv{};
    TrainBufs* tb = &tbv;
    DSO_CUDA(ctx, bufs_for(ctx, tbv));
    st = step_on_stream(ctx, tb, x, y_std, n, ld, lr, global_batch, (ncclComm_t)comm, true);
    if (st) return st;
    if (loss) {
        double h = 0.0;
        Ctx& c = ctx->c;
        DSO_CUDA(ctx, cudaMemcpyAsync(&h, tb->dbl, sizeof(double), cudaMemcpyDeviceToHost, c.stream));
        DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
        *loss = h / ((double)global_batch * c.model.sizes[c.model.n_layers - 1]);
    }
    return kOk;
}

int32_t dso_fit_model(dso_ctx* ctx, const float* x, const float* y_std, int64_t n, int64_t ld,
                      double lr, int32_t batch, int32_t epochs, uint64_t seed, void* comm,
                      int32_t rank, int32_t nranks, double* epoch_loss, int32_t* epochs_run) {
    int32_t st = check(ctx);
    if (st) return st;
    if (n < 1 || ld < n) return fail(ctx, kInvalidArgument, "fit_model needs 1 <= n <= ld");
    if (batch < 1 || epochs < 0) return fail(ctx, kInvalidArgument, "batch >= 1, epochs >= 0");
    if (nranks < 1 || rank < 0 || rank >= nranks || (nranks > 1 && !comm))
        return fail(ctx, kInvalidArgument, "rank / nranks / communicator inconsistent");
    if (epochs_run) *epochs_run = 0;
    Ctx& c = ctx->c;
    const int in = c.model.sizes[0], out = c.model.sizes[c.model.n_layers - 1];
    TrainBufs tbv{};
    TrainBufs* tb = &tbv;
    DSO_CUDA(ctx, bufs_for(ctx, tbv));
    // epoch-ordered copies of the dataset + the order (device), pinned order (host)
    float *xe = nullptr, *ye = nullptr;
    int64_t* idx_d = nullptr;
    int64_t* idx_h = nullptr;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    cudaStream_t caller = c.stream;
    cudaEvent_t ev = nullptr;
    auto cleanup = [&]() {
        if (exec) cudaGraphExecDestroy(exec);
        if (graph) cudaGraphDestroy(graph);
        if (ev) cudaEventDestroy(ev);
        cudaFree(xe);
        cudaFree(ye);
        cudaFree(idx_d);
        cudaFreeHost(idx_h);
        c.stream = caller;
    };
    struct Guard {
        std::function<void()> f;
        ~Guard() { f(); }
    } guard{cleanup};
    DSO_CUDA(ctx, cudaMalloc(&xe, sizeof(float) * (size_t)in * n));
    DSO_CUDA(ctx, cudaMalloc(&ye, sizeof(float) * (size_t)out * n));
    DSO_CUDA(ctx, cudaMalloc(&idx_d, sizeof(int64_t) * n));
    DSO_CUDA(ctx, cudaMallocHost(&idx_h, sizeof(int64_t) * n));
    DSO_CUDA(ctx, train_prepare(c, batch < n ? batch : n));
    // run on the context's own (capturable) stream, ordered after the caller's work
    DSO_CUDA(ctx, cudaEventCreateWithFlags(&ev, cudaEventDisableTiming));
    DSO_CUDA(ctx, cudaEventRecord(ev, caller));
    c.stream = c.own_stream;
    DSO_CUDA(ctx, cudaStreamWaitEvent(c.stream, ev, 0));

    const int64_t n_batches = (n + batch - 1) / batch;
    auto epoch_body = [&]() -> int32_t {
        DSO_CUDA(ctx, cudaMemcpyAsync(idx_d, idx_h, sizeof(int64_t) * n, cudaMemcpyHostToDevice,
                                      c.stream));
        const dim3 g((unsigned)((n + 255) / 256), 8);
        gather_columns<<<g, 256, 0, c.stream>>>(x, ld, in, idx_d, n, xe, n);
        gather_columns<<<g, 256, 0, c.stream>>>(y_std, ld, out, idx_d, n, ye, n);
        zero_d<<<1, 32, 0, c.stream>>>(tb->dbl + 1);
        c.launches += 3;
        for (int64_t s = 0; s < n; s += batch) {
            const int64_t b = std::min<int64_t>(batch, n - s);
            // this rank's share of the global batch (contiguous)
            const int64_t a0 = s + b * rank / nranks, a1 = s + b * (rank + 1) / nranks;
            int32_t r = step_on_stream(ctx, tb, xe + a0, ye + a0, a1 - a0, n, lr, b,
                                       (ncclComm_t)comm, false);
            if (r) return r;
            acc_loss<<<1, 32, 0, c.stream>>>(tb->dbl + 1, tb->dbl, 1.0 / ((double)b * out));
            ++c.launches;
        }
        return kOk;
    };
    // The epoch's launch sequence depends only on (n, batch): captured once into a
    // CUDA graph and replayed with the next shuffled order in the pinned buffer.
    // With a communicator the steps are launched directly (NCCL calls are not
    // captured here).
    const bool use_graph = epochs > 2 && !comm;
    uint64_t rs = rng_fork(seed, 0x5d0);
    for (int e = 0; e < epochs; ++e) {
        DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));  // idx_h is read by the last epoch
        shuffle_into((uint64_t)n, rs, idx_h);
        if (use_graph && !exec) {
            c.model.train_dirty = true;  // the captured first step repacks the weights
            DSO_CUDA(ctx, cudaStreamBeginCapture(c.stream, cudaStreamCaptureModeThreadLocal));
            const int32_t r = epoch_body();
            cudaGraph_t gph = nullptr;
            const cudaError_t ce = cudaStreamEndCapture(c.stream, &gph);
            if (r) {
                if (gph) cudaGraphDestroy(gph);
                return r;
            }
            DSO_CUDA(ctx, ce);
            graph = gph;
            DSO_CUDA(ctx, cudaGraphInstantiate(&exec, graph, 0));
        }
        if (exec) {
            DSO_CUDA(ctx, cudaGraphLaunch(exec, c.stream));
        } else {
            const int32_t r = epoch_body();
            if (r) return r;
        }
        double acc = 0.0;
        DSO_CUDA(ctx, cudaMemcpyAsync(&acc, tb->dbl + 1, sizeof(double), cudaMemcpyDeviceToHost,
                                      c.stream));
        DSO_CUDA(ctx, cudaStreamSynchronize(c.stream));
        double v = acc / (double)n_batches;
        if (!std::isfinite(v)) v = std::numeric_limits<double>::quiet_NaN();
        if (epoch_loss) epoch_loss[e] = v;
        if (epochs_run) *epochs_run = e + 1;
        if (std::isnan(v)) break;  // diverged (mlp.cpp:126)
    }
    // inference kernels see the trained weights
    DSO_CUDA(ctx, launch_repack(c));
    DSO_CUDA(ctx, cudaEventRecord(ev, c.stream));
    DSO_CUDA(ctx, cudaStreamWaitEvent(caller, ev, 0));
    return kOk;
}

}  // extern "C"
