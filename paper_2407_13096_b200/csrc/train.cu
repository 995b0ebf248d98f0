// train.cu — predictor training kernels (placeholder until the batched
// forward/backward kernels land; dso_train_* report InvalidArgument).
#include "common.cuh"

namespace dso_b200 {

cudaError_t launch_train_grad(Ctx&, const float*, const float*, int64_t, int64_t, float*,
                              double*) {
    return cudaErrorNotSupported;
}

cudaError_t launch_train_apply(Ctx&, const float*, float) { return cudaErrorNotSupported; }

}  // namespace dso_b200
