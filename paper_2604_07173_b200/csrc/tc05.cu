// tc05.cu -- tcgen05/TMEM kernels for large segments (placeholder until the
// tensor-core path lands; tc_available() keeps the dispatcher on CUDA cores).
#include "common.cuh"
#include "kernels.h"

namespace lora {
bool tc_available() { return false; }
cudaError_t launch_tc_shrink(const MultiArgs&, const PlanDev&, int, cudaStream_t) { return cudaSuccess; }
cudaError_t launch_tc_expand(const MultiArgs&, const PlanDev&, int, cudaStream_t) { return cudaSuccess; }
}  // namespace lora
