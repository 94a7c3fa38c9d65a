// tcgen05 GEMM (placeholder until implemented).
#include "device.cuh"
#include "kernels_bf16.cuh"
namespace bp {
void launch_gemm_tc(const bf16*, int64_t, const bf16*, int, int, int, void*, int64_t, int, cudaStream_t) {
  fail(BP_ERR_INTERNAL, "tcgen05 GEMM not built");
}
}  // namespace bp
