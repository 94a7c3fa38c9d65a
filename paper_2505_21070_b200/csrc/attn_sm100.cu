// tcgen05 attention (placeholder until implemented).
#include "device.cuh"
#include "kernels_bf16.cuh"
namespace bp {
void launch_attn_tc(const AttnBf16Args&, int64_t, cudaStream_t) { fail(BP_ERR_INTERNAL, "tcgen05 attention not built"); }
}  // namespace bp
