// Tensor-core prefix attention (bf16): placeholder until the kernels land.
#include "cuda/common.cuh"
#include "cuda/ops.h"

namespace spk {

bool attn_tc_supported(DType t, int hd) { return false; }

void attn_fwd_tc(const void*, const void*, void*, float*, int64_t, int64_t, int64_t, int, int, cudaStream_t) {
  throw std::logic_error("attn_fwd_tc not available");
}
void attn_bwd_tc(const void*, const void*, const void*, const void*, const float*, float*, float*, void*, float*,
                 int64_t, int64_t, int64_t, int, int, cudaStream_t) {
  throw std::logic_error("attn_bwd_tc not available");
}

}  // namespace spk
