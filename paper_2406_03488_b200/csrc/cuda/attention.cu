// Attention dispatch: fp32 validation mode -> SIMT kernels; bf16 production
// mode -> tensor-core kernels (attention_tc.cu), head dim 64 / 80 / 128. A bf16
// call the tensor-core kernels cannot take is an error (no silent SIMT fallback);
// SIMT in bf16 only on an explicit request (kAttnSimt: SP_FLAG_NO_TC_ATTN, tests).
#include "cuda/common.cuh"
#include "cuda/ops.h"

namespace spk {

void attn_fwd_simt(DType t, const void* q, const void* kv, void* o, float* lse, int64_t n, int64_t q_off,
                   int64_t kv_len, int H, int hd, cudaStream_t s);
void attn_bwd_simt(DType t, const void* q, const void* kv, const void* o, const void* dout, const float* lse,
                   float* ws_delta, float* ws_dq, void* dq, float* dkv, int64_t n, int64_t q_off, int64_t kv_len, int H,
                   int hd, cudaStream_t s);
bool attn_tc_supported(DType t, int hd);
void attn_fwd_tc(const void* q, const void* kv, void* o, float* lse, int64_t n, int64_t q_off, int64_t kv_len, int H,
                 int hd, cudaStream_t s);
void attn_bwd_tc(bool dkv_overwrite, const void* q, const void* kv, const void* o, const void* dout, const float* lse, float* ws_delta,
                 float* ws_dq, void* dq, float* dkv, int64_t n, int64_t q_off, int64_t kv_len, int H, int hd,
                 cudaStream_t s);

void attn_fwd(DType t, int impl, const void* q, const void* kv, void* o, float* lse, int64_t n, int64_t q_off,
              int64_t kv_len, int H, int hd, cudaStream_t s) {
  if (n == 0) return;
  if (kv_len != q_off + n) throw std::invalid_argument("attention: kv_len must equal q_off + n (causal prefix)");
  const bool tc = impl != kAttnSimt && t == DType::kBF16;
  if (impl == kAttnTensor && t != DType::kBF16) throw std::invalid_argument("attention: tensor-core path needs bf16");
  if (tc && !attn_tc_supported(t, hd))
    throw std::invalid_argument("attention: bf16 tensor-core kernels support head_dim 64, 80, 128 (no SIMT fallback)");
  if (tc)
    attn_fwd_tc(q, kv, o, lse, n, q_off, kv_len, H, hd, s);
  else
    attn_fwd_simt(t, q, kv, o, lse, n, q_off, kv_len, H, hd, s);
}

void attn_bwd(DType t, int impl, const void* q, const void* kv, const void* o, const void* dout, const float* lse,
              float* ws_delta, float* ws_dq, void* dq, float* dkv, int64_t n, int64_t q_off, int64_t kv_len, int H, int hd,
              cudaStream_t s, bool dkv_overwrite) {
  if (n == 0) return;
  if (kv_len != q_off + n) throw std::invalid_argument("attention: kv_len must equal q_off + n (causal prefix)");
  const bool tc = impl != kAttnSimt && t == DType::kBF16;
  if (impl == kAttnTensor && t != DType::kBF16) throw std::invalid_argument("attention: tensor-core path needs bf16");
  if (tc && !attn_tc_supported(t, hd))
    throw std::invalid_argument("attention: bf16 tensor-core kernels support head_dim 64, 80, 128 (no SIMT fallback)");
  if (tc) {
    attn_bwd_tc(dkv_overwrite, q, kv, o, dout, lse, ws_delta, ws_dq, dq, dkv, n, q_off, kv_len, H, hd, s);
  } else {
    if (dkv_overwrite)
      SPK_CUDA(cudaMemsetAsync(dkv, 0, sizeof(float) * static_cast<size_t>(kv_len) * 2 * H * hd, s));
    attn_bwd_simt(t, q, kv, o, dout, lse, ws_delta, ws_dq, dq, dkv, n, q_off, kv_len, H, hd, s);
  }
}

}  // namespace spk
