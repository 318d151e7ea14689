// Host-side launchers of the sm_100a kernels used by the engine (C++ only; the
// C-ABI in include/seqpipe_b200.h exposes the GEMM / attention entry points).
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

#include "cuda/common.cuh"

namespace spk {

// ---------------------------------------------------------------- GEMM
// C[m, n] (op)= sum_k A[m, k] * B[n, k]
//   A[m,k] = a_kmajor ? A[m*lda + k] : A[k*lda + m]
//   B[n,k] = b_kmajor ? B[n*ldb + k] : B[k*ldb + n]
enum class Epi : int {
  kStore = 0,     // C = acc                     (cast to c dtype)
  kAccumF32 = 1,  // C += acc                    (fp32 C: weight-gradient accumulation)
  kAddResid = 2,  // C = acc + R                 (residual stream; R may alias C)
  kGeluGrad = 3,  // C = acc * gelu'(R)          (MLP dgrad fused with the GeLU backward; R = u)
};

struct GemmArgs {
  int64_t M = 0, N = 0, K = 0;
  DType ab = DType::kBF16;
  const void* A = nullptr;
  int64_t lda = 0;
  bool a_kmajor = true;
  const void* B = nullptr;
  int64_t ldb = 0;
  bool b_kmajor = true;
  void* C = nullptr;
  int64_t ldc = 0;
  DType c = DType::kBF16;
  Epi epi = Epi::kStore;
  const void* R = nullptr;
  int64_t ldr = 0;
  // Column split: output columns >= split_n are written to C2 at column (n - split_n).
  void* C2 = nullptr;
  int64_t ldc2 = 0;
  int64_t split_n = -1;
};

enum GemmImpl : int { kGemmAuto = 0, kGemmSimt = 1, kGemmTcgen05 = 2 };

void gemm(const GemmArgs& a, cudaStream_t s, int impl = kGemmAuto);
bool gemm_tc_supported(const GemmArgs& a);
void gemm_simt(const GemmArgs& a, cudaStream_t s);
void gemm_tcgen05(const GemmArgs& a, cudaStream_t s);
// Per host thread: true restricts the tcgen05 GEMM to its 1-CTA kernel (no cta_group::2
// clusters). Set by engines that share one GPU with other engines' threads (in-process
// multi-rank): with several engines launching 2-CTA GEMMs concurrently, a pair's
// cta_group::2 TMEM allocation intermittently never completed (engine.cpp, step()).
void set_gemm_single_cta(bool on);

// ---------------------------------------------------------------- attention
// q [n, H*hd] (row stride H*hd), kv [kv_len, 2*H*hd] (K | V per row),
// o [n, H*hd], lse [H, n] fp32. Query i has global position q_off + i and may
// attend to keys j <= q_off + i (j < kv_len).
enum AttnImpl : int { kAttnAuto = 0, kAttnSimt = 1, kAttnTensor = 2 };
void attn_fwd(DType t, int impl, const void* q, const void* kv, void* o, float* lse, int64_t n, int64_t q_off,
              int64_t kv_len, int H, int hd, cudaStream_t s);
// dq [n, H*hd] (dtype t); dkv_acc [kv_len, 2*H*hd] fp32, accumulated (+=), or written
// (=) when dkv_overwrite (every row [0, kv_len) is covered by the call: the first
// backward op of a micro-batch, which saves the accumulator's memset and read).
// ws_delta: >= attn_bwd_ws_delta_floats(n, H) floats; ws_dq: >= n*H*hd floats.
size_t attn_bwd_ws_delta_floats(int64_t n, int H);
void attn_bwd(DType t, int impl, const void* q, const void* kv, const void* o, const void* dout, const float* lse,
              float* ws_delta, float* ws_dq, void* dq, float* dkv_acc, int64_t n, int64_t q_off, int64_t kv_len, int H,
              int hd, cudaStream_t s, bool dkv_overwrite = false);

// ---------------------------------------------------------------- elementwise / norms
void embed_fwd(DType t, const int32_t* tok, const float* E, const float* pos_table, int64_t pos0, void* x, int64_t n,
               int h, cudaStream_t s);
void embed_bwd(DType t, const int32_t* tok, const void* dx, float* dE, float* dpos, int64_t pos0, int64_t n, int h,
               cudaStream_t s);
// LayerNorm (rms=false, gain only) / RMSNorm (rms=true). mean may be null for rms.
void norm_fwd(DType t, bool rms, const void* x, const float* g, void* y, float* mean, float* rstd, int64_t n, int h,
              float eps, cudaStream_t s);
void norm_apply(DType t, bool rms, const void* x, const float* g, const float* mean, const float* rstd, void* y,
                int64_t n, int h, cudaStream_t s);
// dx = dres + d(norm)/dx . dy ; dg += sum_rows dy * xhat. dres may be null; dx may alias dres.
void norm_bwd(DType t, bool rms, const void* dy, const void* x, const float* g, const float* mean, const float* rstd,
              const void* dres, void* dx, float* dg, int64_t n, int h, cudaStream_t s);
// family 0 (GPT): g = gelu_tanh(u), u [n, F]; family 1 (LLaMA): g = silu(u[:, :F]) * u[:, F:], u [n, 2F].
void act_fwd(DType t, int family, const void* u, void* g, int64_t n, int F, cudaStream_t s);
void act_bwd(DType t, int family, const void* u, const void* dg, void* du, int64_t n, int F, cudaStream_t s);
// Rotary embedding in place on [n, H*hd] rows (row stride ld) at global positions pos0 + i.
void rope(DType t, void* x, int64_t ld, int64_t n, int H, int hd, int64_t pos0, float theta, bool inverse,
          cudaStream_t s);
// dqkv [n, 3h] = [ dq | cast(dkv_rows) ] with dkv_rows [n, 2h] fp32.
void assemble_dqkv(DType t, const void* dq, const float* dkv_rows, void* dqkv, int64_t n, int h, cudaStream_t s);
// In place: logits [n, V] (row stride ld) -> dlogits = (softmax - onehot(label)) * scale;
// loss_acc (fp64) += sum_rows CE.
void ce_fwd_bwd(DType t, void* logits, int64_t ld, const int32_t* labels, int64_t n, int V, float scale,
                double* loss_acc, cudaStream_t s);
void cast_from_f32(DType t, const float* src, void* dst, int64_t n, cudaStream_t s);
void fill_normal(float* p, int64_t n, uint64_t seed, float stddev, cudaStream_t s);
void fill_const(float* p, int64_t n, float v, cudaStream_t s);
// bc: device {1 - b1^t, 1 - b2^t} (so a captured step graph replays with the current t).
void adamw(float* p, const float* g, float* m, float* v, void* pc, DType t, int64_t n, float lr, float b1, float b2,
           float eps, float wd, const float* bc, cudaStream_t s);

// ---------------------------------------------------------------- module loading
// Loads every kernel of this library into the current device's context now. Under lazy
// module loading (CUDA_MODULE_LOADING=LAZY, the CUDA 12 default) a kernel is loaded at its
// first launch and the load waits for the context to go idle; a rank whose streams are
// parked on a peer's transfer (stream wait / NCCL receive) then blocks its host thread in
// the launch, and two ranks doing so wait on each other forever. Multi-rank engines call
// this before their first step. One kernel of each translation unit (module_anchor_*)
// names its module; the rest are enumerated from it.
void preload_kernels();
const void* module_anchor_attention_simt();
const void* module_anchor_attention_tc();
const void* module_anchor_elementwise();
const void* module_anchor_gemm_simt();
const void* module_anchor_gemm_tcgen05();

}  // namespace spk
