// SIMT causal prefix attention (fp32 math): the fp32 validation-mode path and
// the cross-check for the tensor-core kernels.
//
// Forward: one CTA per (32-query block, head), online softmax over 32-key
// blocks of the KV prefix [0, q_off + n).
// Backward: one CTA per (32-key block, head), looping over every query block
// that can see those keys; dK/dV accumulate in shared memory and are added
// once into the fp32 dKV accumulator (each (key row, head) slice has exactly
// one owner CTA: deterministic, no atomics). dQ partials are atomically added
// into an fp32 workspace and cast at the end.
#include "cuda/common.cuh"
#include "cuda/ops.h"

namespace spk {
namespace {

constexpr int BQ = 32, BKV = 32, NT = 128, HD_MAX = 128;

template <typename T>
__global__ void __launch_bounds__(NT) attn_fwd_simt_k(const T* __restrict__ q, const T* __restrict__ kv, T* __restrict__ o,
                                                      float* __restrict__ lse, int64_t n, int64_t q_off, int64_t kv_len,
                                                      int H, int hd, float scale) {
  extern __shared__ float sm[];
  float* Qs = sm;                         // [BQ][hd]
  float* Ks = Qs + BQ * hd;               // [BKV][hd+1]
  float* Vs = Ks + BKV * (hd + 1);        // [BKV][hd]
  float* S = Vs + BKV * hd;               // [BQ][BKV+1]
  float* Os = S + BQ * (BKV + 1);         // [BQ][hd]
  float* mrow = Os + BQ * hd;             // [BQ]
  float* lrow = mrow + BQ;                // [BQ]
  float* alpha = lrow + BQ;               // [BQ]
  const int head = blockIdx.y;
  const int64_t i0 = (int64_t)blockIdx.x * BQ;
  const int64_t h = (int64_t)H * hd;
  for (int e = threadIdx.x; e < BQ * hd; e += NT) {
    const int r = e / hd, d = e % hd;
    Qs[e] = (i0 + r < n) ? to_f(q[(i0 + r) * h + head * hd + d]) : 0.f;
    Os[e] = 0.f;
  }
  if (threadIdx.x < BQ) {
    mrow[threadIdx.x] = -INFINITY;
    lrow[threadIdx.x] = 0.f;
  }
  const int64_t last_q = q_off + (i0 + BQ < n ? i0 + BQ : n) - 1;  // highest query position in the block
  const int64_t kend = (last_q + 1 < kv_len) ? last_q + 1 : kv_len;
  __syncthreads();
  for (int64_t j0 = 0; j0 < kend; j0 += BKV) {
    for (int e = threadIdx.x; e < BKV * hd; e += NT) {
      const int r = e / hd, d = e % hd;
      const bool ok = j0 + r < kv_len;
      Ks[r * (hd + 1) + d] = ok ? to_f(kv[(j0 + r) * 2 * h + head * hd + d]) : 0.f;
      Vs[r * hd + d] = ok ? to_f(kv[(j0 + r) * 2 * h + h + head * hd + d]) : 0.f;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < BQ * BKV; e += NT) {
      const int r = e / BKV, c = e % BKV;
      const int64_t qpos = q_off + i0 + r, kpos = j0 + c;
      float v = -INFINITY;
      if (i0 + r < n && kpos < kv_len && kpos <= qpos) {
        float acc = 0.f;
        for (int d = 0; d < hd; ++d) acc = fmaf(Qs[r * hd + d], Ks[c * (hd + 1) + d], acc);
        v = acc * scale;
      }
      S[r * (BKV + 1) + c] = v;
    }
    __syncthreads();
    if (threadIdx.x < BQ) {
      const int r = threadIdx.x;
      float mx = mrow[r];
      for (int c = 0; c < BKV; ++c) mx = fmaxf(mx, S[r * (BKV + 1) + c]);
      float sum = 0.f;
      for (int c = 0; c < BKV; ++c) {
        const float sv = S[r * (BKV + 1) + c];
        const float p = (sv == -INFINITY) ? 0.f : expf(sv - mx);
        S[r * (BKV + 1) + c] = p;
        sum += p;
      }
      const float a = (mrow[r] == -INFINITY) ? 0.f : expf(mrow[r] - mx);
      alpha[r] = a;
      lrow[r] = lrow[r] * a + sum;
      mrow[r] = mx;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < BQ * hd; e += NT) {
      const int r = e / hd, d = e % hd;
      float acc = Os[e] * alpha[r];
      for (int c = 0; c < BKV; ++c) acc = fmaf(S[r * (BKV + 1) + c], Vs[c * hd + d], acc);
      Os[e] = acc;
    }
    __syncthreads();
  }
  for (int e = threadIdx.x; e < BQ * hd; e += NT) {
    const int r = e / hd, d = e % hd;
    if (i0 + r < n) o[(i0 + r) * h + head * hd + d] = from_f<T>(Os[e] / lrow[r]);
  }
  if (threadIdx.x < BQ && i0 + threadIdx.x < n)
    lse[(int64_t)head * n + i0 + threadIdx.x] = mrow[threadIdx.x] + logf(lrow[threadIdx.x]);
}

// delta[head, i] = sum_d dO[i, head, d] * O[i, head, d]
template <typename T>
__global__ void attn_delta_k(const T* __restrict__ o, const T* __restrict__ dout, float* __restrict__ delta, int64_t n,
                             int H, int hd) {
  const int64_t row = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;  // one warp per (i, head)
  if (row >= n * H) return;
  const int64_t i = row / H;
  const int head = static_cast<int>(row % H);
  const int64_t base = i * (int64_t)H * hd + head * hd;
  float s = 0.f;
  for (int d = threadIdx.x % 32; d < hd; d += 32) s += to_f(o[base + d]) * to_f(dout[base + d]);
  s = warp_sum(s);
  if (threadIdx.x % 32 == 0) delta[(int64_t)head * n + i] = s;
}

template <typename T>
__global__ void __launch_bounds__(NT) attn_bwd_simt_k(const T* __restrict__ q, const T* __restrict__ kv,
                                                      const T* __restrict__ dout, const float* __restrict__ lse,
                                                      const float* __restrict__ delta, float* __restrict__ dq_ws,
                                                      float* __restrict__ dkv, int64_t n, int64_t q_off, int64_t kv_len,
                                                      int H, int hd, float scale) {
  extern __shared__ float sm[];
  float* Ks = sm;                   // [BKV][hd+1]
  float* Vs = Ks + BKV * (hd + 1);  // [BKV][hd+1]
  float* dKs = Vs + BKV * (hd + 1); // [BKV][hd]
  float* dVs = dKs + BKV * hd;      // [BKV][hd]
  float* Qs = dVs + BKV * hd;       // [BQ][hd+1]
  float* dOs = Qs + BQ * (hd + 1);  // [BQ][hd+1]
  float* P = dOs + BQ * (hd + 1);   // [BQ][BKV+1]
  float* dS = P + BQ * (BKV + 1);   // [BQ][BKV+1]
  float* Ls = dS + BQ * (BKV + 1);  // [BQ]
  float* Ds = Ls + BQ;              // [BQ]
  const int head = blockIdx.y;
  const int64_t j0 = (int64_t)blockIdx.x * BKV;
  const int64_t h = (int64_t)H * hd;
  for (int e = threadIdx.x; e < BKV * hd; e += NT) {
    const int r = e / hd, d = e % hd;
    const bool ok = j0 + r < kv_len;
    Ks[r * (hd + 1) + d] = ok ? to_f(kv[(j0 + r) * 2 * h + head * hd + d]) : 0.f;
    Vs[r * (hd + 1) + d] = ok ? to_f(kv[(j0 + r) * 2 * h + h + head * hd + d]) : 0.f;
    dKs[e] = 0.f;
    dVs[e] = 0.f;
  }
  // First query (local index) that can see key j0: q_off + i >= j0.
  int64_t ib = j0 - q_off;
  if (ib < 0) ib = 0;
  ib = (ib / BQ) * BQ;
  for (int64_t i0 = ib; i0 < n; i0 += BQ) {
    __syncthreads();
    for (int e = threadIdx.x; e < BQ * hd; e += NT) {
      const int r = e / hd, d = e % hd;
      const bool ok = i0 + r < n;
      Qs[r * (hd + 1) + d] = ok ? to_f(q[(i0 + r) * h + head * hd + d]) : 0.f;
      dOs[r * (hd + 1) + d] = ok ? to_f(dout[(i0 + r) * h + head * hd + d]) : 0.f;
    }
    if (threadIdx.x < BQ) {
      const bool ok = i0 + threadIdx.x < n;
      Ls[threadIdx.x] = ok ? lse[(int64_t)head * n + i0 + threadIdx.x] : 0.f;
      Ds[threadIdx.x] = ok ? delta[(int64_t)head * n + i0 + threadIdx.x] : 0.f;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < BQ * BKV; e += NT) {
      const int r = e / BKV, c = e % BKV;
      const int64_t qpos = q_off + i0 + r, kpos = j0 + c;
      float p = 0.f, ds = 0.f;
      if (i0 + r < n && kpos < kv_len && kpos <= qpos) {
        float s = 0.f, dp = 0.f;
        for (int d = 0; d < hd; ++d) {
          s = fmaf(Qs[r * (hd + 1) + d], Ks[c * (hd + 1) + d], s);
          dp = fmaf(dOs[r * (hd + 1) + d], Vs[c * (hd + 1) + d], dp);
        }
        p = expf(s * scale - Ls[r]);
        ds = p * (dp - Ds[r]) * scale;
      }
      P[r * (BKV + 1) + c] = p;
      dS[r * (BKV + 1) + c] = ds;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < BKV * hd; e += NT) {
      const int c = e / hd, d = e % hd;
      float dv = dVs[e], dk = dKs[e];
      for (int r = 0; r < BQ; ++r) {
        dv = fmaf(P[r * (BKV + 1) + c], dOs[r * (hd + 1) + d], dv);
        dk = fmaf(dS[r * (BKV + 1) + c], Qs[r * (hd + 1) + d], dk);
      }
      dVs[e] = dv;
      dKs[e] = dk;
    }
    for (int e = threadIdx.x; e < BQ * hd; e += NT) {
      const int r = e / hd, d = e % hd;
      if (i0 + r >= n) continue;
      float acc = 0.f;
      for (int c = 0; c < BKV; ++c) acc = fmaf(dS[r * (BKV + 1) + c], Ks[c * (hd + 1) + d], acc);
      atomicAdd(&dq_ws[(i0 + r) * h + head * hd + d], acc);
    }
  }
  __syncthreads();
  for (int e = threadIdx.x; e < BKV * hd; e += NT) {
    const int r = e / hd, d = e % hd;
    if (j0 + r >= kv_len) continue;
    dkv[(j0 + r) * 2 * h + head * hd + d] += dKs[e];
    dkv[(j0 + r) * 2 * h + h + head * hd + d] += dVs[e];
  }
}

template <typename T>
__global__ void cast_ws_k(const float* __restrict__ src, T* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = from_f<T>(src[i]);
}

size_t fwd_smem(int hd) { return sizeof(float) * (BQ * hd + BKV * (hd + 1) + BKV * hd + BQ * (BKV + 1) + BQ * hd + 3 * BQ); }
size_t bwd_smem(int hd) {
  return sizeof(float) * (2 * BKV * (hd + 1) + 2 * BKV * hd + 2 * BQ * (hd + 1) + 2 * BQ * (BKV + 1) + 2 * BQ);
}

}  // namespace

void attn_fwd_simt(DType t, const void* q, const void* kv, void* o, float* lse, int64_t n, int64_t q_off,
                   int64_t kv_len, int H, int hd, cudaStream_t s) {
  if (n == 0) return;
  if (hd > HD_MAX) throw std::invalid_argument("attention head_dim > 128 unsupported");
  const float scale = 1.f / sqrtf(static_cast<float>(hd));
  dim3 grid((unsigned)((n + BQ - 1) / BQ), (unsigned)H);
  const size_t smem = fwd_smem(hd);
  if (t == DType::kF32) {
    cudaFuncSetAttribute(attn_fwd_simt_k<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_fwd_simt_k<float><<<grid, NT, smem, s>>>((const float*)q, (const float*)kv, (float*)o, lse, n, q_off, kv_len, H,
                                                  hd, scale);
  } else {
    cudaFuncSetAttribute(attn_fwd_simt_k<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_fwd_simt_k<__nv_bfloat16><<<grid, NT, smem, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)kv,
                                                          (__nv_bfloat16*)o, lse, n, q_off, kv_len, H, hd, scale);
  }
  SPK_LAUNCH_CHECK();
}

void attn_delta(DType t, const void* o, const void* dout, float* delta, int64_t n, int H, int hd, cudaStream_t s) {
  const int64_t rows = n * H;
  const int blocks = static_cast<int>((rows + 7) / 8);
  if (t == DType::kF32)
    attn_delta_k<float><<<blocks, 256, 0, s>>>((const float*)o, (const float*)dout, delta, n, H, hd);
  else
    attn_delta_k<__nv_bfloat16><<<blocks, 256, 0, s>>>((const __nv_bfloat16*)o, (const __nv_bfloat16*)dout, delta, n, H, hd);
  SPK_LAUNCH_CHECK();
}

void attn_bwd_simt(DType t, const void* q, const void* kv, const void* o, const void* dout, const float* lse,
                   float* ws_delta, float* ws_dq, void* dq, float* dkv, int64_t n, int64_t q_off, int64_t kv_len, int H,
                   int hd, cudaStream_t s) {
  if (n == 0) return;
  if (hd > HD_MAX) throw std::invalid_argument("attention head_dim > 128 unsupported");
  const float scale = 1.f / sqrtf(static_cast<float>(hd));
  attn_delta(t, o, dout, ws_delta, n, H, hd, s);
  SPK_CUDA(cudaMemsetAsync(ws_dq, 0, sizeof(float) * n * H * hd, s));
  dim3 grid((unsigned)((kv_len + BKV - 1) / BKV), (unsigned)H);
  const size_t smem = bwd_smem(hd);
  if (t == DType::kF32) {
    cudaFuncSetAttribute(attn_bwd_simt_k<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_bwd_simt_k<float><<<grid, NT, smem, s>>>((const float*)q, (const float*)kv, (const float*)dout, lse, ws_delta,
                                                  ws_dq, dkv, n, q_off, kv_len, H, hd, scale);
  } else {
    cudaFuncSetAttribute(attn_bwd_simt_k<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    attn_bwd_simt_k<__nv_bfloat16><<<grid, NT, smem, s>>>((const __nv_bfloat16*)q, (const __nv_bfloat16*)kv,
                                                          (const __nv_bfloat16*)dout, lse, ws_delta, ws_dq, dkv, n,
                                                          q_off, kv_len, H, hd, scale);
  }
  SPK_LAUNCH_CHECK();
  const int64_t total = n * H * hd;
  const int blocks = static_cast<int>(total < 148 * 64 * 256 ? (total + 255) / 256 : 148 * 64);
  if (t == DType::kF32)
    cast_ws_k<float><<<blocks, 256, 0, s>>>(ws_dq, (float*)dq, total);
  else
    cast_ws_k<__nv_bfloat16><<<blocks, 256, 0, s>>>(ws_dq, (__nv_bfloat16*)dq, total);
  SPK_LAUNCH_CHECK();
}

const void* module_anchor_attention_simt() { return reinterpret_cast<const void*>(&attn_fwd_simt_k<float>); }

}  // namespace spk
