// SIMT GEMM: the fp32 validation-mode path (true fp32 products, fp32
// accumulation) and the cross-check for the tcgen05 kernel. Handles every
// operand majorness, split outputs and the three epilogues. 64x64 tiles,
// 256 threads, 4x4 register micro-tile per thread.
#include "cuda/common.cuh"
#include "cuda/ops.h"

namespace spk {
namespace {

constexpr int BM = 64, BN = 64, BK = 16;

template <typename TA, typename TC>
__global__ void __launch_bounds__(256) gemm_simt_k(GemmArgs a) {
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  const TA* A = static_cast<const TA*>(a.A);
  const TA* B = static_cast<const TA*>(a.B);
  const int64_t m0 = (int64_t)blockIdx.y * BM, n0 = (int64_t)blockIdx.x * BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  float acc[4][4] = {};
  for (int64_t k0 = 0; k0 < a.K; k0 += BK) {
    for (int i = threadIdx.x; i < BM * BK; i += 256) {
      // Index so that consecutive threads walk the contiguous dimension.
      int mm, kk;
      if (a.a_kmajor) {
        mm = i / BK;
        kk = i % BK;
      } else {
        kk = i / BM;
        mm = i % BM;
      }
      const int64_t gm = m0 + mm, gk = k0 + kk;
      float v = 0.f;
      if (gm < a.M && gk < a.K) v = to_f(a.a_kmajor ? A[gm * a.lda + gk] : A[gk * a.lda + gm]);
      As[kk][mm] = v;
    }
    for (int i = threadIdx.x; i < BN * BK; i += 256) {
      int nn, kk;
      if (a.b_kmajor) {
        nn = i / BK;
        kk = i % BK;
      } else {
        kk = i / BN;
        nn = i % BN;
      }
      const int64_t gn = n0 + nn, gk = k0 + kk;
      float v = 0.f;
      if (gn < a.N && gk < a.K) v = to_f(a.b_kmajor ? B[gn * a.ldb + gk] : B[gk * a.ldb + gn]);
      Bs[kk][nn] = v;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < BK; ++kk) {
      float av[4], bv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) av[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bv[j] = Bs[kk][tx * 4 + j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(av[i], bv[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + ty * 4 + i;
    if (gm >= a.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + tx * 4 + j;
      if (gn >= a.N) continue;
      TC* C;
      int64_t idx;
      if (a.split_n >= 0 && gn >= a.split_n) {
        C = static_cast<TC*>(a.C2);
        idx = gm * a.ldc2 + (gn - a.split_n);
      } else {
        C = static_cast<TC*>(a.C);
        idx = gm * a.ldc + gn;
      }
      float v = acc[i][j];
      if (a.epi == Epi::kAccumF32) {
        v += to_f(C[idx]);
      } else if (a.epi == Epi::kAddResid) {
        v += to_f(static_cast<const TC*>(a.R)[gm * a.ldr + gn]);
      } else if (a.epi == Epi::kGeluGrad) {
        v *= gelu_tanh_grad(to_f(static_cast<const TC*>(a.R)[gm * a.ldr + gn]));
      }
      C[idx] = from_f<TC>(v);
    }
  }
}

}  // namespace

void gemm_simt(const GemmArgs& a, cudaStream_t s) {
  if (a.M == 0 || a.N == 0) return;
  dim3 grid((unsigned)((a.N + BN - 1) / BN), (unsigned)((a.M + BM - 1) / BM));
  if (a.ab == DType::kF32) {
    if (a.c == DType::kF32)
      gemm_simt_k<float, float><<<grid, 256, 0, s>>>(a);
    else
      gemm_simt_k<float, __nv_bfloat16><<<grid, 256, 0, s>>>(a);
  } else {
    if (a.c == DType::kF32)
      gemm_simt_k<__nv_bfloat16, float><<<grid, 256, 0, s>>>(a);
    else
      gemm_simt_k<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, s>>>(a);
  }
  SPK_LAUNCH_CHECK();
}

const void* module_anchor_gemm_simt() { return reinterpret_cast<const void*>(&gemm_simt_k<float, float>); }

}  // namespace spk
