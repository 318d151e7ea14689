// tcgen05 GEMM for sm_100a: bf16 operands, fp32 accumulation in TMEM.
//
//   warp 0      TMA producer (one elected lane): A/B tiles -> 4-stage SMEM ring
//   warp 1      MMA issuer (one lane): 4 x tcgen05.mma (128x256x16) per 64-wide
//               K block, tcgen05.commit frees the SMEM stage; allocates TMEM
//   warps 2..5  epilogue: tcgen05.ld 32x32b -> registers -> fused epilogue
//               (cast / += fp32 / + residual, split output) -> global
//
// Persistent over 128x256 output tiles with a double-buffered TMEM accumulator
// (2 x 256 columns) so tile i's epilogue overlaps tile i+1's MMAs. Operands are
// loaded with 128-byte swizzle; K-major and MN-major operands use the two
// canonical UMMA layouts, so forward (X W^T), dgrad (dY W) and wgrad (dY^T X)
// all run on this one kernel without transposes.
#include <cudaTypedefs.h>

#include <mutex>

#include "cuda/common.cuh"
#include "cuda/ops.h"
#include "cuda/tc_common.cuh"

namespace spk {
namespace {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2, STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NUM_THREADS = 192;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t TMEM_COLS = 512;

struct __align__(64) TcParams {
  CUtensorMap tma_a;
  CUtensorMap tma_b;
  GemmArgs g;
  int a_mn, b_mn;
  int num_m_blk, num_n_blk, num_k_blk;
};

template <typename TC>
__device__ __forceinline__ void store_chunk(const GemmArgs& g, int64_t row, int64_t col0, const uint32_t (&r)[32]) {
  TC* C;
  int64_t ld, c0;
  if (g.split_n >= 0 && col0 >= g.split_n) {
    C = static_cast<TC*>(g.C2);
    ld = g.ldc2;
    c0 = col0 - g.split_n;
  } else {
    C = static_cast<TC*>(g.C);
    ld = g.ldc;
    c0 = col0;
  }
  float v[32];
#pragma unroll
  for (int j = 0; j < 32; ++j) v[j] = __uint_as_float(r[j]);
  const bool full = col0 + 32 <= g.N;
  TC* dst = C + row * ld + c0;
  if (g.epi == Epi::kAddResid) {
    const TC* R = static_cast<const TC*>(g.R) + row * g.ldr + col0;
    if (full) {
      if constexpr (sizeof(TC) == 2) {
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          uint4 u = reinterpret_cast<const uint4*>(R)[q];
          const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            float2 f = __bfloat1622float2(b[e]);
            v[q * 8 + 2 * e] += f.x;
            v[q * 8 + 2 * e + 1] += f.y;
          }
        }
      } else {
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          float4 f = reinterpret_cast<const float4*>(R)[q];
          v[4 * q] += f.x;
          v[4 * q + 1] += f.y;
          v[4 * q + 2] += f.z;
          v[4 * q + 3] += f.w;
        }
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < g.N; ++j) v[j] += to_f(R[j]);
    }
  }
  if (g.epi == Epi::kAccumF32) {
    if (full) {
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        float4 f = reinterpret_cast<const float4*>(dst)[q];
        v[4 * q] += f.x;
        v[4 * q + 1] += f.y;
        v[4 * q + 2] += f.z;
        v[4 * q + 3] += f.w;
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < g.N; ++j) v[j] += to_f(dst[j]);
    }
  }
  if (full) {
    if constexpr (sizeof(TC) == 2) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint4 u;
        __nv_bfloat162* b = reinterpret_cast<__nv_bfloat162*>(&u);
#pragma unroll
        for (int e = 0; e < 4; ++e) b[e] = __floats2bfloat162_rn(v[q * 8 + 2 * e], v[q * 8 + 2 * e + 1]);
        reinterpret_cast<uint4*>(dst)[q] = u;
      }
    } else {
#pragma unroll
      for (int q = 0; q < 8; ++q)
        reinterpret_cast<float4*>(dst)[q] = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
    }
  } else {
    for (int j = 0; j < 32 && col0 + j < g.N; ++j) dst[j] = from_f<TC>(v[j]);
  }
}

template <typename TC>
__global__ void __launch_bounds__(NUM_THREADS, 1) gemm_tc_k(const __grid_constant__ TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      tc::mbar_init(&full[s], 1);
      tc::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 128);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, TMEM_COLS);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  const int num_tiles = p.num_m_blk * p.num_n_blk;
  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&p.tma_a);
      tc::tma_prefetch(&p.tma_b);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        const int mb = tile % p.num_m_blk, nb = tile / p.num_m_blk;
        for (int kb = 0; kb < p.num_k_blk; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          tc::mbar_expect_tx(&full[stage], STAGE_BYTES);
          uint8_t* a_dst = sA + stage * A_BYTES;
          uint8_t* b_dst = sB + stage * B_BYTES;
          if (!p.a_mn) {
            tc::tma_load_2d(a_dst, &p.tma_a, &full[stage], kb * BK, mb * BM);
          } else {
#pragma unroll
            for (int j = 0; j < BM / 64; ++j) tc::tma_load_2d(a_dst + j * 8192, &p.tma_a, &full[stage], mb * BM + 64 * j, kb * BK);
          }
          if (!p.b_mn) {
            tc::tma_load_2d(b_dst, &p.tma_b, &full[stage], kb * BK, nb * BN);
          } else {
#pragma unroll
            for (int j = 0; j < BN / 64; ++j) tc::tma_load_2d(b_dst + j * 8192, &p.tma_b, &full[stage], nb * BN + 64 * j, kb * BK);
          }
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = tc::idesc_bf16(BM, BN, p.a_mn, p.b_mn);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
        tc::mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem_base + acc * BN;
        for (int kb = 0; kb < p.num_k_blk; ++kb) {
          tc::mbar_wait(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t a_base = tc::smem_u32(sA + stage * A_BYTES);
          const uint32_t b_base = tc::smem_u32(sB + stage * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK / 16; ++kk) {
            // K-major: +32 B per 16-element K step inside the 128 B swizzled row.
            // MN-major: +2 K-groups of 8 rows (2 x 1024 B); MN atoms of 64 are 8 KB apart.
            const uint64_t ad = p.a_mn ? tc::smem_desc(a_base + kk * 2048, 8192, 1024, tc::kSwizzle128B)
                                       : tc::smem_desc(a_base + kk * 32, 16, 1024, tc::kSwizzle128B);
            const uint64_t bd = p.b_mn ? tc::smem_desc(b_base + kk * 2048, 8192, 1024, tc::kSwizzle128B)
                                       : tc::smem_desc(b_base + kk * 32, 16, 1024, tc::kSwizzle128B);
            tc::mma_bf16_ss(d, ad, bd, idesc, (kb | kk) != 0);
          }
          tc::mma_commit(&empty[stage]);
          if (++stage == STAGES) {
            stage = 0;
            phase ^= 1;
          }
        }
        tc::mma_commit(&tfull[acc]);
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    const int quarter = warp % 4;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = blockIdx.x; tile < num_tiles; tile += gridDim.x) {
      const int mb = tile % p.num_m_blk, nb = tile / p.num_m_blk;
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::tc_fence_after();
      const int64_t row = (int64_t)mb * BM + quarter * 32 + lane;
#pragma unroll 1
      for (int c0 = 0; c0 < BN; c0 += 32) {
        const int64_t col0 = (int64_t)nb * BN + c0;
        uint32_t r[32];
        tc::tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * BN + c0, r);
        tc::tmem_ld_wait();
        if (row < p.g.M && col0 < p.g.N) store_chunk<TC>(p.g, row, col0, r);
      }
      tc::tc_fence_before();
      tc::mbar_arrive(&tempty[acc]);
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc(tmem_base, TMEM_COLS);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
  });
  if (!fn) throw CudaError("cuTensorMapEncodeTiled unavailable");
  return fn;
}

void make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_inner,
              uint32_t box_outer) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string(static_cast<int>(r)));
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

}  // namespace

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn() { return encode_fn(); }

bool gemm_tc_supported(const GemmArgs& a) {
  if (a.ab != DType::kBF16) return false;
  if (a.M <= 0 || a.N <= 0 || a.K <= 0) return false;
  if (a.lda % 8 || a.ldb % 8 || !aligned16(a.A) || !aligned16(a.B)) return false;
  const int cvec = a.c == DType::kF32 ? 4 : 8;
  if (a.ldc % cvec || !aligned16(a.C)) return false;
  if (a.epi == Epi::kAddResid && (a.ldr % cvec || !aligned16(a.R))) return false;
  if (a.split_n >= 0 && (a.split_n % 32 || a.ldc2 % cvec || !aligned16(a.C2))) return false;
  return true;
}

void gemm_tcgen05(const GemmArgs& a, cudaStream_t s) {
  if (!gemm_tc_supported(a)) throw std::invalid_argument("gemm_tcgen05: unsupported operand layout/alignment");
  TcParams p;
  p.g = a;
  p.a_mn = !a.a_kmajor;
  p.b_mn = !a.b_kmajor;
  if (a.a_kmajor)
    make_map(&p.tma_a, a.A, a.K, a.M, a.lda, 64, BM);
  else
    make_map(&p.tma_a, a.A, a.M, a.K, a.lda, 64, 64);
  if (a.b_kmajor)
    make_map(&p.tma_b, a.B, a.K, a.N, a.ldb, 64, BN);
  else
    make_map(&p.tma_b, a.B, a.N, a.K, a.ldb, 64, 64);
  p.num_m_blk = static_cast<int>((a.M + BM - 1) / BM);
  p.num_n_blk = static_cast<int>((a.N + BN - 1) / BN);
  p.num_k_blk = static_cast<int>((a.K + BK - 1) / BK);
  const int tiles = p.num_m_blk * p.num_n_blk;
  const int grid = tiles < num_sms() ? tiles : num_sms();
  if (a.c == DType::kF32) {
    SPK_CUDA(cudaFuncSetAttribute(gemm_tc_k<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    gemm_tc_k<float><<<grid, NUM_THREADS, SMEM_BYTES, s>>>(p);
  } else {
    SPK_CUDA(cudaFuncSetAttribute(gemm_tc_k<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
    gemm_tc_k<__nv_bfloat16><<<grid, NUM_THREADS, SMEM_BYTES, s>>>(p);
  }
  SPK_LAUNCH_CHECK();
}

void gemm(const GemmArgs& a, cudaStream_t s, int impl) {
  if (a.M == 0 || a.N == 0) return;
  if (impl == kGemmSimt || a.ab == DType::kF32) return gemm_simt(a, s);
  if (impl == kGemmTcgen05 || gemm_tc_supported(a)) return gemm_tcgen05(a, s);
  gemm_simt(a, s);
}

}  // namespace spk
