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

#include <cstdlib>
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

// Tile raster of the persistent kernels: groups of kGroupM m-blocks, n-blocks walked inside a
// group. The CTAs of one wave (consecutive tiles) then share ~8 A and ~10 B panels instead of
// every A panel of the matrix (m fastest): at the cfg-2 shapes the wave's operand set fits in
// L2 and each panel comes from DRAM about once per wave (ncu: 1.27 GB of DRAM reads for a
// 10170 x 2560 x 10240 GEMM whose operands are 0.26 GB).
#ifndef SPK_GEMM_GROUP_M
#define SPK_GEMM_GROUP_M 8  // tools/build_variant.py -DSPK_GEMM_GROUP_M=1000 reproduces the m-fastest raster
#endif
constexpr int kGroupM = SPK_GEMM_GROUP_M;
__device__ __forceinline__ void tile_coords(int tile, int num_m, int num_n, int& mb, int& nb) {
  const int per_group = kGroupM * num_n;
  const int g = tile / per_group, r = tile - g * per_group;
  const int m0 = g * kGroupM;
  const int gm = num_m - m0 < kGroupM ? num_m - m0 : kGroupM;
  mb = m0 + r % gm;
  nb = r / gm;
}

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
  if (g.epi == Epi::kGeluGrad) {  // bf16 C only (gemm_tc_supported)
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
            v[q * 8 + 2 * e] *= gelu_grad_fast(f.x);
            v[q * 8 + 2 * e + 1] *= gelu_grad_fast(f.y);
          }
        }
      }
    } else {
      for (int j = 0; j < 32 && col0 + j < g.N; ++j) v[j] *= gelu_grad_fast(to_f(R[j]));
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
        int mb, nb;
        tile_coords(tile, p.num_m_blk, p.num_n_blk, mb, nb);
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
      int mb, nb;
        tile_coords(tile, p.num_m_blk, p.num_n_blk, mb, nb);
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

// ----------------------------------------------------------------------------
// 2-CTA (cta_group::2) variant: a CTA pair computes a 256x256 output tile with
// tcgen05.mma.cta_group::2 (M = 256 split 128 per CTA, N = 256 with each CTA
// holding half of the B tile). Per CTA and 64-wide K block the TMA brings
// 16 KB of A + 16 KB of B (vs 48 KB for the 1-CTA 128x256 tile): the L2 ->
// SMEM traffic per FLOP drops by a third, which is what bounds the 1-CTA
// kernel (~16 TB/s of L2 reads at 1.4 PFLOP/s). The leader CTA (rank 0) issues
// the MMAs; both CTAs load their halves with .cta_group::2 TMA completing on
// the leader's barrier, and both drain their own TMEM rows in the epilogue.
constexpr int BM2 = 128, BNH = 128, BK2 = 64, ST2 = 6;
constexpr int A2_BYTES = BM2 * BK2 * 2, B2_BYTES = BNH * BK2 * 2, STAGE2_BYTES = A2_BYTES + B2_BYTES;
constexpr int SMEM2_BYTES = ST2 * STAGE2_BYTES + 1024 + 256;

__device__ __forceinline__ uint32_t mapa_rank0(uint32_t saddr) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, 0;" : "=r"(r) : "r"(saddr));
  return r;
}
__device__ __forceinline__ void tma_load_2d_2cta(uint32_t dst, const CUtensorMap* m, uint32_t bar_cluster, int32_t c0,
                                                 int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(dst),
      "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

template <typename TC>
__global__ void __launch_bounds__(NUM_THREADS, 1) gemm_tc2_k(const __grid_constant__ TcParams p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + ST2 * A2_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + ST2 * B2_BYTES);  // [ST2] used in the leader
  uint64_t* empty = full + ST2;                                         // [ST2] both CTAs
  uint64_t* tfull = empty + ST2;                                        // [2]   both CTAs
  uint64_t* tempty = tfull + 2;                                         // [2]   used in the leader
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = tc::cluster_ctarank();
  const int cid = static_cast<int>(blockIdx.x >> 1), ncl = static_cast<int>(gridDim.x >> 1);
  if (warp == 0 && lane == 0) {
    for (int s = 0; s < ST2; ++s) {
      tc::mbar_init(&full[s], 1);   // leader's arrive.expect_tx (both CTAs' bytes)
      tc::mbar_init(&empty[s], 1);  // leader's multicast MMA commit
    }
    for (int a = 0; a < 2; ++a) {
      tc::mbar_init(&tfull[a], 1);
      tc::mbar_init(&tempty[a], 8);  // 4 epilogue warps x 2 CTAs
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(tc::smem_u32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);

  const int num_tiles = p.num_m_blk * p.num_n_blk;  // 256 x 256 tiles
  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&p.tma_a);
      tc::tma_prefetch(&p.tma_b);
      int stage = 0;
      uint32_t phase = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl) {
        int mb, nb;
        tile_coords(tile, p.num_m_blk, p.num_n_blk, mb, nb);
        const int m0 = mb * 256 + static_cast<int>(rank) * BM2, n0 = nb * 256 + static_cast<int>(rank) * BNH;
        for (int kb = 0; kb < p.num_k_blk; ++kb) {
          tc::mbar_wait(&empty[stage], phase ^ 1);
          const uint32_t bar = mapa_rank0(tc::smem_u32(&full[stage]));
          if (rank == 0) tc::mbar_expect_tx(&full[stage], 2 * STAGE2_BYTES);
          const uint32_t a_dst = tc::smem_u32(sA + stage * A2_BYTES), b_dst = tc::smem_u32(sB + stage * B2_BYTES);
          if (!p.a_mn) {
            tma_load_2d_2cta(a_dst, &p.tma_a, bar, kb * BK2, m0);
          } else {
#pragma unroll
            for (int j = 0; j < BM2 / 64; ++j) tma_load_2d_2cta(a_dst + j * 8192, &p.tma_a, bar, m0 + 64 * j, kb * BK2);
          }
          if (!p.b_mn) {
            tma_load_2d_2cta(b_dst, &p.tma_b, bar, kb * BK2, n0);
          } else {
#pragma unroll
            for (int j = 0; j < BNH / 64; ++j) tma_load_2d_2cta(b_dst + j * 8192, &p.tma_b, bar, n0 + 64 * j, kb * BK2);
          }
          if (++stage == ST2) {
            stage = 0;
            phase ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (rank == 0) {  // leader issues for the pair (whole warp converged; elect inside the asm)
      const uint32_t idesc = tc::idesc_bf16(256, 256, p.a_mn, p.b_mn);
      int stage = 0;
      uint32_t phase = 0;
      int acc = 0;
      uint32_t acc_phase = 0;
      for (int tile = cid; tile < num_tiles; tile += ncl) {
        tc::mbar_wait_w(&tempty[acc], acc_phase ^ 1);
        tc::tc_fence_after();
        const uint32_t d = tmem_base + acc * 256;
        for (int kb = 0; kb < p.num_k_blk; ++kb) {
          tc::mbar_wait_w(&full[stage], phase);
          tc::tc_fence_after();
          const uint32_t a_base = tc::smem_u32(sA + stage * A2_BYTES), b_base = tc::smem_u32(sB + stage * B2_BYTES);
#pragma unroll
          for (int kk = 0; kk < BK2 / 16; ++kk) {
            const uint64_t ad = p.a_mn ? tc::smem_desc(a_base + kk * 2048, 8192, 1024, tc::kSwizzle128B)
                                       : tc::smem_desc(a_base + kk * 32, 16, 1024, tc::kSwizzle128B);
            const uint64_t bd = p.b_mn ? tc::smem_desc(b_base + kk * 2048, 8192, 1024, tc::kSwizzle128B)
                                       : tc::smem_desc(b_base + kk * 32, 16, 1024, tc::kSwizzle128B);
            const uint32_t accum = (kb | kk) != 0;
            asm volatile(
                "{\n\t.reg .pred p, e;\n\t"
                "elect.sync _|e, 0xffffffff;\n\t"
                "setp.ne.b32 p, %4, 0;\n\t"
                "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
                "l"(ad), "l"(bd), "r"(idesc), "r"(accum)
                : "memory");
          }
          asm volatile(  // frees the stage in both CTAs once these MMAs retire
              "{\n\t.reg .pred e;\n\t"
              "elect.sync _|e, 0xffffffff;\n\t"
              "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                  tc::smem_u32(&empty[stage])),
              "h"(static_cast<uint16_t>(3))
              : "memory");
          if (++stage == ST2) {
            stage = 0;
            phase ^= 1;
          }
        }
        asm volatile(
            "{\n\t.reg .pred e;\n\t"
            "elect.sync _|e, 0xffffffff;\n\t"
            "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}" ::"r"(
                tc::smem_u32(&tfull[acc])),
            "h"(static_cast<uint16_t>(3))
            : "memory");
        acc ^= 1;
        if (acc == 0) acc_phase ^= 1;
      }
    }
  } else {
    const int quarter = warp % 4;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int tile = cid; tile < num_tiles; tile += ncl) {
      int mb, nb;
        tile_coords(tile, p.num_m_blk, p.num_n_blk, mb, nb);
      tc::mbar_wait(&tfull[acc], acc_phase);
      tc::tc_fence_after();
      const int64_t row = (int64_t)mb * 256 + rank * BM2 + quarter * 32 + lane;
#pragma unroll 1
      for (int c0 = 0; c0 < 256; c0 += 32) {
        const int64_t col0 = (int64_t)nb * 256 + c0;
        uint32_t r[32];
        tc::tmem_ld32(tmem_base + (static_cast<uint32_t>(quarter * 32) << 16) + acc * 256 + c0, r);
        tc::tmem_ld_wait();
        if (row < p.g.M && col0 < p.g.N) store_chunk<TC>(p.g, row, col0, r);
      }
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_remote(mapa_rank0(tc::smem_u32(&tempty[acc])));
      acc ^= 1;
      if (acc == 0) acc_phase ^= 1;
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "r"(TMEM_COLS) : "memory");
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
  if (a.epi == Epi::kGeluGrad && (a.c != DType::kBF16 || a.ldr % 8 || !aligned16(a.R))) return false;
  if (a.split_n >= 0 && (a.split_n % 32 || a.ldc2 % cvec || !aligned16(a.C2))) return false;
  return true;
}

namespace {
thread_local bool t_single_cta = false;
}
void set_gemm_single_cta(bool on) { t_single_cta = on; }

void gemm_tcgen05(const GemmArgs& a, cudaStream_t s) {
  if (!gemm_tc_supported(a)) throw std::invalid_argument("gemm_tcgen05: unsupported operand layout/alignment");
  static const int env_force = [] {
    const char* e = std::getenv("SP_GEMM_CTA");  // tuning: 1 = force the 1-CTA kernel, 2 = force 2-CTA
    return e ? std::atoi(e) : 0;
  }();
  const int force = env_force == 2 ? 2 : (t_single_cta ? 1 : env_force);
  // 2-CTA 256x256 tiles once the problem has enough of them to fill the pairs.
  const int64_t tiles2 = ((a.M + 255) / 256) * ((a.N + 255) / 256);
  const bool two = force == 2 || (force != 1 && tiles2 >= num_sms() / 2);
  TcParams p;
  p.g = a;
  p.a_mn = !a.a_kmajor;
  p.b_mn = !a.b_kmajor;
  if (a.a_kmajor)
    make_map(&p.tma_a, a.A, a.K, a.M, a.lda, 64, BM);
  else
    make_map(&p.tma_a, a.A, a.M, a.K, a.lda, 64, 64);
  const uint32_t bn_box = two ? BNH : BN;
  if (a.b_kmajor)
    make_map(&p.tma_b, a.B, a.K, a.N, a.ldb, 64, bn_box);
  else
    make_map(&p.tma_b, a.B, a.N, a.K, a.ldb, 64, 64);
  if (two) {
    p.num_m_blk = static_cast<int>((a.M + 255) / 256);
    p.num_n_blk = static_cast<int>((a.N + 255) / 256);
    p.num_k_blk = static_cast<int>((a.K + BK2 - 1) / BK2);
    const int pairs = static_cast<int>(tiles2 < num_sms() / 2 ? tiles2 : num_sms() / 2);
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(2 * pairs);
    lc.blockDim = dim3(NUM_THREADS);
    lc.dynamicSmemBytes = SMEM2_BYTES;
    lc.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    if (a.c == DType::kF32) {
      SPK_CUDA(cudaFuncSetAttribute(gemm_tc2_k<float>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES));
      SPK_CUDA(cudaLaunchKernelEx(&lc, gemm_tc2_k<float>, p));
    } else {
      SPK_CUDA(cudaFuncSetAttribute(gemm_tc2_k<__nv_bfloat16>, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM2_BYTES));
      SPK_CUDA(cudaLaunchKernelEx(&lc, gemm_tc2_k<__nv_bfloat16>, p));
    }
    return;
  }
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
  // fp32 validation mode (or an explicit SIMT request) -> SIMT; bf16 -> tcgen05 only. A bf16
  // shape the tensor-core path cannot take is an error, never a silent SIMT fallback.
  if (impl == kGemmSimt || a.ab == DType::kF32) return gemm_simt(a, s);
  if (!gemm_tc_supported(a))
    throw std::invalid_argument("gemm: bf16 operands need 16-byte aligned pointers and row strides (multiples of 8 "
                                "elements) for the tcgen05/TMA path; no SIMT fallback in bf16 mode");
  gemm_tcgen05(a, s);
}

const void* module_anchor_gemm_tcgen05() { return reinterpret_cast<const void*>(&gemm_tc_k<float>); }

}  // namespace spk
