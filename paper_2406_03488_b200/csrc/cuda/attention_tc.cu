// tcgen05 causal prefix attention for Seq1F1B (bf16 in, fp32 softmax and
// accumulation, sm_100a).
//
// A sub-sequence s of n queries (global positions q_off..q_off+n-1) attends to
// the micro-batch's KV-prefix slab rows [0, q_off + n): the causal edge
// F(m,s-1) -> F(m,s) of the reference dependency model
// (/root/reference/proj/core/src/sim.cpp:24-27). The backward adds dK/dV for
// those rows into the stage's fp32 accumulator (reverse edge, sim.cpp:34-36).
//
// Head-dim tiling. A [rows x hd] bf16 tile is stored as a 64-column chunk in
// the canonical 128-byte-swizzled layout plus, for hd > 64, a second chunk:
// hd 128 -> another 64-column SW128 chunk; hd 80 -> a 16-column chunk in the
// 32-byte-swizzled layout (no padding: 160 B per row instead of 256 B). A tile
// serves both as a K-major operand (rows = M/N) and, unchanged, as an MN-major
// operand (rows = K); MN-major GEMMs with N = hd 80 issue an N=64 and an N=16
// MMA into adjacent TMEM columns.
//
// Forward: one CTA per (128 queries, head). warp 0 = TMA (Q once, K/V rings, K
// running one block ahead of V), warp 1 = MMA issuer polling two queues (S_j =
// Q K_j^T and O += P_j V_j), warps 4-7 = softmax (one query row per thread, S
// row in registers, P to SMEM, O accumulated in TMEM with lazy rescaling).
// Backward: dK/dV kernel (2-CTA clusters of 128-key blocks, Q/dO tiles
// multicast to both CTAs, 8 softmax warps) and dQ kernel (128-query blocks);
// both deterministic, no atomics.
#include <cudaTypedefs.h>

#include <cstdlib>

#include "cuda/common.cuh"
#include "cuda/ops.h"
#include "cuda/tc_common.cuh"

namespace spk {

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn();  // gemm_tcgen05.cu

namespace {

constexpr int BQ = 128, BKV = 128;

#ifndef SPK_ATTN_NARROW80
#define SPK_ATTN_NARROW80 0  // measured slower on B200 (extra N=16 MMAs, 32-byte TMA rows)
#endif

template <int HD>
struct Lay {
  static constexpr bool NARROW = HD == 80 && SPK_ATTN_NARROW80;  // hd 80: SW32 16-column second chunk
  static constexpr int C1 = HD <= 64 ? 0 : (NARROW ? 16 : 64);  // columns held by the second chunk
  static constexpr int R1 = C1 * 2;                              // bytes per row of the second chunk
  static constexpr int bytes(int rows) { return rows * (128 + R1); }
};

// K-major descriptor of head-dim step kk (16 dims) of a [rows x hd] tile.
template <int HD>
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int rows, int kk) {
  if (kk < 4) return tc::smem_desc(base + kk * 32, 16, 1024, tc::kSwizzle128B);
  if constexpr (Lay<HD>::NARROW) {
    return tc::smem_desc(base + rows * 128, 16, 256, tc::kSwizzle32B);
  } else {
    return tc::smem_desc(base + rows * 128 + (kk - 4) * 32, 16, 1024, tc::kSwizzle128B);
  }
}

// D[128 x hd] (+)= A[128 x 16 (K step kk)] * B[K rows of a [rows x hd] tile]^T, B MN-major.
template <int HD>
__device__ __forceinline__ void mma_nhd(uint32_t d, uint64_t adesc, uint32_t bbase, int rows, int kk, bool acc) {
  if constexpr (Lay<HD>::NARROW) {
    constexpr uint32_t i64 = tc::idesc_bf16(128, 64, false, true), i16 = tc::idesc_bf16(128, 16, false, true);
    tc::mma_bf16_ss(d, adesc, tc::smem_desc(bbase + kk * 2048, rows * 128, 1024, tc::kSwizzle128B), i64, acc);
    tc::mma_bf16_ss(d + 64, adesc, tc::smem_desc(bbase + rows * 128 + kk * 512, 256, 256, tc::kSwizzle32B), i16, acc);
  } else {  // padded second chunk: one N = hd MMA
    constexpr uint32_t id = tc::idesc_bf16(128, HD, false, true);
    tc::mma_bf16_ss(d, adesc, tc::smem_desc(bbase + kk * 2048, rows * 128, 1024, tc::kSwizzle128B), id, acc);
  }
}

// Same with A (M=128 x K=16, bf16 packed two per 32-bit column) read from TMEM.
template <int HD>
__device__ __forceinline__ void mma_nhd_ts(uint32_t d, uint32_t a_tmem, uint32_t bbase, int rows, int kk, bool acc) {
  if constexpr (Lay<HD>::NARROW) {
    constexpr uint32_t i64 = tc::idesc_bf16(128, 64, false, true), i16 = tc::idesc_bf16(128, 16, false, true);
    tc::mma_bf16_ts(d, a_tmem, tc::smem_desc(bbase + kk * 2048, rows * 128, 1024, tc::kSwizzle128B), i64, acc);
    tc::mma_bf16_ts(d + 64, a_tmem, tc::smem_desc(bbase + rows * 128 + kk * 512, 256, 256, tc::kSwizzle32B), i16, acc);
  } else {
    constexpr uint32_t id = tc::idesc_bf16(128, HD, false, true);
    tc::mma_bf16_ts(d, a_tmem, tc::smem_desc(bbase + kk * 2048, rows * 128, 1024, tc::kSwizzle128B), id, acc);
  }
}

// TMEM column of K-step kk (16 columns of a 64-wide bf16 operand) when each
// half (32 columns) of the operand was packed at the start of its own 32
// fp32 columns (the softmax half that produced it overwrites only its slice).
__device__ __forceinline__ uint32_t half_packed_col(int kk) { return 32 * (kk >> 1) + 8 * (kk & 1); }

__device__ __forceinline__ float4 lds_f4(const void* p) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))));
  return v;
}

struct Maps {  // chunk-0 and chunk-1 tensor maps of one [rows, cols] bf16 tensor
  CUtensorMap m0, m1;
};

// TMA a [rows x hd] tile at (col, row) of the tensor into dst (both chunks).
template <int HD>
__device__ __forceinline__ void load_tile(uint8_t* dst, const Maps& t, uint64_t* bar, int col, int row, int rows,
                                          uint16_t mc) {
  if (mc) {
    tc::tma_load_2d_mc(dst, &t.m0, bar, col, row, mc);
    if constexpr (HD > 64) tc::tma_load_2d_mc(dst + rows * 128, &t.m1, bar, col + 64, row, mc);
  } else {
    tc::tma_load_2d(dst, &t.m0, bar, col, row);
    if constexpr (HD > 64) tc::tma_load_2d(dst + rows * 128, &t.m1, bar, col + 64, row);
  }
}

struct __align__(64) AttnParams {
  Maps tq;   // q [n, h], 128-row boxes
  Maps tkv;  // kv [kv_len, 2h], 128-row boxes
  __nv_bfloat16* o;
  float* lse;
  int64_t n, q_off, kv_len;
  int H, h;
  float scale_log2;
};


__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// One MUFU.EX2 (exp2f() adds range-reduction FMUL/FSETP/FSEL around it).
__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t pack_bf16(float a, float b) {
  __nv_bfloat162 v = __floats2bfloat162_rn(a, b);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int HD>
constexpr size_t fwd_smem_n(int st) {
  return Lay<HD>::bytes(128) * (1 + 2 * st) + (10 + 4 * st) * 8 + 8 + 1024;
}
// Ring depths: as many stages as the opt-in SMEM (227 KB) holds, capped at 4 / 6 / 8.
template <int HD>
constexpr int fwd_stages() {
  int st = 4;
  while (fwd_smem_n<HD>(st) > 232448) --st;
  return st;
}
template <int HD>
constexpr size_t fwd_smem() {
  return fwd_smem_n<HD>(fwd_stages<HD>());
}

// ============================================================================ forward

template <int HD>
__global__ void __launch_bounds__(256, 1) attn_fwd_tc_k(const __grid_constant__ AttnParams p) {
  constexpr int KVS = fwd_stages<HD>();
  constexpr int TB = Lay<HD>::bytes(128);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sK = sQ + TB;           // [KVS]
  uint8_t* sV = sK + KVS * TB;     // [KVS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + KVS * TB);
  uint64_t* q_full = bars;
  uint64_t* s_full = bars + 1;   // [2]
  uint64_t* p_full = bars + 5;   // [2]
  uint64_t* p_empty = bars + 7;  // [2]
  uint64_t* k_full = bars + 10;          // [KVS]
  uint64_t* k_empty = k_full + KVS;      // [KVS]
  uint64_t* v_full = k_empty + KVS;      // [KVS]
  uint64_t* v_empty = v_full + KVS;      // [KVS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + KVS);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_qb = static_cast<int>((p.n + BQ - 1) / BQ);
  const int qb = num_qb - 1 - static_cast<int>(blockIdx.x);  // heaviest blocks first
  const int head = blockIdx.y;
  const int64_t q0 = static_cast<int64_t>(qb) * BQ;
  const int64_t q_hi = (q0 + BQ < p.n ? q0 + BQ : p.n);
  const int64_t kend = (p.q_off + q_hi < p.kv_len) ? p.q_off + q_hi : p.kv_len;
  const int nblk = static_cast<int>((kend + BKV - 1) / BKV);

  if (threadIdx.x == 0) {
    tc::mbar_init(q_full, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], 128);
      tc::mbar_init(&p_empty[i], 1);
    }
    for (int i = 0; i < KVS; ++i) {
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&k_empty[i], 1);
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&v_empty[i], 1);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: S0 [0,128) S1 [128,256) O [256, 256+hd). P_j (bf16) overwrites the
  // first 64 columns of its S buffer and feeds the PV MMA straight from TMEM.

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&p.tq.m0);
      tc::tma_prefetch(&p.tkv.m0);
      tc::mbar_expect_tx(q_full, TB);
      load_tile<HD>(sQ, p.tq, q_full, head * HD, static_cast<int>(q0), 128, 0);
      // K runs one block ahead of V: K_{j+1} (freed after S_{j+1-KVS}) is
      // requested before V_j (freed after PV_{j-KVS}), so PV never starves S.
      auto load_k = [&](int j) {
        const int st = j % KVS;
        tc::mbar_wait(&k_empty[st], ((j / KVS) & 1) ^ 1);
        tc::mbar_expect_tx(&k_full[st], TB);
        load_tile<HD>(sK + st * TB, p.tkv, &k_full[st], head * HD, j * BKV, 128, 0);
      };
      if (nblk > 0) load_k(0);
      for (int j = 0; j < nblk; ++j) {
        if (j + 1 < nblk) load_k(j + 1);
        const int st = j % KVS;
        tc::mbar_wait(&v_empty[st], ((j / KVS) & 1) ^ 1);
        tc::mbar_expect_tx(&v_full[st], TB);
        load_tile<HD>(sV + st * TB, p.tkv, &v_full[st], p.h + head * HD, j * BKV, 128, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16(128, BKV, false, false);
      tc::mbar_wait(q_full, 0);
      const uint32_t q_base = tc::smem_u32(sQ);
      // Poll two queues: S_j (needs K_j, and PV_{j-2} issued: S_j overwrites
      // the buffer P_{j-2} is read from; MMAs execute in issue order) and PV_j
      // (needs P_j and V_j).
      int sj = 0, pj = 0;
      while (pj < nblk) {
        if (sj < nblk && sj < pj + 2 && tc::mbar_test(&k_full[sj % KVS], (sj / KVS) & 1)) {
          const int b = sj & 1, st = sj % KVS;
          tc::tc_fence_after();
          const uint32_t k_base = tc::smem_u32(sK + st * TB);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk)
            tc::mma_bf16_ss(tmem + b * 128, kdesc<HD>(q_base, 128, kk), kdesc<HD>(k_base, 128, kk), idesc_s, kk > 0);
          tc::mma_commit(&s_full[b]);
          tc::mma_commit(&k_empty[st]);
          ++sj;
          continue;
        }
        if (pj < sj && tc::mbar_test(&p_full[pj & 1], (pj >> 1) & 1) &&
            tc::mbar_test(&v_full[pj % KVS], (pj / KVS) & 1)) {
          const int b = pj & 1, st = pj % KVS;
          tc::tc_fence_after();
          const uint32_t v_base = tc::smem_u32(sV + st * TB);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)  // O accumulates in TMEM; A = P_j from TMEM
            mma_nhd_ts<HD>(tmem + 256, tmem + b * 128 + kk * 8, v_base, 128, kk, pj > 0 || kk > 0);
          tc::mma_commit(&p_empty[b]);  // also marks PV_pj (and every earlier MMA) complete
          tc::mma_commit(&v_empty[st]);
          ++pj;
        }
      }
    }
  } else if (warp >= 4) {
    // Softmax: S row in registers (one pass), P -> TMEM, O stays in TMEM. The
    // running max used for exponentiation only moves when a block raises it by
    // more than 2^8 (log2 domain); then the O row in TMEM is rescaled once
    // PV_{j-1} has landed. Otherwise the softmax never waits for the PV MMAs.
    const int quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int64_t row = q0 + r;
    const bool valid = row < p.n;
    const int64_t qpos = p.q_off + row;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t obase = tmem + lane_base + 256;
    constexpr float kRescale = 8.f;
    float m = -INFINITY, l = 0.f;

    for (int j = 0; j < nblk; ++j) {
      const int b = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      const int64_t lim64 = (valid ? (qpos < p.kv_len - 1 ? qpos : p.kv_len - 1) : -1) - static_cast<int64_t>(j) * BKV;
      const int lim = lim64 > 1000000 ? 1000000 : static_cast<int>(lim64);  // columns <= lim are visible
      tc::mbar_wait(&s_full[b], ph);
      tc::tc_fence_after();
      const uint32_t sbase = tmem + lane_base + b * 128;
      uint32_t sv[128];
#pragma unroll
      for (int c = 0; c < 4; ++c) tc::tmem_ld32(sbase + c * 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[c * 32]));
      tc::tmem_ld_wait();
      // Raw scores stay unscaled (scale > 0 commutes with max); masking only on
      // blocks that touch the causal diagonal or the prefix end.
      float mx = -INFINITY;
      if (__all_sync(0xffffffffu, lim >= BKV - 1)) {
#pragma unroll
        for (int c = 0; c < 128; ++c) mx = fmaxf(mx, __uint_as_float(sv[c]));
      } else {
#pragma unroll
        for (int c = 0; c < 128; ++c) {
          if (c > lim) sv[c] = __float_as_uint(-INFINITY);
          mx = fmaxf(mx, __uint_as_float(sv[c]));
        }
      }
      mx *= p.scale_log2;
      const bool need = (m == -INFINITY) ? (mx > -INFINITY || j == 0) : (mx > m + kRescale);
      if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? fmaxf(m, mx) : m;
        const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - m_new);
        if (j > 0) {  // rescale the O row accumulated so far (PV_{j-1} must have landed)
          // PV_{j-1} landed <=> phase (j-1)>>1 of p_empty[(j-1)&1] completed. The
          // softmax already waited for that buffer's previous phase, so the
          // parity wait cannot alias an older phase.
          tc::mbar_wait(&p_empty[(j - 1) & 1], ((j - 1) >> 1) & 1);
          tc::tc_fence_after();
#pragma unroll
          for (int c = 0; c < HD / 16; ++c) {
            uint32_t v[16];
            tmem_ld16(obase + c * 16, v);
            tc::tmem_ld_wait();
#pragma unroll
            for (int e = 0; e < 16; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * alpha);
            tc::tmem_st16(obase + c * 16, v);
          }
          tc::tmem_st_wait();
        }
        l *= alpha;
        m = m_new;
      }
      const float neg_m = m == -INFINITY ? 0.f : -m;
      float rs0 = 0.f, rs1 = 0.f;
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float p0 = ex2(fmaf(__uint_as_float(sv[c * 32 + e]), p.scale_log2, neg_m));
          const float p1 = ex2(fmaf(__uint_as_float(sv[c * 32 + e + 1]), p.scale_log2, neg_m));
          rs0 += p0;
          rs1 += p1;
          w[e / 2] = pack_bf16(p0, p1);
        }
        tc::tmem_st16(sbase + c * 16, w);  // P keys [32c, 32c+32) -> columns [16c, 16c+16)
      }
      l += rs0 + rs1;
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&p_full[b]);
    }
    if (nblk > 0) tc::mbar_wait(&p_empty[(nblk - 1) & 1], ((nblk - 1) >> 1) & 1);  // last PV landed
    tc::tc_fence_after();
    const float inv = l > 0.f ? 1.f / l : 0.f;
    __nv_bfloat16* orow = p.o + (valid ? row : 0) * p.h + head * HD;
#pragma unroll
    for (int c = 0; c < HD / 16; ++c) {
      uint32_t v[16];
      tmem_ld16(obase + c * 16, v);  // warp-collective
      tc::tmem_ld_wait();
      if (!valid) continue;
      uint4 u0 = make_uint4(pack_bf16(__uint_as_float(v[0]) * inv, __uint_as_float(v[1]) * inv),
                            pack_bf16(__uint_as_float(v[2]) * inv, __uint_as_float(v[3]) * inv),
                            pack_bf16(__uint_as_float(v[4]) * inv, __uint_as_float(v[5]) * inv),
                            pack_bf16(__uint_as_float(v[6]) * inv, __uint_as_float(v[7]) * inv));
      uint4 u1 = make_uint4(pack_bf16(__uint_as_float(v[8]) * inv, __uint_as_float(v[9]) * inv),
                            pack_bf16(__uint_as_float(v[10]) * inv, __uint_as_float(v[11]) * inv),
                            pack_bf16(__uint_as_float(v[12]) * inv, __uint_as_float(v[13]) * inv),
                            pack_bf16(__uint_as_float(v[14]) * inv, __uint_as_float(v[15]) * inv));
      *reinterpret_cast<uint4*>(orow + c * 16) = u0;
      *reinterpret_cast<uint4*>(orow + c * 16 + 8) = u1;
    }
    if (valid) p.lse[static_cast<int64_t>(head) * p.n + row] = (m + log2f(l)) * 0.69314718055994531f;
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ============================================================================ backward

struct __align__(64) AttnBwdParams {
  Maps tq;           // q  [n, h]
  Maps tdo;          // dO [n, h]
  Maps tkv;          // kv [kv_len, 2h]
  const float* ld;   // [H, n_pad] x (LSE * log2e, delta), zero padded (attn_prep_k)
  int64_t n_pad;     // n rounded up to 64
  float* dkv;        // [kv_len, 2h] fp32 accumulator
  __nv_bfloat16* dq; // [n, h]
  int64_t n, q_off, kv_len;
  int H, h;
  float scale, scale_log2;
  int dbg;  // profiling only (SP_ATTN_DBG): 1 = skip dK/dV MMAs, 2 = skip dK/dV softmax math
};

template <int HD>
constexpr size_t dkv_smem_n(int st) {
  return 2 * Lay<HD>::bytes(128) + 2 * st * Lay<HD>::bytes(64) + st * 512 + (10 + 2 * st) * 8 + 8 + 1024;
}
template <int HD>
constexpr int dkv_stages() {
  int st = 6;
  while (dkv_smem_n<HD>(st) > 232448) --st;
  return st;
}
template <int HD>
constexpr size_t dkv_smem() {
  return dkv_smem_n<HD>(dkv_stages<HD>());
}
template <int HD>
constexpr size_t dq_smem_n(int st) {
  return 2 * Lay<HD>::bytes(128) + 2 * st * Lay<HD>::bytes(64) + (10 + 2 * st) * 8 + 8 + 1024;
}
template <int HD>
constexpr int dq_stages() {
  int st = 8;
  while (dq_smem_n<HD>(st) > 232448) --st;
  return st;
}
template <int HD>
constexpr size_t dq_smem() {
  return dq_smem_n<HD>(dq_stages<HD>());
}

// dK/dV: one CTA per (128-key block, head), looping over 64-query blocks that
// can see those keys: S^T = K Q_i^T and dP^T = V dO_i^T into TMEM; the softmax
// warps form P^T = exp2(S^T*c - LSE) and dS^T = P^T (dP^T - delta) as bf16
// over their S^T / dP^T columns in TMEM; dV += P^T dO_i and dK += dS^T Q_i
// take A from TMEM and accumulate in TMEM. Each (key row, head) slice of the
// fp32 dKV accumulator has exactly one owner CTA.
template <int HD>
__global__ void __launch_bounds__(384, 1) attn_bwd_dkv_k(const __grid_constant__ AttnBwdParams p) {
  constexpr int QST = dkv_stages<HD>();
  constexpr int KV_T = Lay<HD>::bytes(128), Q_T = Lay<HD>::bytes(64);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;
  uint8_t* sV = sK + KV_T;
  uint8_t* sQ = sV + KV_T;          // [QST]
  uint8_t* sdO = sQ + QST * Q_T;    // [QST]
  float* sLD = reinterpret_cast<float*>(sdO + QST * Q_T);  // [QST][64 x (lse*log2e, delta)]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sLD + QST * 128);
  uint64_t* kv_full = bars;
  uint64_t* s_full = bars + 1;   // [2]
  uint64_t* p_full = bars + 5;   // [2]
  uint64_t* done = bars + 9;
  uint64_t* q_full = bars + 10;          // [QST]
  uint64_t* q_empty = q_full + QST;      // [QST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_empty + QST);

  // 2-CTA cluster: CTAs own adjacent 128-key blocks and stream the same query
  // blocks; each Q_i / dO_i tile is fetched once from L2 and multicast to both
  // (rank 0 issues Q, rank 1 issues dO).
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = tc::cluster_ctarank();
  const int num_kb = static_cast<int>((p.kv_len + 127) / 128);
  const int num_kb2 = (num_kb + 1) & ~1;
  const int kb = num_kb2 - 1 - static_cast<int>(blockIdx.x);  // heaviest first; may be == num_kb (idle keys)
  const int head = blockIdx.y;
  const int64_t j0 = static_cast<int64_t>(kb) * 128;
  const int64_t j0_lo = static_cast<int64_t>(num_kb2 - 2 - 2 * static_cast<int>(blockIdx.x / 2)) * 128;
  int64_t ib0 = j0_lo - p.q_off;  // first query block any key of the pair can see (common to the cluster)
  if (ib0 < 0) ib0 = 0;
  ib0 = ib0 / 64 * 64;
  const int niter = static_cast<int>((p.n - ib0 + 63) / 64);

  if (threadIdx.x == 0) {
    tc::mbar_init(kv_full, 1);
    tc::mbar_init(done, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&p_full[i], 256);
    }
    for (int i = 0; i < QST; ++i) {
      tc::mbar_init(&q_full[i], 1);
      tc::mbar_init(&q_empty[i], 2);  // freed by both CTAs' MMA commits
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: S^T[2] at 0/64, dP^T[2] at 128/192, dV at 256, dK at 384. P^T and
  // dS^T (bf16) overwrite the S^T / dP^T columns they were computed from.

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&p.tq.m0);
      tc::tma_prefetch(&p.tdo.m0);
      tc::tma_prefetch(&p.tkv.m0);
      tc::mbar_expect_tx(kv_full, 2 * KV_T);
      load_tile<HD>(sK, p.tkv, kv_full, head * HD, static_cast<int>(j0), 128, 0);
      load_tile<HD>(sV, p.tkv, kv_full, p.h + head * HD, static_cast<int>(j0), 128, 0);
      for (int it = 0; it < niter; ++it) {
        const int st = it % QST;
        const int64_t i0 = ib0 + static_cast<int64_t>(it) * 64;
        tc::mbar_wait(&q_empty[st], ((it / QST) & 1) ^ 1);  // stage free in both CTAs
        tc::mbar_expect_tx(&q_full[st], 2 * Q_T + 512);
        if (rank == 0)
          load_tile<HD>(sQ + st * Q_T, p.tq, &q_full[st], head * HD, static_cast<int>(i0), 64, 3);
        else
          load_tile<HD>(sdO + st * Q_T, p.tdo, &q_full[st], head * HD, static_cast<int>(i0), 64, 3);
        // (LSE*log2e, delta) pairs of the 64 queries: one async 512-byte bulk copy
        tc::bulk_load(sLD + st * 128, p.ld + (static_cast<int64_t>(head) * p.n_pad + i0) * 2, 512, &q_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16(128, 64, false, false);
      tc::mbar_wait(kv_full, 0);
      const uint32_t k_base = tc::smem_u32(sK), v_base = tc::smem_u32(sV);
      // Two independent issue queues polled without blocking: S^T/dP^T of block
      // s_it (once dV/dK of block s_it-2, which read its TMEM buffer, have been
      // issued: MMAs execute in issue order) and dV/dK of block g_it.
      int s_it = 0, g_it = 0;
      while (g_it < niter) {
        if (s_it < niter && s_it < g_it + 2 && tc::mbar_test(&q_full[s_it % QST], (s_it / QST) & 1)) {
          const int it = s_it++;
          const int b = it & 1, st = it % QST;
          tc::tc_fence_after();
          const uint32_t q_base = tc::smem_u32(sQ + st * Q_T), do_base = tc::smem_u32(sdO + st * Q_T);
          if (!(p.dbg & 1)) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
              tc::mma_bf16_ss(tmem + b * 64, kdesc<HD>(k_base, 128, kk), kdesc<HD>(q_base, 64, kk), idesc_s, kk > 0);
              tc::mma_bf16_ss(tmem + 128 + b * 64, kdesc<HD>(v_base, 128, kk), kdesc<HD>(do_base, 64, kk), idesc_s,
                              kk > 0);
            }
          }
          tc::mma_commit(&s_full[b]);
          continue;
        }
        if (g_it < s_it && tc::mbar_test(&p_full[g_it & 1], (g_it >> 1) & 1)) {
          const int it = g_it++;
          const int b = it & 1, st = it % QST;
          tc::tc_fence_after();
          const uint32_t q_base = tc::smem_u32(sQ + st * Q_T), do_base = tc::smem_u32(sdO + st * Q_T);
          if (!(p.dbg & 1)) {
#pragma unroll
            for (int kk = 0; kk < 4; ++kk) {  // K = 64 queries
              const bool acc = it > 0 || kk > 0;
              mma_nhd_ts<HD>(tmem + 256, tmem + b * 64 + half_packed_col(kk), do_base, 64, kk, acc);
              mma_nhd_ts<HD>(tmem + 384, tmem + 128 + b * 64 + half_packed_col(kk), q_base, 64, kk, acc);
            }
          }
          tc::mma_commit_mc(&q_empty[st], 3);  // this CTA is done with the multicast stage
        }
      }
      tc::mma_commit(done);
    }
  } else if (warp >= 4) {
    // 8 softmax warps: warps w and w+4 share TMEM lane quarter w%4 (one key row
    // per lane) and split the 64 query columns in halves -> two warps per SMSP.
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int r = quarter * 32 + lane;  // key row
    const int64_t kpos = j0 + r;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    for (int it = 0; it < niter; ++it) {
      const int b = it & 1, st = it % QST;
      const uint32_t ph = (it >> 1) & 1;
      const int64_t i0 = ib0 + static_cast<int64_t>(it) * 64;
      const float* ld = sLD + st * 128 + half * 64;  // this half's 32 (lse, delta) pairs
      tc::mbar_wait(&q_full[st], (it / QST) & 1);    // LSE / delta of this block are in SMEM
      // visible query columns c (local to this half): q_off + i0 + 32*half + c >= kpos, i0 + 32*half + c < n
      const int64_t cbase = i0 + half * 32;
      int64_t cmin = kpos - p.q_off - cbase;
      const int c_lo = cmin < 0 ? 0 : (cmin > 32 ? 32 : static_cast<int>(cmin));
      const int64_t chi = p.n - cbase;
      const int c_hi = chi < 0 ? 0 : (chi > 32 ? 32 : static_cast<int>(chi));  // exclusive
      tc::mbar_wait(&s_full[b], ph);
      tc::tc_fence_after();
      uint32_t sv[32], dpv[32];
      tc::tmem_ld32(tmem + lane_base + b * 64 + half * 32, sv);
      tc::tmem_ld32(tmem + lane_base + 128 + b * 64 + half * 32, dpv);
      tc::tmem_ld_wait();
      const bool full_blk = __all_sync(0xffffffffu, c_lo == 0 && c_hi == 32);
      uint32_t wp[16], wd[16];
#pragma unroll
      for (int e = 0; e < 32; e += 4) {
        if (p.dbg & 2) break;
        const float4 a4 = lds_f4(ld + 2 * e);      // (lse, delta) of queries e, e+1 (warp broadcast)
        const float4 b4 = lds_f4(ld + 2 * e + 4);  // (lse, delta) of queries e+2, e+3
        const float lv[4] = {a4.x, a4.z, b4.x, b4.z}, dl[4] = {a4.y, a4.w, b4.y, b4.w};
        float pv[4], dv[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int c = e + u;
          float pr = ex2(fmaf(__uint_as_float(sv[c]), p.scale_log2, -lv[u]));
          if (!full_blk && (c < c_lo || c >= c_hi)) pr = 0.f;
          pv[u] = pr;
          dv[u] = pr * (__uint_as_float(dpv[c]) - dl[u]);
        }
        wp[e / 2] = pack_bf16(pv[0], pv[1]);
        wp[e / 2 + 1] = pack_bf16(pv[2], pv[3]);
        wd[e / 2] = pack_bf16(dv[0], dv[1]);
        wd[e / 2 + 1] = pack_bf16(dv[2], dv[3]);
      }
      tc::tmem_st16(tmem + lane_base + b * 64 + half * 32, wp);
      tc::tmem_st16(tmem + lane_base + 128 + b * 64 + half * 32, wd);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&p_full[b]);
    }
    tc::mbar_wait(done, 0);
    tc::tc_fence_after();
    const bool own = kpos < p.kv_len;
    float* dk_row = p.dkv + (own ? kpos : 0) * 2 * p.h + head * HD;
    float* dv_row = dk_row + p.h;
    constexpr int NCH = HD / 16, SPLIT = (NCH + 1) / 2;
    for (int c = half ? SPLIT : 0; c < (half ? NCH : SPLIT); ++c) {
      uint32_t v[16], k[16];
      // tcgen05.ld is warp-collective: every lane loads, only owners store.
      tmem_ld16(tmem + lane_base + 256 + c * 16, v);
      tmem_ld16(tmem + lane_base + 384 + c * 16, k);
      tc::tmem_ld_wait();
      if (own) {
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          float4 a = *reinterpret_cast<float4*>(dv_row + c * 16 + e);
          a.x += __uint_as_float(v[e]);
          a.y += __uint_as_float(v[e + 1]);
          a.z += __uint_as_float(v[e + 2]);
          a.w += __uint_as_float(v[e + 3]);
          *reinterpret_cast<float4*>(dv_row + c * 16 + e) = a;
          float4 g = *reinterpret_cast<float4*>(dk_row + c * 16 + e);
          g.x += __uint_as_float(k[e]) * p.scale;
          g.y += __uint_as_float(k[e + 1]) * p.scale;
          g.z += __uint_as_float(k[e + 2]) * p.scale;
          g.w += __uint_as_float(k[e + 3]) * p.scale;
          *reinterpret_cast<float4*>(dk_row + c * 16 + e) = g;
        }
      }
    }
  }
  tc::tc_fence_before();
  tc::cluster_sync();  // no multicast data / remote arrive may target an exited CTA
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// dQ: one CTA per (128-query block, head), looping over 64-key blocks:
// S = Q K_j^T, dP = dO V_j^T; dS = P (dP - delta) (bf16, over the dP columns
// in TMEM); dQ += dS K_j with A from TMEM.
template <int HD>
__global__ void __launch_bounds__(384, 1) attn_bwd_dq_k(const __grid_constant__ AttnBwdParams p) {
  constexpr int KST = dq_stages<HD>();
  constexpr int Q_T = Lay<HD>::bytes(128), K_T = Lay<HD>::bytes(64);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sdO = sQ + Q_T;
  uint8_t* sK = sdO + Q_T;        // [KST]
  uint8_t* sV = sK + KST * K_T;   // [KST]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + KST * K_T);
  uint64_t* qo_full = bars;
  uint64_t* s_full = bars + 1;    // [2]
  uint64_t* ds_full = bars + 5;   // [2]
  uint64_t* done = bars + 9;
  uint64_t* kv_full = bars + 10;       // [KST]
  uint64_t* kv_empty = kv_full + KST;  // [KST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(kv_empty + KST);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_qb = static_cast<int>((p.n + 127) / 128);
  const int qb = num_qb - 1 - static_cast<int>(blockIdx.x);
  const int head = blockIdx.y;
  const int64_t q0 = static_cast<int64_t>(qb) * 128;
  const int64_t q_hi = (q0 + 128 < p.n ? q0 + 128 : p.n);
  const int64_t kend = (p.q_off + q_hi < p.kv_len) ? p.q_off + q_hi : p.kv_len;
  const int nblk = static_cast<int>((kend + 63) / 64);

  if (threadIdx.x == 0) {
    tc::mbar_init(qo_full, 1);
    tc::mbar_init(done, 1);
    for (int i = 0; i < 2; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&ds_full[i], 256);
    }
    for (int i = 0; i < KST; ++i) {
      tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // TMEM: S[2] at 0/64, dP[2] at 128/192 (dS overwrites dP), dQ at 256.

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&p.tq.m0);
      tc::tma_prefetch(&p.tdo.m0);
      tc::tma_prefetch(&p.tkv.m0);
      tc::mbar_expect_tx(qo_full, 2 * Q_T);
      load_tile<HD>(sQ, p.tq, qo_full, head * HD, static_cast<int>(q0), 128, 0);
      load_tile<HD>(sdO, p.tdo, qo_full, head * HD, static_cast<int>(q0), 128, 0);
      for (int j = 0; j < nblk; ++j) {
        const int st = j % KST;
        tc::mbar_wait(&kv_empty[st], ((j / KST) & 1) ^ 1);
        tc::mbar_expect_tx(&kv_full[st], 2 * K_T);
        load_tile<HD>(sK + st * K_T, p.tkv, &kv_full[st], head * HD, j * 64, 64, 0);
        load_tile<HD>(sV + st * K_T, p.tkv, &kv_full[st], p.h + head * HD, j * 64, 64, 0);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16(128, 64, false, false);
      tc::mbar_wait(qo_full, 0);
      const uint32_t q_base = tc::smem_u32(sQ), do_base = tc::smem_u32(sdO);
      // Polled issue queues: S/dP of block sj (once dQ of block sj-2, which
      // reads dS from the same TMEM buffer, is issued) and dQ += dS K of block gj.
      int sj = 0, gj = 0;
      while (gj < nblk) {
        if (sj < nblk && sj < gj + 2 && tc::mbar_test(&kv_full[sj % KST], (sj / KST) & 1)) {
          const int j = sj++;
          const int b = j & 1, st = j % KST;
          tc::tc_fence_after();
          const uint32_t k_base = tc::smem_u32(sK + st * K_T), v_base = tc::smem_u32(sV + st * K_T);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            tc::mma_bf16_ss(tmem + b * 64, kdesc<HD>(q_base, 128, kk), kdesc<HD>(k_base, 64, kk), idesc_s, kk > 0);
            tc::mma_bf16_ss(tmem + 128 + b * 64, kdesc<HD>(do_base, 128, kk), kdesc<HD>(v_base, 64, kk), idesc_s,
                            kk > 0);
          }
          tc::mma_commit(&s_full[b]);
          continue;
        }
        if (gj < sj && tc::mbar_test(&ds_full[gj & 1], (gj >> 1) & 1)) {
          const int j = gj++;
          const int b = j & 1, st = j % KST;
          tc::tc_fence_after();
          const uint32_t k_base = tc::smem_u32(sK + st * K_T);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // K = 64 keys
            mma_nhd_ts<HD>(tmem + 256, tmem + 128 + b * 64 + half_packed_col(kk), k_base, 64, kk, j > 0 || kk > 0);
          tc::mma_commit(&kv_empty[st]);
        }
      }
      tc::mma_commit(done);
    }
  } else if (warp >= 4) {
    // 8 softmax warps: warps w and w+4 share lane quarter w%4 (one query row per
    // lane) and split the 64 key columns of each block in halves.
    const int quarter = warp & 3, half = (warp - 4) >> 2;
    const int r = quarter * 32 + lane;
    const int64_t row = q0 + r;
    const bool valid = row < p.n;
    const int64_t qpos = p.q_off + row;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const float2 ldv = *reinterpret_cast<const float2*>(p.ld + (static_cast<int64_t>(head) * p.n_pad + row) * 2);
    const float lse2 = ldv.x, dlt = ldv.y;  // zero-padded past n
    for (int j = 0; j < nblk; ++j) {
      const int b = j & 1;
      const uint32_t ph = (j >> 1) & 1;
      // key columns c (local to this half) with j*64 + 32*half + c <= qpos are visible
      const int64_t lim64 = valid ? qpos - static_cast<int64_t>(j) * 64 - half * 32 : -1;
      const int lim = lim64 > 1000 ? 1000 : static_cast<int>(lim64);
      tc::mbar_wait(&s_full[b], ph);
      tc::tc_fence_after();
      uint32_t sv[32], dpv[32];
      tc::tmem_ld32(tmem + lane_base + b * 64 + half * 32, sv);
      tc::tmem_ld32(tmem + lane_base + 128 + b * 64 + half * 32, dpv);
      tc::tmem_ld_wait();
      const bool full_blk = __all_sync(0xffffffffu, lim >= 31);
      uint32_t w[16];
#pragma unroll
      for (int e = 0; e < 32; e += 2) {
        float d2[2];
#pragma unroll
        for (int u = 0; u < 2; ++u) {
          const int c = e + u;
          float pr = ex2(fmaf(__uint_as_float(sv[c]), p.scale_log2, -lse2));
          if (!full_blk && c > lim) pr = 0.f;
          d2[u] = pr * (__uint_as_float(dpv[c]) - dlt);
        }
        w[e / 2] = pack_bf16(d2[0], d2[1]);
      }
      tc::tmem_st16(tmem + lane_base + 128 + b * 64 + half * 32, w);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      tc::mbar_arrive(&ds_full[b]);
    }
    tc::mbar_wait(done, 0);
    tc::tc_fence_after();
    __nv_bfloat16* dq_row = p.dq + (valid ? row : 0) * p.h + head * HD;
    constexpr int NCH = HD / 16, SPLIT = (NCH + 1) / 2;
    for (int c = half ? SPLIT : 0; c < (half ? NCH : SPLIT); ++c) {
      uint32_t v[16];
      tmem_ld16(tmem + lane_base + 256 + c * 16, v);  // warp-collective: all lanes
      tc::tmem_ld_wait();
      if (!valid) continue;
      uint4 u0 = make_uint4(pack_bf16(__uint_as_float(v[0]) * p.scale, __uint_as_float(v[1]) * p.scale),
                            pack_bf16(__uint_as_float(v[2]) * p.scale, __uint_as_float(v[3]) * p.scale),
                            pack_bf16(__uint_as_float(v[4]) * p.scale, __uint_as_float(v[5]) * p.scale),
                            pack_bf16(__uint_as_float(v[6]) * p.scale, __uint_as_float(v[7]) * p.scale));
      uint4 u1 = make_uint4(pack_bf16(__uint_as_float(v[8]) * p.scale, __uint_as_float(v[9]) * p.scale),
                            pack_bf16(__uint_as_float(v[10]) * p.scale, __uint_as_float(v[11]) * p.scale),
                            pack_bf16(__uint_as_float(v[12]) * p.scale, __uint_as_float(v[13]) * p.scale),
                            pack_bf16(__uint_as_float(v[14]) * p.scale, __uint_as_float(v[15]) * p.scale));
      *reinterpret_cast<uint4*>(dq_row + c * 16) = u0;
      *reinterpret_cast<uint4*>(dq_row + c * 16 + 8) = u1;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ld[head][i] = (lse * log2e, sum_d dO*O) for i < n, zeros up to n_pad: the
// per-query vectors the backward kernels stream (one warp per (i, head)).
__global__ void attn_prep_k(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                            const float* __restrict__ lse, float* __restrict__ ld, int64_t n, int64_t n_pad, int H,
                            int hd) {
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x / 32) + threadIdx.x / 32;
  const int lane = threadIdx.x % 32;
  if (w >= n_pad * H) return;
  const int head = static_cast<int>(w / n_pad);
  const int64_t i = w % n_pad;
  float d = 0.f, l = 0.f;
  if (i < n) {
    const int64_t base = i * (int64_t)H * hd + head * hd;
    for (int c = lane; c < hd; c += 32) d += __bfloat162float(o[base + c]) * __bfloat162float(dout[base + c]);
    d = warp_sum(d);
    l = lse[(int64_t)head * n + i] * 1.4426950408889634f;
  }
  if (lane == 0) *reinterpret_cast<float2*>(ld + (head * n_pad + i) * 2) = make_float2(l, d);
}

// ---------------------------------------------------------------------------- host

void make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t box_inner,
              uint32_t rows, CUtensorMapSwizzle sw) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {box_inner, rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = tma_encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                               CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (attention) failed: " + std::to_string((int)r));
}

// Chunk maps of a [outer, inner] bf16 tensor for [rows x hd] tiles.
void make_maps(Maps* t, const void* ptr, uint64_t inner, uint64_t outer, int hd, uint32_t rows) {
  make_map(&t->m0, ptr, inner, outer, inner, 64, rows, CU_TENSOR_MAP_SWIZZLE_128B);
  if (hd == 80 && Lay<80>::NARROW)
    make_map(&t->m1, ptr, inner, outer, inner, 16, rows, CU_TENSOR_MAP_SWIZZLE_32B);
  else
    t->m1 = t->m0;  // second chunk = another 64-wide SW128 box (hd 80: padded); hd 64: unused
}

}  // namespace

bool attn_tc_supported(DType t, int hd) { return t == DType::kBF16 && (hd == 64 || hd == 80 || hd == 128); }

void attn_fwd_tc(const void* q, const void* kv, void* o, float* lse, int64_t n, int64_t q_off, int64_t kv_len, int H,
                 int hd, cudaStream_t s) {
  AttnParams p;
  const int h = H * hd;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(kv) | reinterpret_cast<uintptr_t>(o)) & 15)
    throw std::invalid_argument("attention: operands must be 16-byte aligned");
  make_maps(&p.tq, q, h, n, hd, 128);
  make_maps(&p.tkv, kv, 2 * h, kv_len, hd, 128);
  p.o = static_cast<__nv_bfloat16*>(o);
  p.lse = lse;
  p.n = n;
  p.q_off = q_off;
  p.kv_len = kv_len;
  p.H = H;
  p.h = h;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(hd));
  auto run = [&](auto hd_tag) {
    constexpr int HD = decltype(hd_tag)::value;
    constexpr size_t smem = fwd_smem<HD>();
    static_assert(smem <= 232448, "attention fwd smem");
    SPK_CUDA(cudaFuncSetAttribute(attn_fwd_tc_k<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    dim3 grid(static_cast<unsigned>((n + BQ - 1) / BQ), static_cast<unsigned>(H));
    attn_fwd_tc_k<HD><<<grid, 256, smem, s>>>(p);
    SPK_LAUNCH_CHECK();
  };
  switch (hd) {
    case 64: run(std::integral_constant<int, 64>{}); break;
    case 80: run(std::integral_constant<int, 80>{}); break;
    case 128: run(std::integral_constant<int, 128>{}); break;
    default: throw std::invalid_argument("attention tc: head_dim must be 64, 80 or 128");
  }
}

size_t attn_bwd_ws_delta_floats(int64_t n, int H) { return static_cast<size_t>(H) * ((n + 63) / 64 * 64) * 2; }

void attn_bwd_tc(const void* q, const void* kv, const void* o, const void* dout, const float* lse, float* ws_delta,
                 float* ws_dq, void* dq, float* dkv, int64_t n, int64_t q_off, int64_t kv_len, int H, int hd,
                 cudaStream_t s) {
  const int h = H * hd;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(kv) | reinterpret_cast<uintptr_t>(dout) |
       reinterpret_cast<uintptr_t>(dq) | reinterpret_cast<uintptr_t>(dkv)) & 15)
    throw std::invalid_argument("attention: operands must be 16-byte aligned");
  (void)ws_dq;
  const int64_t n_pad = (n + 63) / 64 * 64;
  {
    const int64_t warps = n_pad * H;
    attn_prep_k<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), lse, ws_delta, n, n_pad, H, hd);
    SPK_LAUNCH_CHECK();
  }
  // dKV kernel: Q/dO tiles of 64 rows, K/V tiles of 128 rows; dQ kernel: the reverse.
  AttnBwdParams a;
  make_maps(&a.tq, q, h, n, hd, 64);
  make_maps(&a.tdo, dout, h, n, hd, 64);
  make_maps(&a.tkv, kv, 2 * h, kv_len, hd, 128);
  a.ld = ws_delta;
  a.n_pad = n_pad;
  a.dkv = dkv;
  a.dq = static_cast<__nv_bfloat16*>(dq);
  a.n = n;
  a.q_off = q_off;
  a.kv_len = kv_len;
  a.H = H;
  a.h = h;
  a.scale = 1.f / sqrtf(static_cast<float>(hd));
  a.scale_log2 = 1.4426950408889634f * a.scale;
  static const int dbg = [] {
    const char* e = std::getenv("SP_ATTN_DBG");
    return e ? std::atoi(e) : 0;
  }();
  a.dbg = dbg;
  AttnBwdParams b = a;
  make_maps(&b.tq, q, h, n, hd, 128);
  make_maps(&b.tdo, dout, h, n, hd, 128);
  make_maps(&b.tkv, kv, 2 * h, kv_len, hd, 64);
  auto run = [&](auto hd_tag) {
    constexpr int HD = decltype(hd_tag)::value;
    constexpr size_t smem_dkv = dkv_smem<HD>(), smem_dq = dq_smem<HD>();
    static_assert(smem_dkv <= 232448 && smem_dq <= 232448, "attention bwd smem");
    SPK_CUDA(cudaFuncSetAttribute(attn_bwd_dkv_k<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_dkv));
    SPK_CUDA(cudaFuncSetAttribute(attn_bwd_dq_k<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_dq));
    {
      const unsigned nkb2 = static_cast<unsigned>(((kv_len + 127) / 128 + 1) & ~int64_t(1));
      cudaLaunchConfig_t lc = {};
      lc.gridDim = dim3(nkb2, static_cast<unsigned>(H));
      lc.blockDim = dim3(384);
      lc.dynamicSmemBytes = smem_dkv;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      SPK_CUDA(cudaLaunchKernelEx(&lc, attn_bwd_dkv_k<HD>, a));
    }
    dim3 g2(static_cast<unsigned>((n + 127) / 128), static_cast<unsigned>(H));
    attn_bwd_dq_k<HD><<<g2, 384, smem_dq, s>>>(b);
    SPK_LAUNCH_CHECK();
  };
  switch (hd) {
    case 64: run(std::integral_constant<int, 64>{}); break;
    case 80: run(std::integral_constant<int, 80>{}); break;
    case 128: run(std::integral_constant<int, 128>{}); break;
    default: throw std::invalid_argument("attention tc: head_dim must be 64, 80 or 128");
  }
}

}  // namespace spk
