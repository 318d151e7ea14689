// tcgen05 causal prefix attention (bf16 in, fp32 softmax/accumulation).
//
// Forward: one CTA per (128-query block, head) of sub-sequence s, streaming the
// KV prefix [0, q_off + n) of the micro-batch's KV slab in 128-key blocks.
//   warp 0     TMA: Q once; K_j / V_j into a 2-stage ring (one tensor map over
//              the [kv_len, 2h] slab serves both: K at column head*hd, V at
//              h + head*hd)
//   warp 1     MMA: S_j = Q K_j^T (128x128xhd, SS) into TMEM S[j%2]; then
//              O_{j-1} = P_{j-1} V_{j-1} (128 x hd x 128, A = P from SMEM,
//              B = V as the MN-major operand) into TMEM O[(j-1)%2]
//   warps 4-7  softmax, one query row per thread: tcgen05.ld S row, online
//              max / exp2 / sum in fp32, P (bf16) written to SMEM in the
//              canonical K-major SW128 layout; O_{j-1} read back from TMEM
//              and rescaled into registers while the tensor core already
//              works on S_{j+1} / O_j.
// TMEM: S0 [0,128) S1 [128,256) O0 [256,384) O1 [384,512).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "cuda/common.cuh"
#include "cuda/ops.h"
#include "cuda/tc_common.cuh"

namespace spk {

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn();  // gemm_tcgen05.cu

namespace {

constexpr int BQ = 128, BKV = 128;
constexpr int CHUNK = 128 * 128;  // bytes of one [128 rows x 64 bf16] SW128 chunk

struct __align__(64) AttnParams {
  CUtensorMap tq;   // q [n, h]
  CUtensorMap tkv;  // kv [kv_len, 2h]
  __nv_bfloat16* o;
  float* lse;
  int64_t n, q_off, kv_len;
  int H, hd, h;
  float scale_log2;
};

__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&r)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
      : "r"(taddr));
}

// Store 32 bf16 values (16 packed words) of row r, columns [c32*32, c32*32+32) of a
// K-major SW128 [128 x 128] tile made of two 64-column chunks.
__device__ __forceinline__ void st_tile_row32(uint8_t* tile, int r, int c32, const uint32_t (&w)[16]) {
  uint8_t* chunk = tile + (c32 >> 1) * CHUNK + r * 128;
#pragma unroll
  for (int u = 0; u < 4; ++u) {
    const int unit = ((c32 & 1) * 4 + u) ^ (r & 7);
    *reinterpret_cast<uint4*>(chunk + unit * 16) = make_uint4(w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
  }
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
__global__ void __launch_bounds__(256, 1) attn_fwd_tc_k(const __grid_constant__ AttnParams p) {
  constexpr int NC = (HD + 63) / 64;  // 64-wide K chunks of the head dim
  constexpr int QBYTES = NC * CHUNK, KBYTES = NC * CHUNK, VBYTES = NC * CHUNK, PBYTES = 2 * CHUNK;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;
  uint8_t* sK = sQ + QBYTES;          // [2][KBYTES]
  uint8_t* sV = sK + 2 * KBYTES;      // [2][VBYTES]
  uint8_t* sP = sV + 2 * VBYTES;      // [2][PBYTES]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sP + 2 * PBYTES);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;   // [2]
  uint64_t* v_full = bars + 3;   // [2]
  uint64_t* kv_empty = bars + 5; // [2]
  uint64_t* s_full = bars + 7;   // [2]
  uint64_t* s_empty = bars + 9;  // [2]
  uint64_t* p_full = bars + 11;  // [2]
  uint64_t* p_empty = bars + 13; // [2]
  uint64_t* o_done = bars + 15;  // one phase per PV MMA group
  uint64_t* v_empty = bars + 16; // [2]  (kv_empty above now releases K stages only)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bars + 19);

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
      tc::mbar_init(&k_full[i], 1);
      tc::mbar_init(&v_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
      tc::mbar_init(&v_empty[i], 1);
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&s_empty[i], 128);
      tc::mbar_init(&p_full[i], 128);
      tc::mbar_init(&p_empty[i], 1);
    }
    tc::mbar_init(o_done, 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&p.tq);
      tc::tma_prefetch(&p.tkv);
      tc::mbar_expect_tx(q_full, QBYTES);
      for (int c = 0; c < NC; ++c)
        tc::tma_load_2d(sQ + c * CHUNK, &p.tq, q_full, head * HD + 64 * c, static_cast<int>(q0));
      // K runs one block ahead of V: K_{j+1} (freed after S_{j-1}) is requested
      // before V_j (freed after PV_{j-2}) so a slow PV never starves S.
      auto load_k = [&](int j) {
        const int st = j & 1;
        tc::mbar_wait(&kv_empty[st], ((j >> 1) & 1) ^ 1);
        tc::mbar_expect_tx(&k_full[st], KBYTES);
        for (int c = 0; c < NC; ++c)
          tc::tma_load_2d(sK + st * KBYTES + c * CHUNK, &p.tkv, &k_full[st], head * HD + 64 * c, j * BKV);
      };
      if (nblk > 0) load_k(0);
      for (int j = 0; j < nblk; ++j) {
        if (j + 1 < nblk) load_k(j + 1);
        const int st = j & 1;
        tc::mbar_wait(&v_empty[st], ((j >> 1) & 1) ^ 1);
        tc::mbar_expect_tx(&v_full[st], VBYTES);
        for (int c = 0; c < NC; ++c)
          tc::tma_load_2d(sV + st * VBYTES + c * CHUNK, &p.tkv, &v_full[st], p.h + head * HD + 64 * c, j * BKV);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16(128, BKV, false, false);
      constexpr uint32_t idesc_o = tc::idesc_bf16(128, HD, false, true);
      tc::mbar_wait(q_full, 0);
      const uint32_t q_base = tc::smem_u32(sQ);
      // Poll two queues: S_j (needs K_j and a free S buffer) and PV_j (needs P_j
      // and V_j). K and V stages are released separately (K after S_j, V after
      // PV_j), so S can run two blocks ahead of the softmax.
      int sj = 0, pj = 0;
      while (pj < nblk) {
        if (sj < nblk && tc::mbar_test(&k_full[sj & 1], (sj >> 1) & 1) &&
            tc::mbar_test(&s_empty[sj & 1], ((sj >> 1) & 1) ^ 1)) {
          const int b = sj & 1;
          tc::tc_fence_after();
          const uint32_t k_base = tc::smem_u32(sK + b * KBYTES);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off = (kk >> 2) * CHUNK + (kk & 3) * 32;
            tc::mma_bf16_ss(tmem + b * 128, tc::smem_desc(q_base + off, 16, 1024, tc::kSwizzle128B),
                            tc::smem_desc(k_base + off, 16, 1024, tc::kSwizzle128B), idesc_s, kk > 0);
          }
          tc::mma_commit(&s_full[b]);
          tc::mma_commit(&kv_empty[b]);  // K stage free
          ++sj;
          continue;
        }
        if (pj < sj && tc::mbar_test(&p_full[pj & 1], (pj >> 1) & 1) && tc::mbar_test(&v_full[pj & 1], (pj >> 1) & 1)) {
          const int b = pj & 1;
          tc::tc_fence_after();
          const uint32_t p_base = tc::smem_u32(sP + b * PBYTES);
          const uint32_t v_base = tc::smem_u32(sV + b * VBYTES);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk) {
            const uint64_t ad = tc::smem_desc(p_base + (kk >> 2) * CHUNK + (kk & 3) * 32, 16, 1024, tc::kSwizzle128B);
            const uint64_t bd = tc::smem_desc(v_base + kk * 2048, CHUNK, 1024, tc::kSwizzle128B);
            tc::mma_bf16_ss(tmem + 256, ad, bd, idesc_o, pj > 0 || kk > 0);  // O accumulates in TMEM
          }
          tc::mma_commit(o_done);
          tc::mma_commit(&p_empty[b]);
          tc::mma_commit(&v_empty[b]);  // V stage free
          ++pj;
        }
      }
    }
  } else if (warp >= 4) {
    // Softmax: S row in registers (one pass), P -> SMEM, O stays in TMEM. The
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
      tc::tc_fence_before();
      tc::mbar_arrive(&s_empty[b]);  // S buffer free: the MMA warp may issue S_{j+2}
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
          tc::mbar_wait(o_done, (j - 1) & 1);
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
      tc::mbar_wait(&p_empty[b], ph ^ 1);
      uint8_t* ptile = sP + b * PBYTES;
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
        st_tile_row32(ptile, r, c, w);
      }
      const float rs = rs0 + rs1;
      l += rs;
      tc::tc_fence_before();
      fence_async_smem();
      tc::mbar_arrive(&p_full[b]);
    }
    tc::mbar_wait(o_done, (nblk - 1) & 1);  // last PV landed
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
//
// dK/dV kernel: one CTA per (128-key block, head), looping over 64-query
// blocks that can see those keys:
//   S^T = K Q_i^T, dP^T = V dO_i^T (M = 128 keys, N = 64 queries) into TMEM;
//   one thread per key row: P^T = exp2(S^T*c - LSE), dS^T = P^T (dP^T - D)
//   written to SMEM (K-major); dV += P^T dO_i and dK += dS^T Q_i accumulate in
//   TMEM (the Q_i / dO_i tiles double as MN-major B operands: a [rows x 64]
//   SW128 tile is both layouts). The block's dK/dV are added once into the fp32
//   dKV accumulator: each (key row, head) slice has one owner (no atomics).
// dQ kernel: one CTA per (128-query block, head), looping over 64-key blocks:
//   S = Q K_j^T, dP = dO V_j^T; dS = P (dP - D) -> SMEM; dQ += dS K_j in TMEM.
// Together: 7 tensor-core GEMMs per (q,k) block pair, fully deterministic.

struct __align__(64) AttnBwdParams {
  CUtensorMap tq;    // q   [n, h]      box 64 rows
  CUtensorMap tdo;   // dO  [n, h]      box 64 rows (dKV kernel) / 128 rows (dQ kernel)
  CUtensorMap tkv;   // kv  [kv_len, 2h] box 128 rows (dKV kernel) / 64 rows (dQ kernel)
  const float* ld;     // [H, n_pad] x (LSE * log2e, delta), zero padded (attn_prep_k)
  int64_t n_pad;       // n rounded up to 64
  float* dkv;        // [kv_len, 2h] fp32 accumulator
  __nv_bfloat16* dq; // [n, h]
  int64_t n, q_off, kv_len;
  int H, h;
  float scale, scale_log2;
  int dbg;  // profiling only (SP_ATTN_DBG): 1 = skip MMAs, 2 = skip softmax math
};

template <int HD>
__global__ void __launch_bounds__(384, 1) attn_bwd_dkv_k(const __grid_constant__ AttnBwdParams p) {
  constexpr int NC = (HD + 63) / 64;
  constexpr int KV_T = NC * CHUNK;       // [128 rows x hd] tile
  constexpr int Q_T = NC * CHUNK / 2;    // [64 rows x hd] tile (chunks of 8 KB)
  constexpr int QCH = CHUNK / 2;
  constexpr int PT = CHUNK;              // [128 keys x 64 queries] bf16 tile
  constexpr int QST = NC == 1 ? 4 : 3;   // Q / dO / (LSE, delta) ring depth
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;
  uint8_t* sV = sK + KV_T;
  uint8_t* sQ = sV + KV_T;          // [QST]
  uint8_t* sdO = sQ + QST * Q_T;    // [QST]
  uint8_t* sPt = sdO + QST * Q_T;   // [2]
  uint8_t* sdSt = sPt + 2 * PT;     // [2]
  float* sLD = reinterpret_cast<float*>(sdSt + 2 * PT);  // [QST][64 x (lse*log2e, delta)]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sLD + QST * 128);
  uint64_t* kv_full = bars;
  uint64_t* s_full = bars + 1;   // [2]
  uint64_t* s_empty = bars + 3;  // [2]
  uint64_t* p_full = bars + 5;   // [2]
  uint64_t* p_empty = bars + 7;  // [2]
  uint64_t* done = bars + 9;
  uint64_t* q_full = bars + 10;          // [QST]
  uint64_t* q_empty = q_full + QST;      // [QST]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(q_empty + QST);

  // 2-CTA cluster: CTAs own adjacent 128-key blocks and stream the same query
  // blocks; each Q_i / dO_i tile is fetched once from L2 and multicast to both
  // (rank 0 issues Q, rank 1 issues dO), halving the dominant L2 -> SMEM traffic.
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = tc::cluster_ctarank();
  const int num_kb = static_cast<int>((p.kv_len + 127) / 128);
  const int num_kb2 = (num_kb + 1) & ~1;
  const int kb = num_kb2 - 1 - static_cast<int>(blockIdx.x);   // heaviest first; may be == num_kb (idle keys)
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
      tc::mbar_init(&s_empty[i], 256);
      tc::mbar_init(&p_full[i], 256);
      tc::mbar_init(&p_empty[i], 1);
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
  // TMEM: S^T[2] at 0/64, dP^T[2] at 128/192, dV at 256, dK at 384.

  if (warp == 0) {
    // Producer warp: K/V once; per query block the Q / dO tiles (TMA) and the
    // block's LSE / delta vectors (all 32 lanes), QST stages ahead of the consumers.
    if (lane == 0) {
      tc::tma_prefetch(&p.tq);
      tc::tma_prefetch(&p.tdo);
      tc::tma_prefetch(&p.tkv);
      tc::mbar_expect_tx(kv_full, 2 * KV_T);
      for (int c = 0; c < NC; ++c) {
        tc::tma_load_2d(sK + c * CHUNK, &p.tkv, kv_full, head * HD + 64 * c, static_cast<int>(j0));
        tc::tma_load_2d(sV + c * CHUNK, &p.tkv, kv_full, p.h + head * HD + 64 * c, static_cast<int>(j0));
      }
    }
    if (lane == 0) {
      for (int it = 0; it < niter; ++it) {
        const int st = it % QST;
        const int64_t i0 = ib0 + static_cast<int64_t>(it) * 64;
        tc::mbar_wait(&q_empty[st], ((it / QST) & 1) ^ 1);  // stage free in both CTAs
        tc::mbar_expect_tx(&q_full[st], 2 * Q_T + 512);
        for (int c = 0; c < NC; ++c) {
          if (rank == 0)
            tc::tma_load_2d_mc(sQ + st * Q_T + c * QCH, &p.tq, &q_full[st], head * HD + 64 * c, static_cast<int>(i0), 3);
          else
            tc::tma_load_2d_mc(sdO + st * Q_T + c * QCH, &p.tdo, &q_full[st], head * HD + 64 * c, static_cast<int>(i0),
                               3);
        }
        // (LSE*log2e, delta) pairs of the 64 queries: one async 512-byte bulk copy
        tc::bulk_load(sLD + st * 128, p.ld + (static_cast<int64_t>(head) * p.n_pad + i0) * 2, 512, &q_full[st]);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16(128, 64, false, false);
      constexpr uint32_t idesc_g = tc::idesc_bf16(128, HD, false, true);
      tc::mbar_wait(kv_full, 0);
      const uint32_t k_base = tc::smem_u32(sK), v_base = tc::smem_u32(sV);
      // Two independent issue queues polled without blocking: S^T/dP^T of block
      // s_it (needs its Q/dO stage and a free S buffer — released by the softmax
      // warps right after their TMEM load) and dV/dK of block g_it (needs that
      // block's P^T/dS^T). S can therefore run up to two blocks ahead of the
      // softmax instead of waiting behind the previous dV/dK in program order.
      int s_it = 0, g_it = 0;
      while (g_it < niter) {
        const bool s_ready = s_it < niter && tc::mbar_test(&q_full[s_it % QST], (s_it / QST) & 1) &&
                             tc::mbar_test(&s_empty[s_it & 1], ((s_it >> 1) & 1) ^ 1);
        if (s_ready) {
          const int it = s_it++;
          const int b = it & 1, st = it % QST;
          tc::tc_fence_after();
          const uint32_t q_base = tc::smem_u32(sQ + st * Q_T), do_base = tc::smem_u32(sdO + st * Q_T);
          if (!(p.dbg & 1)) {
#pragma unroll
            for (int kk = 0; kk < HD / 16; ++kk) {
              const uint32_t off_kv = (kk >> 2) * CHUNK + (kk & 3) * 32;
              const uint32_t off_q = (kk >> 2) * QCH + (kk & 3) * 32;
              tc::mma_bf16_ss(tmem + b * 64, tc::smem_desc(k_base + off_kv, 16, 1024, tc::kSwizzle128B),
                              tc::smem_desc(q_base + off_q, 16, 1024, tc::kSwizzle128B), idesc_s, kk > 0);
              tc::mma_bf16_ss(tmem + 128 + b * 64, tc::smem_desc(v_base + off_kv, 16, 1024, tc::kSwizzle128B),
                              tc::smem_desc(do_base + off_q, 16, 1024, tc::kSwizzle128B), idesc_s, kk > 0);
            }
          }
          tc::mma_commit(&s_full[b]);
          continue;
        }
        if (g_it < s_it && tc::mbar_test(&p_full[g_it & 1], (g_it >> 1) & 1)) {
          const int it = g_it++;
          const int b = it & 1, st = it % QST;
          tc::tc_fence_after();
          const uint32_t pt = tc::smem_u32(sPt + b * PT), dst = tc::smem_u32(sdSt + b * PT);
          const uint32_t q_base = tc::smem_u32(sQ + st * Q_T), do_base = tc::smem_u32(sdO + st * Q_T);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // K = 64 queries
            if (p.dbg & 1) break;
            const bool acc = it > 0 || kk > 0;
            tc::mma_bf16_ss(tmem + 256, tc::smem_desc(pt + kk * 32, 16, 1024, tc::kSwizzle128B),
                            tc::smem_desc(do_base + kk * 2048, QCH, 1024, tc::kSwizzle128B), idesc_g, acc);
            tc::mma_bf16_ss(tmem + 384, tc::smem_desc(dst + kk * 32, 16, 1024, tc::kSwizzle128B),
                            tc::smem_desc(q_base + kk * 2048, QCH, 1024, tc::kSwizzle128B), idesc_g, acc);
          }
          tc::mma_commit(&p_empty[b]);
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
      tc::mbar_wait(&q_full[st], (it / QST) & 1);  // LSE / delta of this block are in SMEM
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
      tc::tc_fence_before();
      tc::mbar_arrive(&s_empty[b]);
      tc::mbar_wait(&p_empty[b], ph ^ 1);
      const bool full_blk = __all_sync(0xffffffffu, c_lo == 0 && c_hi == 32);
      uint32_t wp[16], wd[16];
#pragma unroll
      for (int e = 0; e < 32; e += 4) {
        if (p.dbg & 2) break;
        const float4 a4 = *reinterpret_cast<const float4*>(ld + 2 * e);      // (lse, delta) of queries e, e+1
        const float4 b4 = *reinterpret_cast<const float4*>(ld + 2 * e + 4);  // (lse, delta) of queries e+2, e+3
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
      st_tile_row32(sPt + b * PT, r, half, wp);
      st_tile_row32(sdSt + b * PT, r, half, wd);
      fence_async_smem();
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

template <int HD>
__global__ void __launch_bounds__(384, 1) attn_bwd_dq_k(const __grid_constant__ AttnBwdParams p) {
  constexpr int NC = (HD + 63) / 64;
  constexpr int Q_T = NC * CHUNK;        // [128 rows x hd]
  constexpr int K_T = NC * CHUNK / 2;    // [64 rows x hd]
  constexpr int KCH = CHUNK / 2;
  constexpr int DS_T = CHUNK;            // [128 q x 64 keys]
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  constexpr int KST = 4;  // K/V ring depth
  uint8_t* sQ = sm;
  uint8_t* sdO = sQ + Q_T;
  uint8_t* sK = sdO + Q_T;       // [KST]
  uint8_t* sV = sK + KST * K_T;  // [KST]
  uint8_t* sdS = sV + KST * K_T; // [2]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sdS + 2 * DS_T);
  uint64_t* qo_full = bars;
  uint64_t* s_full = bars + 1;    // [2]
  uint64_t* s_empty = bars + 3;   // [2]
  uint64_t* ds_full = bars + 5;   // [2]
  uint64_t* ds_empty = bars + 7;  // [2]
  uint64_t* done = bars + 9;
  uint64_t* kv_full = bars + 10;          // [KST]
  uint64_t* kv_empty = kv_full + KST;     // [KST]
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
      tc::mbar_init(&s_empty[i], 256);
      tc::mbar_init(&ds_full[i], 256);
      tc::mbar_init(&ds_empty[i], 1);
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
  // TMEM: S[2] at 0/64, dP[2] at 128/192, dQ at 256.

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&p.tq);
      tc::tma_prefetch(&p.tdo);
      tc::tma_prefetch(&p.tkv);
      tc::mbar_expect_tx(qo_full, 2 * Q_T);
      for (int c = 0; c < NC; ++c) {
        tc::tma_load_2d(sQ + c * CHUNK, &p.tq, qo_full, head * HD + 64 * c, static_cast<int>(q0));
        tc::tma_load_2d(sdO + c * CHUNK, &p.tdo, qo_full, head * HD + 64 * c, static_cast<int>(q0));
      }
      for (int j = 0; j < nblk; ++j) {
        const int st = j % KST;
        tc::mbar_wait(&kv_empty[st], ((j / KST) & 1) ^ 1);
        tc::mbar_expect_tx(&kv_full[st], 2 * K_T);
        for (int c = 0; c < NC; ++c) {
          tc::tma_load_2d(sK + st * K_T + c * KCH, &p.tkv, &kv_full[st], head * HD + 64 * c, j * 64);
          tc::tma_load_2d(sV + st * K_T + c * KCH, &p.tkv, &kv_full[st], p.h + head * HD + 64 * c, j * 64);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc_s = tc::idesc_bf16(128, 64, false, false);
      constexpr uint32_t idesc_q = tc::idesc_bf16(128, HD, false, true);
      tc::mbar_wait(qo_full, 0);
      const uint32_t q_base = tc::smem_u32(sQ), do_base = tc::smem_u32(sdO);
      int sj = 0, gj = 0;  // polled issue queues: S/dP of block sj, dQ += dS K of block gj
      while (gj < nblk) {
        if (sj < nblk && tc::mbar_test(&kv_full[sj % KST], (sj / KST) & 1) &&
            tc::mbar_test(&s_empty[sj & 1], ((sj >> 1) & 1) ^ 1)) {
          const int j = sj++;
          const int b = j & 1, st = j % KST;
          tc::tc_fence_after();
          const uint32_t k_base = tc::smem_u32(sK + st * K_T), v_base = tc::smem_u32(sV + st * K_T);
#pragma unroll
          for (int kk = 0; kk < HD / 16; ++kk) {
            const uint32_t off_q = (kk >> 2) * CHUNK + (kk & 3) * 32;
            const uint32_t off_k = (kk >> 2) * KCH + (kk & 3) * 32;
            tc::mma_bf16_ss(tmem + b * 64, tc::smem_desc(q_base + off_q, 16, 1024, tc::kSwizzle128B),
                            tc::smem_desc(k_base + off_k, 16, 1024, tc::kSwizzle128B), idesc_s, kk > 0);
            tc::mma_bf16_ss(tmem + 128 + b * 64, tc::smem_desc(do_base + off_q, 16, 1024, tc::kSwizzle128B),
                            tc::smem_desc(v_base + off_k, 16, 1024, tc::kSwizzle128B), idesc_s, kk > 0);
          }
          tc::mma_commit(&s_full[b]);
          continue;
        }
        if (gj < sj && tc::mbar_test(&ds_full[gj & 1], (gj >> 1) & 1)) {
          const int j = ++gj;  // j - 1 == the block being consumed (keeps the (j - 1) terms below)
          const int b = (j - 1) & 1, st = (j - 1) % KST;
          tc::tc_fence_after();
          const uint32_t ds = tc::smem_u32(sdS + b * DS_T), k_base = tc::smem_u32(sK + st * K_T);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)  // K = 64 keys
            tc::mma_bf16_ss(tmem + 256, tc::smem_desc(ds + kk * 32, 16, 1024, tc::kSwizzle128B),
                            tc::smem_desc(k_base + kk * 2048, KCH, 1024, tc::kSwizzle128B), idesc_q,
                            (j - 1) > 0 || kk > 0);
          tc::mma_commit(&ds_empty[b]);
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
      tc::tc_fence_before();
      tc::mbar_arrive(&s_empty[b]);
      tc::mbar_wait(&ds_empty[b], ph ^ 1);
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
      st_tile_row32(sdS + b * DS_T, r, half, w);
      fence_async_smem();
      tc::mbar_arrive(&ds_full[b]);
    }
    tc::mbar_wait(done, 0);
    tc::tc_fence_after();
    {
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
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

void make_map(CUtensorMap* m, const void* ptr, uint64_t inner, uint64_t outer, uint64_t ld_elems, uint32_t rows = 128) {
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {64, rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = tma_encode_fn()(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(ptr), dims, strides, box, estr,
                               CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                               CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (attention) failed: " + std::to_string((int)r));
}

template <int HD>
size_t fwd_smem_bytes() {
  constexpr int NC = (HD + 63) / 64;
  return NC * CHUNK * 5 + 4 * CHUNK + 1024 + 256;
}

template <int HD>
void launch_fwd(const AttnParams& p, cudaStream_t s) {
  const size_t smem = fwd_smem_bytes<HD>();
  SPK_CUDA(cudaFuncSetAttribute(attn_fwd_tc_k<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid(static_cast<unsigned>((p.n + BQ - 1) / BQ), static_cast<unsigned>(p.H));
  attn_fwd_tc_k<HD><<<grid, 256, smem, s>>>(p);
  SPK_LAUNCH_CHECK();
}

}  // namespace

bool attn_tc_supported(DType t, int hd) { return t == DType::kBF16 && (hd == 64 || hd == 80 || hd == 128); }

void attn_fwd_tc(const void* q, const void* kv, void* o, float* lse, int64_t n, int64_t q_off, int64_t kv_len, int H,
                 int hd, cudaStream_t s) {
  AttnParams p;
  const int h = H * hd;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(kv) | reinterpret_cast<uintptr_t>(o)) & 15)
    throw std::invalid_argument("attention: operands must be 16-byte aligned");
  make_map(&p.tq, q, h, n, h);
  make_map(&p.tkv, kv, 2 * h, kv_len, 2 * h);
  p.o = static_cast<__nv_bfloat16*>(o);
  p.lse = lse;
  p.n = n;
  p.q_off = q_off;
  p.kv_len = kv_len;
  p.H = H;
  p.hd = hd;
  p.h = h;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(hd));
  switch (hd) {
    case 64: launch_fwd<64>(p, s); break;
    case 80: launch_fwd<80>(p, s); break;
    case 128: launch_fwd<128>(p, s); break;
    default: throw std::invalid_argument("attention tc: head_dim must be 64, 80 or 128");
  }
}

namespace {
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
}  // namespace

size_t attn_bwd_ws_delta_floats(int64_t n, int H) { return static_cast<size_t>(H) * ((n + 63) / 64 * 64) * 2; }

void attn_bwd_tc(const void* q, const void* kv, const void* o, const void* dout, const float* lse, float* ws_delta,
                 float* ws_dq, void* dq, float* dkv, int64_t n, int64_t q_off, int64_t kv_len, int H, int hd,
                 cudaStream_t s) {
  const int h = H * hd;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(kv) | reinterpret_cast<uintptr_t>(dout) |
       reinterpret_cast<uintptr_t>(dq) | reinterpret_cast<uintptr_t>(dkv)) & 15)
    throw std::invalid_argument("attention: operands must be 16-byte aligned");
  const int64_t n_pad = (n + 63) / 64 * 64;
  {
    const int64_t warps = n_pad * H;
    attn_prep_k<<<static_cast<unsigned>((warps + 7) / 8), 256, 0, s>>>(
        static_cast<const __nv_bfloat16*>(o), static_cast<const __nv_bfloat16*>(dout), lse, ws_delta, n, n_pad, H, hd);
    SPK_LAUNCH_CHECK();
  }
  // dKV kernel: Q/dO boxes of 64 rows, KV boxes of 128 rows; dQ kernel: the reverse.
  AttnBwdParams a;
  make_map(&a.tq, q, h, n, h, 64);
  make_map(&a.tdo, dout, h, n, h, 64);
  make_map(&a.tkv, kv, 2 * h, kv_len, 2 * h, 128);
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
  make_map(&b.tq, q, h, n, h, 128);
  make_map(&b.tdo, dout, h, n, h, 128);
  make_map(&b.tkv, kv, 2 * h, kv_len, 2 * h, 64);
  (void)ws_dq;
  auto run = [&](auto hd_tag) {
    constexpr int HD = decltype(hd_tag)::value;
    constexpr int NC = (HD + 63) / 64;
    constexpr int QST = NC == 1 ? 4 : 3, KST = 4;
    const size_t smem_dkv = 2 * NC * CHUNK + 2 * QST * (NC * CHUNK / 2) + 4 * CHUNK + QST * 512 + (10 + 2 * QST) * 8 + 8 +
                            1024;
    const size_t smem_dq = 2 * NC * CHUNK + 2 * KST * (NC * CHUNK / 2) + 2 * CHUNK + (6 + 2 * KST) * 8 + 8 + 1024;
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
    SPK_LAUNCH_CHECK();
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
