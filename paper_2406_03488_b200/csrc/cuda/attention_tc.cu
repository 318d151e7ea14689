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

#include <cstdio>
#include <cstdlib>
#include <type_traits>

#include "cuda/common.cuh"
#include "cuda/ops.h"
#include "cuda/tc_common.cuh"

namespace spk {

PFN_cuTensorMapEncodeTiled_v12000 tma_encode_fn();  // gemm_tcgen05.cu

namespace {

constexpr int BQ = 128, BKV = 128;

template <int HD>
struct Lay {
  // hd 80 holds its last 16 columns in a second 64-wide SW128 chunk (padded): one N = hd MMA per
  // K step. (A 64 + 16 SW32 split measured slower: N = 16 MMAs and 32-byte TMA rows.)
  static constexpr int C1 = HD <= 64 ? 0 : 64;  // columns held by the second chunk
  static constexpr int R1 = C1 * 2;                              // bytes per row of the second chunk
  static constexpr int bytes(int rows) { return rows * (128 + R1); }
};

// K-major descriptor of head-dim step kk (16 dims) of a [rows x hd] tile.
template <int HD>
__device__ __forceinline__ uint64_t kdesc(uint32_t base, int rows, int kk) {
  if (kk < 4) return tc::smem_desc(base + kk * 32, 16, 1024, tc::kSwizzle128B);
  return tc::smem_desc(base + rows * 128 + (kk - 4) * 32, 16, 1024, tc::kSwizzle128B);
}

// D[128 x hd] (+)= A[128 x 16 (K step kk)] * B[K rows of a [rows x hd] tile]^T, B MN-major.
template <int HD>
__device__ __forceinline__ void mma_nhd(uint32_t d, uint64_t adesc, uint32_t bbase, int rows, int kk, bool acc) {
  constexpr uint32_t id = tc::idesc_bf16(128, HD, false, true);  // padded second chunk: one N = hd MMA
  tc::mma_bf16_ss_w(d, adesc, tc::smem_desc(bbase + kk * 2048, rows * 128, 1024, tc::kSwizzle128B), id, acc);
}

// Same with A (M=128 x K=16, bf16 packed two per 32-bit column) read from TMEM.
template <int HD>
__device__ __forceinline__ void mma_nhd_ts(uint32_t d, uint32_t a_tmem, uint32_t bbase, int rows, int kk, bool acc) {
  constexpr uint32_t id = tc::idesc_bf16(128, HD, false, true);
  tc::mma_bf16_ts_w(d, a_tmem, tc::smem_desc(bbase + kk * 2048, rows * 128, 1024, tc::kSwizzle128B), id, acc);
}


// One arrive per warp (count barriers in warps): a 512-thread arrive costs
// hundreds of cycles of shared-memory atomics per phase.
__device__ __forceinline__ void warp_arrive(uint64_t* bar) {
  __syncwarp();
  if ((threadIdx.x & 31) == 0) tc::mbar_arrive(bar);
}

__device__ __forceinline__ void sts_f32(const void* p, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))), "f"(v) : "memory");
}
__device__ __forceinline__ float lds_f32(const void* p) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(p))) : "memory");
  return v;
}

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
  const __nv_bfloat16* q;  // raw rows (copied into TMEM as the S-MMA A operand, hd <= 80)
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

__device__ __forceinline__ int clamp_i32(int64_t v) {  // to +-2^30: mask bounds stay exact
  return static_cast<int>(v < -(int64_t(1) << 30) ? -(int64_t(1) << 30) : (v > (int64_t(1) << 30) ? (int64_t(1) << 30) : v));
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

// Packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2: two lanes per issue
// slot) and the 3-input max (FMNMX3). The softmax loops are issue-bound, so
// these halve their FMA-pipe instruction count.
__device__ __forceinline__ float2 ffma2(float2 a, float2 b, float2 c) {
  float2 d;
  asm("{\n\t.reg .b64 a, b, c, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\tmov.b64 c, {%6, %7};\n\t"
      "fma.rn.f32x2 d, a, b, c;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y));
  return d;
}
__device__ __forceinline__ float2 fadd2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "add.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float2 fmul2(float2 a, float2 b) {
  float2 d;
  asm("{\n\t.reg .b64 a, b, d;\n\t"
      "mov.b64 a, {%2, %3};\n\tmov.b64 b, {%4, %5};\n\t"
      "mul.rn.f32x2 d, a, b;\n\tmov.b64 {%0, %1}, d;\n\t}"
      : "=f"(d.x), "=f"(d.y)
      : "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y));
  return d;
}
__device__ __forceinline__ float fmax3(float a, float b, float c) {
  float d;
  asm("max.f32 %0, %1, %2, %3;" : "=f"(d) : "f"(a), "f"(b), "f"(c));
  return d;
}
__device__ __forceinline__ float2 u2f2(uint32_t a, uint32_t b) { return make_float2(__uint_as_float(a), __uint_as_float(b)); }
__device__ __forceinline__ uint32_t pack2(float2 v) { return pack_bf16(v.x, v.y); }
__device__ __forceinline__ float2 ex2x2(float2 v) { return make_float2(ex2(v.x), ex2(v.y)); }

// exp2 of a pair on the FMA pipe (no MUFU): x = j + f with j = rint(x) (magic-number
// add), 2^f on [-0.5, 0.5] by a degree-3 polynomial (max relative error 7.7e-5,
// far below the bf16 rounding of P), then j added into the exponent field.
// Inputs are clamped at -126 (2^-126 ~ 1e-38 stands in for 0). The softmax loops
// send a fixed fraction of their exponentials here so the MUFU pipe (16/clk/SM)
// stops being the bound at head_dim 80.
__device__ __forceinline__ float2 ex2x2_poly(float2 x) {
  x.x = fmaxf(x.x, -126.f);
  x.y = fmaxf(x.y, -126.f);
  const float2 t = fadd2(x, make_float2(12582912.f, 12582912.f));        // 1.5 * 2^23 + rint(x)
  const float2 j = fadd2(t, make_float2(-12582912.f, -12582912.f));      // rint(x)
  const float2 f = ffma2(j, make_float2(-1.f, -1.f), x);                 // x - rint(x) in [-0.5, 0.5]
  float2 q = ffma2(make_float2(0.05508868f, 0.05508868f), f, make_float2(0.24260405f, 0.24260405f));
  q = ffma2(q, f, make_float2(0.69327624f, 0.69327624f));
  q = ffma2(q, f, make_float2(0.99992894f, 0.99992894f));
  // low bits of t are rint(x) (two's complement), so t << 23 is rint(x) << 23
  return make_float2(__uint_as_float(__float_as_uint(q.x) + (__float_as_uint(t.x) << 23)),
                     __uint_as_float(__float_as_uint(q.y) + (__float_as_uint(t.y) << 23)));
}
// `poly` is a constant after the softmax loops are unrolled.
__device__ __forceinline__ float2 ex2x2_sel(bool poly, float2 v) { return poly ? ex2x2_poly(v) : ex2x2(v); }
// Which groups of a fully unrolled softmax loop use the FMA-pipe exponential: 3 of 8.
#ifndef SPK_DKV_NS
#define SPK_DKV_NS 3  // hd <= 80 dK/dV: score buffers (the dP^T buffers take the remaining 4 - NS)
#endif
#ifndef SPK_DQ_NS
#define SPK_DQ_NS 3  // hd <= 80 dQ: score / dP buffers (3 + 2: -0.5 % bwd at sustained clocks vs 3 + 1)
#endif
#ifndef SPK_DQ_ND
#define SPK_DQ_ND 2
#endif
#ifndef SPK_POLY_FWD
#define SPK_POLY_FWD 2
#endif
#ifndef SPK_POLY_BWD
#define SPK_POLY_BWD 0
#endif
#ifndef SPK_POLY_DQ
#define SPK_POLY_DQ SPK_POLY_BWD
#endif
// Which 4-element groups of a fully unrolled softmax loop use the FMA-pipe
// exponential: SPK_POLY_* of every 8, spread out.
__host__ __device__ constexpr bool poly_pick(int g, int k) { return (g % 8) * k % 8 + k > 7 || (k >= 8); }
__host__ __device__ constexpr bool poly_group(int g) { return SPK_POLY_FWD > 0 && poly_pick(g, SPK_POLY_FWD); }
__host__ __device__ constexpr bool bwd_poly_group(int g) { return SPK_POLY_BWD > 0 && poly_pick(g, SPK_POLY_BWD); }
__host__ __device__ constexpr bool dq_poly_group(int g) { return SPK_POLY_DQ > 0 && poly_pick(g, SPK_POLY_DQ); }

// Copy this lane's [HD] bf16 row (`src`, or zeros when !valid) into TMEM as an
// MMA A operand: column c of the lane holds elements (2c, 2c+1).
template <int HD>
__device__ __forceinline__ void row_to_tmem(uint32_t taddr, const __nv_bfloat16* src, bool valid) {
  uint32_t v[HD / 2];
#pragma unroll
  for (int c = 0; c < HD / 8; ++c) {
    const uint4 u = valid ? __ldg(reinterpret_cast<const uint4*>(src) + c) : make_uint4(0, 0, 0, 0);
    v[4 * c] = u.x;
    v[4 * c + 1] = u.y;
    v[4 * c + 2] = u.z;
    v[4 * c + 3] = u.w;
  }
#pragma unroll
  for (int c = 0; c < HD / 16; ++c) tc::tmem_st8(taddr + 8 * c, v + 8 * c);
}

// Same for half of the row: elements [0, HD/2) of `src` -> HD/4 columns at taddr.
template <int HD>
__device__ __forceinline__ void row_part_to_tmem(uint32_t taddr, const __nv_bfloat16* src, bool valid) {
  constexpr int NC = HD / 4;  // 32-bit columns (bf16 pairs): 20 (hd 80) / 16 (hd 64) / 32 (hd 128)
  uint32_t v[NC];
#pragma unroll
  for (int c = 0; c < NC / 4; ++c) {
    const uint4 u = valid ? __ldg(reinterpret_cast<const uint4*>(src) + c) : make_uint4(0, 0, 0, 0);
    v[4 * c] = u.x;
    v[4 * c + 1] = u.y;
    v[4 * c + 2] = u.z;
    v[4 * c + 3] = u.w;
  }
#pragma unroll
  for (int c = 0; c + 8 <= NC; c += 8) tc::tmem_st8(taddr + c, v + c);
  if constexpr (NC % 8 == 4) tc::tmem_st4(taddr + NC - 4, v + NC - 4);
}

// Forward CTA = two 128-query tiles (A, B) of one head, ping-ponged so that one
// tile's softmax overlaps the other tile's MMAs. TMEM (512 columns):
//   S_A [0,128) | S_B [128,256) | O_A, Q_A (hd <= 80: Q as TS-MMA A operand) | O_B, Q_B
// hd 128 keeps Q in shared memory (SS form): S_A | S_B | O_A [256,384) | O_B [384,512).
template <int HD>
struct FwdCfg {
  static constexpr bool QT = HD <= 80;
  __host__ __device__ static constexpr uint32_t t_o(int t) { return t ? 384 : 256; }
  __host__ __device__ static constexpr uint32_t t_q(int t) { return t_o(t) + HD; }
  static_assert(!QT || 384 + HD + HD / 2 <= 512, "fwd TMEM budget");
};

template <int HD>
constexpr size_t fwd_smem_n(int st) {
  return (FwdCfg<HD>::QT ? 0 : 2 * Lay<HD>::bytes(128)) + 2 * st * Lay<HD>::bytes(128) + (16 + 4 * st) * 8 + 16 +
         2 * 2 * 2 * 128 * 4 + 1024;  // + softmax row-max / row-sum exchange
}
// Ring depths: as many K / V stages as the opt-in SMEM (227 KB) holds, capped at 6.
template <int HD>
constexpr int fwd_stages() {
  int st = 6;
  while (fwd_smem_n<HD>(st) > 232448) --st;
  return st;
}
template <int HD>
constexpr size_t fwd_smem() {
  return fwd_smem_n<HD>(fwd_stages<HD>());
}

// ============================================================================ forward

template <int HD>
__global__ void __launch_bounds__(640, 1) attn_fwd_tc_k(const __grid_constant__ AttnParams p) {
  using C = FwdCfg<HD>;
  constexpr int KVS = fwd_stages<HD>();
  constexpr int TB = Lay<HD>::bytes(128);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sQ = sm;                          // [2] (hd 128 only)
  uint8_t* sK = sQ + (C::QT ? 0 : 2 * TB);   // [KVS]
  uint8_t* sV = sK + KVS * TB;               // [KVS]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + KVS * TB);
  uint64_t* q_ready = bars;      // Q of both tiles resident (TMEM copy or TMA)
  uint64_t* s_full = bars + 1;   // [2 tiles]
  uint64_t* p_full = bars + 3;   // [2 tiles]  P packed into the tile's S buffer
  uint64_t* pv_done = bars + 5;  // [2 tiles]  O += P V completed
  uint64_t* k_full = bars + 16;          // [KVS]
  uint64_t* k_empty = k_full + KVS;      // [KVS]
  uint64_t* v_full = k_empty + KVS;      // [KVS]
  uint64_t* v_empty = v_full + KVS;      // [KVS]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(v_empty + KVS);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_qb = static_cast<int>((p.n + BQ - 1) / BQ);
  const int npair = (num_qb + 1) / 2;
  const int pair = npair - 1 - static_cast<int>(blockIdx.x);  // heaviest pairs first
  const int head = blockIdx.y;
  int nblk_t[2];
  int64_t q0_t[2];
#pragma unroll
  for (int t = 0; t < 2; ++t) {
    const int qb = 2 * pair + t;
    q0_t[t] = static_cast<int64_t>(qb) * BQ;
    if (qb >= num_qb) {
      nblk_t[t] = 0;
      continue;
    }
    const int64_t q_hi = (q0_t[t] + BQ < p.n ? q0_t[t] + BQ : p.n);
    const int64_t kend = (p.q_off + q_hi < p.kv_len) ? p.q_off + q_hi : p.kv_len;
    nblk_t[t] = static_cast<int>((kend + BKV - 1) / BKV);
  }
  const int nblk = nblk_t[0] > nblk_t[1] ? nblk_t[0] : nblk_t[1];

  if (threadIdx.x == 0) {
    tc::mbar_init(q_ready, C::QT ? 16 : 1);  // softmax warps (TMEM copy) or the TMA
    for (int t = 0; t < 2; ++t) {
      tc::mbar_init(&s_full[t], 1);
      tc::mbar_init(&p_full[t], 8);  // the tile's softmax warps
      tc::mbar_init(&pv_done[t], 1);
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
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform (keeps MMA operands in uniform registers)

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&p.tkv.m0);
      if constexpr (!C::QT) {
        tc::tma_prefetch(&p.tq.m0);
        tc::mbar_expect_tx(q_ready, (nblk_t[1] > 0 ? 2 : 1) * TB);
        for (int t = 0; t < 2; ++t)
          if (nblk_t[t] > 0) load_tile<HD>(sQ + t * TB, p.tq, q_ready, head * HD, static_cast<int>(q0_t[t]), 128, 0);
      }
      // K runs one block ahead of V: K_{j+1} (freed after S(j+1-KVS)) is
      // requested before V_j (freed after PV(j-KVS)), so PV never starves S.
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
    // S-issuing warp (converged; tc::*_w elect the issuing lane): S_t(j) = Q_t K_j^T
    // once K_j landed and PV_t(j-1) (which read P_t(j-1) from the same buffer)
    // completed.
    constexpr uint32_t idesc_s = tc::idesc_bf16(128, BKV, false, false);
    tc::mbar_wait_w(q_ready, 0);
    tc::tc_fence_after();
    for (int j = 0; j < nblk; ++j) {
      const int st = j % KVS;
      tc::mbar_wait_w(&k_full[st], (j / KVS) & 1);
      const uint32_t k_base = tc::smem_u32(sK + st * TB);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (j >= nblk_t[t]) continue;
        if (j > 0) tc::mbar_wait_w(&pv_done[t], (j - 1) & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk) {
          if constexpr (C::QT)
            tc::mma_bf16_ts_w(tmem + t * 128, tmem + C::t_q(t) + 8 * kk, kdesc<HD>(k_base, 128, kk), idesc_s, kk > 0);
          else
            tc::mma_bf16_ss_w(tmem + t * 128, kdesc<HD>(tc::smem_u32(sQ + t * TB), 128, kk), kdesc<HD>(k_base, 128, kk),
                              idesc_s, kk > 0);
        }
        tc::mma_commit_w(&s_full[t]);
      }
      tc::mma_commit_w(&k_empty[st]);
    }
  } else if (warp == 2) {
    // PV-issuing warp: O_t += P_t(j) V_j (A = P from TMEM) once P_t(j) is packed.
    for (int j = 0; j < nblk; ++j) {
      const int st = j % KVS;
      tc::mbar_wait_w(&v_full[st], (j / KVS) & 1);
      const uint32_t v_base = tc::smem_u32(sV + st * TB);
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        if (j >= nblk_t[t]) continue;
        tc::mbar_wait_w(&p_full[t], j & 1);
        tc::tc_fence_after();
#pragma unroll
        for (int kk = 0; kk < BKV / 16; ++kk)  // P of keys [64hf, 64hf+64) is packed at columns [64hf, 64hf+32)
          mma_nhd_ts<HD>(tmem + C::t_o(t), tmem + t * 128 + 64 * (kk >> 2) + 8 * (kk & 3), v_base, 128, kk,
                         j > 0 || kk > 0);
        tc::mma_commit_w(&pv_done[t]);
      }
      tc::mma_commit_w(&v_empty[st]);
    }
  } else if (warp >= 4) {
    // 16 softmax warps: tile t = (w-4)/8, column half hf = ((w-4)/4)&1, TMEM lane
    // quarter w%4 (one query row per lane). The two warps of a (tile, quarter)
    // share their rows: each takes 64 of the block's 128 key columns, they swap
    // row maxima through shared memory (one 64-thread named barrier per block)
    // and keep partial row sums that are combined once at the end.
    const int sw = warp - 4, t = sw >> 3, hf = (sw >> 2) & 1, quarter = warp & 3;
    const int r = quarter * 32 + lane;
    const int64_t row = q0_t[t] + r;
    const bool valid = nblk_t[t] > 0 && row < p.n;
    const int64_t qpos = p.q_off + row;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    const uint32_t obase = tmem + lane_base + C::t_o(t);
    const int nb = nblk_t[t];
    const int bar_id = 1 + t * 4 + quarter;  // named barrier of this row group's two warps
    float* xch = reinterpret_cast<float*>(tmem_slot + 4);  // [2 parity][2 tiles][2 halves][128 rows]
    if constexpr (C::QT) {  // each half copies half of this lane's Q row
      row_part_to_tmem<HD>(tmem + lane_base + C::t_q(t) + hf * (HD / 4),
                           p.q + (valid ? row : 0) * p.h + head * HD + hf * (HD / 2), valid);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      warp_arrive(q_ready);
    }
    constexpr int NCH = HD / 16, SPLIT = (NCH + 1) / 2;  // O column chunks owned by half 0 / half 1
    const int c_begin = hf ? SPLIT : 0, c_end = hf ? NCH : SPLIT;
    constexpr float kRescale = 8.f;
    float m = -INFINITY, l = 0.f;

    for (int j = 0; j < nb; ++j) {
      const int64_t lim64 =
          (valid ? (qpos < p.kv_len - 1 ? qpos : p.kv_len - 1) : -1) - static_cast<int64_t>(j) * BKV - 64 * hf;
      const int lim = lim64 > 1000000 ? 1000000 : static_cast<int>(lim64);  // local columns <= lim are visible
      tc::mbar_wait(&s_full[t], j & 1);
      tc::tc_fence_after();
      const uint32_t sbase = tmem + lane_base + t * 128 + 64 * hf;
      uint32_t sv[64];
      tc::tmem_ld32(sbase, *reinterpret_cast<uint32_t(*)[32]>(&sv[0]));
      tc::tmem_ld32(sbase + 32, *reinterpret_cast<uint32_t(*)[32]>(&sv[32]));
      tc::tmem_ld_wait();
      if (!__all_sync(0xffffffffu, lim >= 63)) {
#pragma unroll
        for (int c = 0; c < 64; ++c)
          if (c > lim) sv[c] = __float_as_uint(-INFINITY);
      }
      float mx;
      {
        float m0 = -INFINITY, m1 = -INFINITY, m2 = -INFINITY, m3 = -INFINITY;
#pragma unroll
        for (int c = 0; c < 64; c += 8) {
          m0 = fmax3(m0, __uint_as_float(sv[c]), __uint_as_float(sv[c + 1]));
          m1 = fmax3(m1, __uint_as_float(sv[c + 2]), __uint_as_float(sv[c + 3]));
          m2 = fmax3(m2, __uint_as_float(sv[c + 4]), __uint_as_float(sv[c + 5]));
          m3 = fmax3(m3, __uint_as_float(sv[c + 6]), __uint_as_float(sv[c + 7]));
        }
        mx = fmax3(m0, m1, fmaxf(m2, m3));
      }
      {  // row max over both halves (parity-buffered slots: one barrier per block)
        float* slot = xch + (((j & 1) * 2 + t) * 2) * 128;
        sts_f32(slot + hf * 128 + r, mx);
        tc::named_bar_sync(bar_id, 64);
        mx = fmaxf(mx, lds_f32(slot + (hf ^ 1) * 128 + r));
      }
      mx *= p.scale_log2;
      const bool need = (m == -INFINITY) ? (mx > -INFINITY || j == 0) : (mx > m + kRescale);
      if (__any_sync(0xffffffffu, need)) {
        const float m_new = need ? fmaxf(m, mx) : m;
        const float alpha = (m == -INFINITY) ? 0.f : exp2f(m - m_new);
        if (j > 0) {  // rescale this half's O columns (PV_t(j-1) must have landed)
          // pv_done[t] cannot be past phase j-1 here: PV_t(j) needs this P_t(j).
          tc::mbar_wait(&pv_done[t], (j - 1) & 1);
          tc::tc_fence_after();
          for (int c = c_begin; c < c_end; ++c) {
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
      const float2 sc2 = make_float2(p.scale_log2, p.scale_log2), nm2 = make_float2(neg_m, neg_m);
      float2 rs_a = make_float2(0.f, 0.f), rs_b = make_float2(0.f, 0.f);
#pragma unroll
      for (int c = 0; c < 2; ++c) {
        uint32_t w[16];
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const bool poly = poly_group(c * 8 + e / 4);
          const float2 x0 = ex2x2_sel(poly, ffma2(u2f2(sv[c * 32 + e], sv[c * 32 + e + 1]), sc2, nm2));
          const float2 x1 = ex2x2_sel(poly, ffma2(u2f2(sv[c * 32 + e + 2], sv[c * 32 + e + 3]), sc2, nm2));
          rs_a = fadd2(rs_a, x0);
          rs_b = fadd2(rs_b, x1);
          w[e / 2] = pack2(x0);
          w[e / 2 + 1] = pack2(x1);
        }
        tc::tmem_st16(sbase + c * 16, w);  // P keys [64hf + 32c, +32) -> columns [64hf + 16c, +16)
      }
      l += (rs_a.x + rs_a.y) + (rs_b.x + rs_b.y);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      warp_arrive(&p_full[t]);
    }
    if (nb > 0) {
      {  // combine the two halves' partial row sums
        float* slot = xch + (((nb & 1) * 2 + t) * 2) * 128;
        sts_f32(slot + hf * 128 + r, l);
        tc::named_bar_sync(bar_id, 64);
        l += lds_f32(slot + (hf ^ 1) * 128 + r);
      }
      tc::mbar_wait(&pv_done[t], (nb - 1) & 1);  // last PV_t landed
      tc::tc_fence_after();
      const float inv = l > 0.f ? 1.f / l : 0.f;
      __nv_bfloat16* orow = p.o + (valid ? row : 0) * p.h + head * HD;
      for (int c = c_begin; c < c_end; ++c) {
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
      if (valid && hf == 0) p.lse[static_cast<int64_t>(head) * p.n + row] = (m + log2f(l)) * 0.69314718055994531f;
    }
  }
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// ============================================================================ backward

// Profiling hooks (skip MMAs / softmax, cycle-stamp one CTA) exist only in builds made with
// -DSPK_ATTN_PROFILING=1 (tools/); release builds compile them out and read no environment.
#ifndef SPK_ATTN_PROFILING
#define SPK_ATTN_PROFILING 0
#endif

struct __align__(64) AttnBwdParams {
  CUtensorMap tdkv;  // dkv fp32 [kv_len, 2h], [128 x HD] boxes (TMA reduce-add of dK / dV)
  CUtensorMap tdkv32;  // the same tensor, [128 x 32] boxes, 128-byte swizzle (swizzled dK/dV staging)
  CUtensorMap tdkv16;  // [128 x 16] boxes, 64-byte swizzle (the last 16 columns of head dim 80)
  Maps tq;           // q  [n, h]
  Maps tdo;          // dO [n, h]
  Maps tkv;          // kv [kv_len, 2h]
  const __nv_bfloat16 *q, *dout, *kv;  // raw rows (copied into TMEM as constant MMA operands)
  const float* ld;   // [H][n_pad / 64][-LSE*log2e x 64, -delta x 64], zero padded (attn_prep_k)
  int64_t n_pad;     // n rounded up to 128
  float* dkv;        // [kv_len, 2h] fp32 accumulator
  int dkv_store;     // dK/dV epilogue writes (TMA store) instead of adding (first op of a micro-batch)
  __nv_bfloat16* dq; // [n, h]
  int64_t n, q_off, kv_len;
  int H, h;
  float scale, scale_log2;
  int dbg;  // profiling builds only (SPK_ATTN_PROFILING): 1 = skip dK/dV MMAs, 2 = skip the dK/dV softmax
  unsigned long long* trace;  // profiling builds only: cycle stamps of one CTA, [event][iteration]
};

// ---------------------------------------------------------------- backward layout
// dK/dV kernel (CTA = 128 keys, loops over 64-query blocks) and dQ kernel
// (CTA = 128 queries, loops over 64-key blocks). In both, the operand that is
// constant for the CTA (K and V, resp. Q and dO) is copied once into TMEM and
// used as the A operand of the S / dP MMAs (128x64x16 "TS" MMAs run at the
// tensor floor, 32 cycles; the SS form reads A and B from shared memory and is
// bound at 48 cycles by the 128 B/cycle SMEM port). TMEM (512 columns):
//   S[NS] x 64 | dP[ND] x 64 | accumulators | constant operands (bf16 pairs).
// P / dS are packed (bf16) back into the score buffer they came from; the dP
// buffer is released as soon as the softmax warps have loaded it.
template <int HD>
struct DkvCfg {
  static constexpr bool KVT = HD <= 80;  // K, V in TMEM (hd 128: no room; SS form)
  static constexpr int NS = KVT ? SPK_DKV_NS : 2, ND = KVT ? 4 - SPK_DKV_NS : 2;
  static constexpr uint32_t T_DP = NS * 64, T_DV = T_DP + ND * 64;
  static constexpr uint32_t T_DK = T_DV + (HD == 80 ? 96 : HD);
  static constexpr uint32_t T_K = T_DK + HD, T_V = T_K + HD / 2;
  static_assert((KVT ? T_V + HD / 2 : T_DK + HD) <= 512, "dK/dV TMEM budget");
};
template <int HD>
struct DqCfg {
  static constexpr int NS = HD == 128 ? 2 : SPK_DQ_NS, ND = HD == 128 ? 2 : SPK_DQ_ND;
  static constexpr uint32_t T_DP = NS * 64, T_DQ = T_DP + ND * 64;
  static constexpr uint32_t T_Q = T_DQ + (HD == 80 ? 96 : HD), T_DO = T_Q + HD / 2;
  static_assert(T_DO + HD / 2 <= 512, "dQ TMEM budget");
};

template <int HD>
constexpr size_t dkv_smem_n(int st) {
  return (DkvCfg<HD>::KVT ? 0 : 2 * Lay<HD>::bytes(128)) + 2 * st * Lay<HD>::bytes(64) + st * 512 + (20 + 2 * st) * 8 +
         8 + 1024;
}
#ifndef SPK_DKV_QST_MAX
#define SPK_DKV_QST_MAX 8
#endif
template <int HD>
constexpr int dkv_stages() {
  int st = SPK_DKV_QST_MAX;
  while (dkv_smem_n<HD>(st) > 232448) --st;
  return st;
}
template <int HD>
constexpr size_t dkv_smem() {
  return dkv_smem_n<HD>(dkv_stages<HD>());
}
template <int HD>
constexpr size_t dq_smem_n(int st) {
  return 2 * st * Lay<HD>::bytes(64) + (20 + 2 * st) * 8 + 8 + 1024;
}
__device__ __forceinline__ int prof_dbg(const AttnBwdParams& p) { return SPK_ATTN_PROFILING ? p.dbg : 0; }

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

// Debug timeline (SP_ATTN_TRACE=1): clock64 stamps of the last CTA of head 0,
// 16 events x 64 iterations; printed by the host after the launch.
__device__ __forceinline__ void trace_mark(const AttnBwdParams& p, int ev, int it) {
  if constexpr (!SPK_ATTN_PROFILING) return;
  // every lane stores the same stamp: no lane-divergent branch in the MMA warp
  if (p.trace && it < 64 && blockIdx.x == gridDim.x - 1 && blockIdx.y == 0) p.trace[ev * 64 + it] = clock64();
}

// dK/dV: one CTA per (128-key block, head), looping over 64-query blocks that
// can see those keys: S^T = K Q_i^T and dP^T = V dO_i^T into TMEM; the softmax
// warps form P^T = exp2(S^T*c - LSE) and dS^T = P^T (dP^T - delta) and pack
// both (bf16) into the S^T buffer they came from (P^T in the first, dS^T in the
// second 16 columns of each 32-column half); dV += P^T dO_i and dK += dS^T Q_i
// take A from TMEM and accumulate in TMEM. Each (key row, head) slice of the
// fp32 dKV accumulator has exactly one owner CTA.
template <int HD>
__global__ void __launch_bounds__(640, 1) attn_bwd_dkv_k(const __grid_constant__ AttnBwdParams p) {
  using C = DkvCfg<HD>;
  constexpr int QST = dkv_stages<HD>();
  constexpr int NS = C::NS, ND = C::ND;
  constexpr int KV_T = C::KVT ? 0 : Lay<HD>::bytes(128), Q_T = Lay<HD>::bytes(64);
  static_assert(2 * 128 * HD * 4 <= 2 * KV_T + QST * (2 * Q_T + 512), "dK/dV epilogue staging must fit the ring");
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;                 // (hd 128 only)
  uint8_t* sV = sK + KV_T;
  uint8_t* sQ = sV + KV_T;          // [QST]
  uint8_t* sdO = sQ + QST * Q_T;    // [QST]
  float* sLD = reinterpret_cast<float*>(sdO + QST * Q_T);  // [QST][-LSE*log2e x 64, -delta x 64]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sLD + QST * 128);
  uint64_t* kv_full = bars;       // K/V resident (SMEM tiles, or TMEM copy)
  uint64_t* done = bars + 1;
  uint64_t* s_full = bars + 2;    // [NS]  S^T_i landed
  uint64_t* sm_done = bars + 5;   // [NS]  P^T_i and dS^T_i packed into S buffer i % NS
  uint64_t* dp_full = bars + 8;   // [ND]  dP^T_i landed
  uint64_t* dp_free = bars + 10;  // [ND]  dP^T_i loaded into registers (buffer reusable)
  uint64_t* q_full = bars + 12;          // [QST]
  uint64_t* q_empty = q_full + QST;      // [QST]
  uint64_t* s_free = q_empty + QST;      // [NS]  dV/dK_i completed: score buffer i % NS reusable
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_free + NS);

  // 2-CTA cluster: CTAs own adjacent 128-key blocks and stream the same query
  // blocks; each Q_i / dO_i tile is fetched once from L2 and multicast to both
  // (rank 0 issues Q, rank 1 issues dO).
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const uint32_t rank = tc::cluster_ctarank();
  const int num_kb = static_cast<int>((p.kv_len + 127) / 128);
  const int num_kb2 = (num_kb + 1) & ~1;
  const int kb = num_kb2 - 1 - static_cast<int>(blockIdx.x);  // may be == num_kb (idle keys)
  const int head = blockIdx.y;
  const int64_t j0 = static_cast<int64_t>(kb) * 128;
  const int64_t j0_lo = static_cast<int64_t>(num_kb2 - 2 - 2 * static_cast<int>(blockIdx.x / 2)) * 128;
  int64_t ib0 = j0_lo - p.q_off;  // first query block any key of the pair can see (common to the cluster)
  if (ib0 < 0) ib0 = 0;
  ib0 = ib0 / 64 * 64;
  const int niter = static_cast<int>((p.n - ib0 + 63) / 64);

  if (threadIdx.x == 0) {
    tc::mbar_init(kv_full, C::KVT ? 16 : 1);  // softmax warps (TMEM copy) or the TMA
    tc::mbar_init(done, 1);
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&sm_done[i], 16);
    }
    for (int i = 0; i < ND; ++i) {
      tc::mbar_init(&dp_full[i], 1);
      tc::mbar_init(&dp_free[i], 16);
    }
    for (int i = 0; i < QST; ++i) {
      tc::mbar_init(&q_full[i], 1);
      tc::mbar_init(&q_empty[i], 2);  // freed by both CTAs' MMA commits
    }
    for (int i = 0; i < NS; ++i) tc::mbar_init(&s_free[i], 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  tc::cluster_sync();
  tc::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform (keeps MMA operands in uniform registers)

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&p.tq.m0);
      tc::tma_prefetch(&p.tdo.m0);
      if constexpr (!C::KVT) {
        tc::tma_prefetch(&p.tkv.m0);
        tc::mbar_expect_tx(kv_full, 2 * Lay<HD>::bytes(128));
        load_tile<HD>(sK, p.tkv, kv_full, head * HD, static_cast<int>(j0), 128, 0);
        load_tile<HD>(sV, p.tkv, kv_full, p.h + head * HD, static_cast<int>(j0), 128, 0);
      }
      for (int it = 0; it < niter; ++it) {
        const int st = it % QST;
        const int64_t i0 = ib0 + static_cast<int64_t>(it) * 64;
        tc::mbar_wait(&q_empty[st], ((it / QST) & 1) ^ 1);  // stage free in both CTAs
        trace_mark(p, 0, it);
        tc::mbar_expect_tx(&q_full[st], 2 * Q_T + 512);
        if (rank == 0)
          load_tile<HD>(sQ + st * Q_T, p.tq, &q_full[st], head * HD, static_cast<int>(i0), 64, 3);
        else
          load_tile<HD>(sdO + st * Q_T, p.tdo, &q_full[st], head * HD, static_cast<int>(i0), 64, 3);
        // (-LSE*log2e, -delta) of the 64 queries: one async 512-byte bulk copy
        tc::bulk_load(sLD + st * 128, p.ld + (static_cast<int64_t>(head) * p.n_pad + i0) * 2, 512, &q_full[st]);
      }
    }
  } else if (warp >= 1 && warp <= 3) {
    // Three MMA-issuing warps (whole warp converged; tc::*_w elect the issuing
    // lane): warp 1 dP^T, warp 2 dV/dK, warp 3 S^T. A tcgen05.mma issue returns
    // only about when the tensor pipe takes it, so every cycle an issuing warp
    // spends on a barrier wait or commit is a pipe bubble unless another warp
    // has MMAs ready; S^T reuse of a score buffer waits for dV/dK of the block
    // that read it (s_free).
    constexpr uint32_t idesc_s = tc::idesc_bf16(128, 64, false, false);
    tc::mbar_wait_w(kv_full, 0);
    tc::tc_fence_after();
    const uint32_t k_base = tc::smem_u32(sK), v_base = tc::smem_u32(sV);
    // S^T = K Q^T / dP^T = V dO^T: A = K / V (TMEM copy, or SMEM tile for hd 128).
    auto kv_mma = [&](uint32_t d, uint32_t t_a, uint32_t a_base, uint32_t b_base) {
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk) {
        if constexpr (C::KVT)
          tc::mma_bf16_ts_w(d, tmem + t_a + 8 * kk, kdesc<HD>(b_base, 64, kk), idesc_s, kk > 0);
        else
          tc::mma_bf16_ss_w(d, kdesc<HD>(a_base, 128, kk), kdesc<HD>(b_base, 64, kk), idesc_s, kk > 0);
      }
    };
    auto issue_s = [&](int it) {  // S^T_it into score buffer it % NS
      const int st = it % QST;
      tc::mbar_wait_w(&q_full[st], (it / QST) & 1);
      tc::tc_fence_after();
      if (!(prof_dbg(p) & 1)) kv_mma(tmem + (it % NS) * 64, C::T_K, k_base, tc::smem_u32(sQ + st * Q_T));
      tc::mma_commit_w(&s_full[it % NS]);
      trace_mark(p, 3, it);
    };
    if (warp == 1) {
      // dP^T issuer: dP^T_it as soon as the softmax has loaded dP^T_{it-ND} (its
      // buffer) -- the dP path is the one the softmax waits on, so it gets a warp
      // of its own with a single wait per block.
      for (int it = 0; it < niter; ++it) {
        const int st = it % QST;
        tc::mbar_wait_w(&q_full[st], (it / QST) & 1);
        if (it >= ND) tc::mbar_wait_w(&dp_free[it % ND], ((it / ND) - 1) & 1);
        tc::tc_fence_after();
        if (!(prof_dbg(p) & 1)) kv_mma(tmem + C::T_DP + (it % ND) * 64, C::T_V, v_base, tc::smem_u32(sdO + st * Q_T));
        tc::mma_commit_w(&dp_full[it % ND]);
        trace_mark(p, 2, it);
      }
    } else if (warp == 3) {
      for (int it = 0; it < niter; ++it) {
        if (it >= NS) tc::mbar_wait_w(&s_free[it % NS], ((it / NS) - 1) & 1);
        issue_s(it);
      }
    } else {
      for (int it = 0; it < niter; ++it) {
        const int b = it % NS, st = it % QST;
        tc::mbar_wait_w(&sm_done[b], (it / NS) & 1);
        tc::tc_fence_after();
        const uint32_t q_base = tc::smem_u32(sQ + st * Q_T), do_base = tc::smem_u32(sdO + st * Q_T);
        if (!(prof_dbg(p) & 1)) {
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {  // K = 64 queries
            const bool acc = it > 0 || kk > 0;
            const uint32_t col = b * 64 + 16 * kk;  // softmax group kk packed P^T | dS^T here
            mma_nhd_ts<HD>(tmem + C::T_DV, tmem + col, do_base, 64, kk, acc);
            mma_nhd_ts<HD>(tmem + C::T_DK, tmem + col + 8, q_base, 64, kk, acc);
          }
        }
        tc::mma_commit_mc_w(&q_empty[st], 3);  // this CTA is done with the multicast stage
        tc::mma_commit_w(&s_free[b]);
        trace_mark(p, 1, it);
      }
      tc::mma_commit_w(done);
    }
  } else if (warp >= 4) {
    // 16 softmax warps: warp w reads TMEM lane quarter w%4 (one key row per
    // lane) and query columns [16g, 16g+16) of each 64-query block, g = (w-4)/4:
    // four warps per SMSP hide the TMEM-load / MUFU / barrier latencies.
    const int quarter = warp & 3, g = (warp - 4) >> 2;
    const int r = quarter * 32 + lane;  // key row
    const int64_t kpos = j0 + r;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    if constexpr (C::KVT) {  // groups 0/1 copy halves of this lane's K row, groups 2/3 of its V row
      const bool kv_ok = kpos < p.kv_len;
      const int part = g & 1;
      row_part_to_tmem<HD>(tmem + lane_base + (g >= 2 ? C::T_V : C::T_K) + part * (HD / 4),
                           p.kv + (kv_ok ? kpos : 0) * 2 * p.h + (g >= 2 ? p.h : 0) + head * HD + part * (HD / 2),
                           kv_ok);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      warp_arrive(kv_full);
    }
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    // Per-iteration bookkeeping as running counters: ring / buffer indices and mbarrier
    // parities advance without div / mod, and the causal-mask bounds are int32 values
    // stepped by 64 (the 64-bit per-iteration index math was ~2 instructions per score).
    // Visible query columns c (local) of block it: c >= cmin, c < chi, where
    // cmin = kpos - q_off - (ib0 + 64 it + 16g) and chi = n - (ib0 + 64 it + 16g).
    int b = 0, st = 0, d = 0;
    uint32_t ph_b = 0, ph_st = 0, ph_d = 0;
    int cmin = clamp_i32(kpos - p.q_off - ib0 - g * 16);
    int cmin_w = clamp_i32(j0 + quarter * 32 + 31 - p.q_off - ib0 - g * 16);  // the warp's largest cmin
    int chi = clamp_i32(p.n - ib0 - g * 16);
    auto advance = [&] {
      cmin -= 64;
      cmin_w -= 64;
      chi -= 64;
      if (++b == NS) b = 0, ph_b ^= 1;
      if (++st == QST) st = 0, ph_st ^= 1;
      if (++d == ND) d = 0, ph_d ^= 1;
    };
    for (int it = 0; it < niter; ++it, advance()) {
      const float* nl = sLD + st * 128 + g * 16;  // -LSE*log2e of this group's 16 queries
      const float* nd = nl + 64;                  // -delta of the same queries
      const int c_lo = cmin < 0 ? 0 : (cmin > 16 ? 16 : cmin);
      const int c_hi = chi < 0 ? 0 : (chi > 16 ? 16 : chi);  // exclusive
      const bool full_blk = cmin_w <= 0 && chi >= 16;        // warp-uniform
      tc::mbar_wait(&q_full[st], ph_st);  // LSE / delta of this block are in SMEM
      if (warp == 4) trace_mark(p, 4, it);
      uint32_t sv[16], dpv[16];
      tc::mbar_wait(&s_full[b], ph_b);
      if (warp == 4) trace_mark(p, 5, it);
      if (prof_dbg(p) & 2) {  // protocol only
        tc::mbar_wait(&dp_full[d], ph_d);
        __syncwarp();
        if (lane == 0) tc::mbar_arrive(&dp_free[d]);
        warp_arrive(&sm_done[b]);
        continue;
      }
      tc::tc_fence_after();
      tmem_ld16(tmem + lane_base + b * 64 + g * 16, sv);
      tc::mbar_wait(&dp_full[d], ph_d);
      if (warp == 4) trace_mark(p, 6, it);
      tc::tc_fence_after();
      tmem_ld16(tmem + lane_base + C::T_DP + d * 64 + g * 16, dpv);
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dp_free[d]);  // the next dP MMA may overwrite the buffer
      uint32_t wp[8], wd[8];
      // P^T = exp2(S^T*c - LSE), dS^T = P^T (dP^T - delta): packed FFMA2 / FADD2 / FMUL2;
      // the mask is only evaluated on blocks that touch the diagonal or the end.
      auto body = [&](auto masked) {
#pragma unroll
        for (int e = 0; e < 16; e += 4) {
          const float4 l4 = lds_f4(nl + e), d4 = lds_f4(nd + e);  // warp broadcast
          const bool poly = bwd_poly_group(2 * (e / 4));
          float2 p0 = ex2x2_sel(poly, ffma2(u2f2(sv[e], sv[e + 1]), sc2, make_float2(l4.x, l4.y)));
          float2 p1 = ex2x2_sel(poly, ffma2(u2f2(sv[e + 2], sv[e + 3]), sc2, make_float2(l4.z, l4.w)));
          if constexpr (decltype(masked)::value) {
            if (e < c_lo || e >= c_hi) p0.x = 0.f;
            if (e + 1 < c_lo || e + 1 >= c_hi) p0.y = 0.f;
            if (e + 2 < c_lo || e + 2 >= c_hi) p1.x = 0.f;
            if (e + 3 < c_lo || e + 3 >= c_hi) p1.y = 0.f;
          }
          const float2 g0 = fmul2(p0, fadd2(u2f2(dpv[e], dpv[e + 1]), make_float2(d4.x, d4.y)));
          const float2 g1 = fmul2(p1, fadd2(u2f2(dpv[e + 2], dpv[e + 3]), make_float2(d4.z, d4.w)));
          wp[e / 2] = pack2(p0);
          wp[e / 2 + 1] = pack2(p1);
          wd[e / 2] = pack2(g0);
          wd[e / 2 + 1] = pack2(g1);
        }
      };
      if (full_blk)
        body(std::false_type{});
      else
        body(std::true_type{});
      tc::tmem_st8(tmem + lane_base + b * 64 + g * 16, wp);      // P^T  -> columns [16g, 16g+8)
      tc::tmem_st8(tmem + lane_base + b * 64 + g * 16 + 8, wd);  // dS^T -> columns [16g+8, 16g+16)
      tc::tmem_st_wait();
      tc::tc_fence_before();
      warp_arrive(&sm_done[b]);
      if (warp == 4) trace_mark(p, 7, it);
    }
    tc::mbar_wait(done, 0);
    tc::tc_fence_after();
    if (warp == 4) trace_mark(p, 8, 0);
    // Epilogue: dK (scaled) / dV rows -> SMEM [2][128][HD] fp32 (the Q/dO ring is
    // idle: every MMA completed and every multicast stage was consumed), then one
    // thread adds both tiles into the fp32 accumulator with TMA reduce-add
    // (coalesced, asynchronous in L2; rows >= kv_len are clipped by the map).
    float* out = reinterpret_cast<float*>(sm);
    constexpr int NCH = HD / 16;
    for (int t = g; t < 2 * NCH; t += 4) {  // 16-column chunks of dV (t < NCH) then dK
      const bool is_k = t >= NCH;
      const int c = is_k ? t - NCH : t;
      uint32_t v[16];
      tmem_ld16(tmem + lane_base + (is_k ? C::T_DK : C::T_DV) + c * 16, v);
      tc::tmem_ld_wait();
      const float sc = is_k ? p.scale : 1.f;
      // staging = the reduce boxes: 32-column [128 x 128 B] tiles (128-byte swizzle) and,
      // for head dim 80, a 16-column [128 x 64 B] tile (64-byte swizzle): the per-row
      // float4 stores are bank-conflict free (a dense [128 x HD] tile is 16-way).
      uint8_t* tile = reinterpret_cast<uint8_t*>(out + (is_k ? 0 : 128 * HD));
#pragma unroll
      for (int e = 0; e < 16; e += 4) {
        uint8_t* dst;
        if (c < 2 * (HD / 32)) {
          const int u = (c & 1) * 4 + e / 4;
          dst = tile + (c >> 1) * 16384 + r * 128 + ((u ^ (r & 7)) << 4);
        } else {
          const int u = e / 4;
          dst = tile + (HD / 32) * 16384 + r * 64 + ((u ^ ((r >> 1) & 3)) << 4);
        }
        *reinterpret_cast<float4*>(dst) =
            make_float4(__uint_as_float(v[e]) * sc, __uint_as_float(v[e + 1]) * sc, __uint_as_float(v[e + 2]) * sc,
                        __uint_as_float(v[e + 3]) * sc);
      }
    }
    tc::fence_proxy_async_smem();
    tc::named_bar_sync(1, 512);
    if (warp == 4 && lane == 0) {
#pragma unroll
      for (int is_v = 0; is_v < 2; ++is_v) {
        const float* tile = out + is_v * 128 * HD;
        const int col = (is_v ? p.h : 0) + head * HD;
#pragma unroll
        for (int b = 0; b < HD / 32; ++b) {
          if (p.dkv_store)
            tc::tma_store_2d(&p.tdkv32, tile + b * 4096, col + 32 * b, static_cast<int>(j0));
          else
            tc::tma_reduce_add_2d(&p.tdkv32, tile + b * 4096, col + 32 * b, static_cast<int>(j0));
        }
        if constexpr (HD % 32 == 16) {
          if (p.dkv_store)
            tc::tma_store_2d(&p.tdkv16, tile + (HD / 32) * 4096, col + HD - 16, static_cast<int>(j0));
          else
            tc::tma_reduce_add_2d(&p.tdkv16, tile + (HD / 32) * 4096, col + HD - 16, static_cast<int>(j0));
        }
      }
      tc::bulk_commit();
      tc::bulk_wait_read0();  // SMEM must outlive the copy-out
    }
    if (warp == 4) trace_mark(p, 9, 0);
  }
  tc::tc_fence_before();
  tc::cluster_sync();  // no multicast data / remote arrive may target an exited CTA
  tc::tc_fence_after();
  if (warp == 1) tc::tmem_dealloc(tmem, 512);
}

// dQ: one CTA per (128-query block, head), looping over 64-key blocks:
// S = Q K_j^T, dP = dO V_j^T (A = Q / dO copied into TMEM once); dS = P (dP -
// delta) is packed (bf16) into the S buffer it came from; dQ += dS K_j with A
// from TMEM.
template <int HD>
__global__ void __launch_bounds__(640, 1) attn_bwd_dq_k(const __grid_constant__ AttnBwdParams p) {
  using C = DqCfg<HD>;
  constexpr int KST = dq_stages<HD>();
  constexpr int NS = C::NS, ND = C::ND;
  constexpr int K_T = Lay<HD>::bytes(64);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sK = sm;               // [KST]
  uint8_t* sV = sK + KST * K_T;   // [KST]
  uint64_t* bars = reinterpret_cast<uint64_t*>(sV + KST * K_T);
  uint64_t* qo_full = bars;       // Q, dO copied into TMEM
  uint64_t* done = bars + 1;
  uint64_t* s_full = bars + 2;    // [NS]
  uint64_t* ds_full = bars + 5;   // [NS]
  uint64_t* dp_full = bars + 8;   // [ND]
  uint64_t* dp_free = bars + 10;  // [ND]
  uint64_t* kv_full = bars + 12;       // [KST]
  uint64_t* kv_empty = kv_full + KST;  // [KST]
  uint64_t* s_free = kv_empty + KST;   // [NS]  dQ_j completed: score buffer j % NS reusable
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_free + NS);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int num_qb = static_cast<int>((p.n + 127) / 128);
  const int qb = num_qb - 1 - static_cast<int>(blockIdx.x);
  const int head = blockIdx.y;
  const int64_t q0 = static_cast<int64_t>(qb) * 128;
  const int64_t q_hi = (q0 + 128 < p.n ? q0 + 128 : p.n);
  const int64_t kend = (p.q_off + q_hi < p.kv_len) ? p.q_off + q_hi : p.kv_len;
  const int nblk = static_cast<int>((kend + 63) / 64);

  if (threadIdx.x == 0) {
    tc::mbar_init(qo_full, 16);
    tc::mbar_init(done, 1);
    for (int i = 0; i < NS; ++i) {
      tc::mbar_init(&s_full[i], 1);
      tc::mbar_init(&ds_full[i], 16);
    }
    for (int i = 0; i < ND; ++i) {
      tc::mbar_init(&dp_full[i], 1);
      tc::mbar_init(&dp_free[i], 16);
    }
    for (int i = 0; i < KST; ++i) {
      tc::mbar_init(&kv_full[i], 1);
      tc::mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < NS; ++i) tc::mbar_init(&s_free[i], 1);
    tc::fence_mbar_init();
  }
  if (warp == 1) tc::tmem_alloc(tmem_slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);  // warp-uniform (keeps MMA operands in uniform registers)

  if (warp == 0) {
    if (lane == 0) {
      tc::tma_prefetch(&p.tkv.m0);
      for (int j = 0; j < nblk; ++j) {
        const int st = j % KST;
        tc::mbar_wait(&kv_empty[st], ((j / KST) & 1) ^ 1);
        tc::mbar_expect_tx(&kv_full[st], 2 * K_T);
        load_tile<HD>(sK + st * K_T, p.tkv, &kv_full[st], head * HD, j * 64, 64, 0);
        load_tile<HD>(sV + st * K_T, p.tkv, &kv_full[st], p.h + head * HD, j * 64, 64, 0);
      }
    }
  } else if (warp >= 1 && warp <= 3) {
    // Three MMA-issuing warps (see the dK/dV kernel): warp 1 dP_j, warp 2
    // dQ += dS_j K_j, warp 3 S_j (after dQ_{j-NS} released its score buffer).
    constexpr uint32_t idesc_s = tc::idesc_bf16(128, 64, false, false);
    tc::mbar_wait_w(qo_full, 0);
    tc::tc_fence_after();
    auto issue_s = [&](int j) {  // S_j into score buffer j % NS
      const int st = j % KST;
      tc::mbar_wait_w(&kv_full[st], (j / KST) & 1);
      tc::tc_fence_after();
      const uint32_t k_base = tc::smem_u32(sK + st * K_T);
#pragma unroll
      for (int kk = 0; kk < HD / 16; ++kk)
        tc::mma_bf16_ts_w(tmem + (j % NS) * 64, tmem + C::T_Q + 8 * kk, kdesc<HD>(k_base, 64, kk), idesc_s, kk > 0);
      tc::mma_commit_w(&s_full[j % NS]);
    };
    if (warp == 1) {  // dP issuer (see the dK/dV kernel)
      for (int j = 0; j < nblk; ++j) {
        const int st = j % KST;
        tc::mbar_wait_w(&kv_full[st], (j / KST) & 1);
        if (j >= ND) tc::mbar_wait_w(&dp_free[j % ND], ((j / ND) - 1) & 1);  // softmax loaded dP_{j-ND}
        tc::tc_fence_after();
        const uint32_t v_base = tc::smem_u32(sV + st * K_T);
#pragma unroll
        for (int kk = 0; kk < HD / 16; ++kk)
          tc::mma_bf16_ts_w(tmem + C::T_DP + (j % ND) * 64, tmem + C::T_DO + 8 * kk, kdesc<HD>(v_base, 64, kk), idesc_s,
                            kk > 0);
        tc::mma_commit_w(&dp_full[j % ND]);
      }
    } else if (warp == 3) {
      for (int j = 0; j < nblk; ++j) {
        if (j >= NS) tc::mbar_wait_w(&s_free[j % NS], ((j / NS) - 1) & 1);
        issue_s(j);
      }
    } else {  // dQ issuer
      for (int j = 0; j < nblk; ++j) {
        const int b = j % NS, st = j % KST;
        tc::mbar_wait_w(&ds_full[b], (j / NS) & 1);
        tc::tc_fence_after();
        const uint32_t k_base = tc::smem_u32(sK + st * K_T);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk)  // K = 64 keys
          mma_nhd_ts<HD>(tmem + C::T_DQ, tmem + b * 64 + 16 * kk, k_base, 64, kk, j > 0 || kk > 0);
        // kv stage j is released after dQ_j AND dP_j (other warp): dP_j completed before
        // the softmax could publish dS_j, so this commit covers every reader of the stage.
        tc::mma_commit_w(&kv_empty[st]);
        tc::mma_commit_w(&s_free[b]);
      }
      tc::mma_commit_w(done);
    }
  } else if (warp >= 4) {
    // 16 softmax warps: warp w reads lane quarter w%4 (one query row per lane)
    // and key columns [16g, 16g+16) of each 64-key block, g = (w-4)/4.
    const int quarter = warp & 3, g = (warp - 4) >> 2;
    const int r = quarter * 32 + lane;
    const int64_t row = q0 + r;
    const bool valid = row < p.n;
    const int64_t qpos = p.q_off + row;
    const uint32_t lane_base = static_cast<uint32_t>(quarter * 32) << 16;
    {  // groups 0/1 copy halves of this lane's Q row into TMEM, groups 2/3 of its dO row
      const int part = g & 1;
      row_part_to_tmem<HD>(tmem + lane_base + (g >= 2 ? C::T_DO : C::T_Q) + part * (HD / 4),
                           (g >= 2 ? p.dout : p.q) + (valid ? row : 0) * p.h + head * HD + part * (HD / 2), valid);
      tc::tmem_st_wait();
      tc::tc_fence_before();
      warp_arrive(qo_full);
    }
    // (-LSE*log2e, -delta) of this query row (zero padded past n): blocks of 64 queries.
    const int64_t ldi = (static_cast<int64_t>(head) * p.n_pad + (row & ~int64_t(63))) * 2 + (row & 63);
    const float2 nl2 = make_float2(p.ld[ldi], p.ld[ldi]), nd2 = make_float2(p.ld[ldi + 64], p.ld[ldi + 64]);
    const float2 sc2 = make_float2(p.scale_log2, p.scale_log2);
    // running counters as in the dK/dV kernel: key columns c (local) with c <= lim are
    // visible, lim = qpos - 64 j - 16g (-1 for rows past n); the warp's smallest lim is
    // that of its first row.
    int b = 0, d = 0;
    uint32_t ph_b = 0, ph_d = 0;
    int lim_r = valid ? clamp_i32(qpos - g * 16) : -(1 << 30);
    const bool warp_valid = q0 + quarter * 32 + 31 < p.n;
    int lim_w = clamp_i32(p.q_off + q0 + quarter * 32 - g * 16);
    for (int j = 0; j < nblk; ++j, lim_r -= 64, lim_w -= 64) {
      const int lim = lim_r < -1 ? -1 : (lim_r > 1000 ? 1000 : lim_r);
      const bool full_blk = warp_valid && lim_w >= 15;  // warp-uniform
      uint32_t sv[16], dpv[16];
      tc::mbar_wait(&s_full[b], ph_b);
      tc::tc_fence_after();
      tmem_ld16(tmem + lane_base + b * 64 + g * 16, sv);
      tc::mbar_wait(&dp_full[d], ph_d);
      tc::tc_fence_after();
      tmem_ld16(tmem + lane_base + C::T_DP + d * 64 + g * 16, dpv);
      tc::tmem_ld_wait();
      tc::tc_fence_before();
      __syncwarp();
      if (lane == 0) tc::mbar_arrive(&dp_free[d]);
      uint32_t w[8];
      auto body = [&](auto masked) {
#pragma unroll
        for (int e = 0; e < 16; e += 2) {
          float2 pr = ex2x2_sel(dq_poly_group(e / 2), ffma2(u2f2(sv[e], sv[e + 1]), sc2, nl2));
          if constexpr (decltype(masked)::value) {
            if (e > lim) pr.x = 0.f;
            if (e + 1 > lim) pr.y = 0.f;
          }
          w[e / 2] = pack2(fmul2(pr, fadd2(u2f2(dpv[e], dpv[e + 1]), nd2)));
        }
      };
      if (full_blk)
        body(std::false_type{});
      else
        body(std::true_type{});
      tc::tmem_st8(tmem + lane_base + b * 64 + g * 16, w);  // dS -> columns [16g, 16g+8) of the S buffer
      tc::tmem_st_wait();
      tc::tc_fence_before();
      warp_arrive(&ds_full[b]);
      if (++b == NS) b = 0, ph_b ^= 1;
      if (++d == ND) d = 0, ph_d ^= 1;
    }
    tc::mbar_wait(done, 0);
    tc::tc_fence_after();
    __nv_bfloat16* dq_row = p.dq + (valid ? row : 0) * p.h + head * HD;
    constexpr int NCH = HD / 16;
    for (int c = g; c < NCH; c += 4) {
      uint32_t v[16];
      tmem_ld16(tmem + lane_base + C::T_DQ + c * 16, v);  // warp-collective: all lanes
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

// ld: per head, blocks of 64 queries laid out as [64 x -LSE*log2e][64 x -delta],
// delta = sum_d dO*O; zeros up to n_pad. One thread per (query, head), heads
// fastest: a warp reads whole 16-byte vectors of one query row (coalesced through
// L1), each thread reduces its own head in registers. The dK/dV kernel
// bulk-copies one 512-byte block per 64-query step.
template <int HD>
__global__ void attn_prep_k(const __nv_bfloat16* __restrict__ o, const __nv_bfloat16* __restrict__ dout,
                            const float* __restrict__ lse, float* __restrict__ ld, int64_t n, int64_t n_pad, int H) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n_pad * H) return;
  const int64_t i = t / H;
  const int head = static_cast<int>(t % H);
  float d = 0.f, l = 0.f;
  if (i < n) {
    const uint4* ov = reinterpret_cast<const uint4*>(o + i * (int64_t)H * HD + head * HD);
    const uint4* dv = reinterpret_cast<const uint4*>(dout + i * (int64_t)H * HD + head * HD);
#pragma unroll
    for (int c = 0; c < HD / 8; ++c) {
      const uint4 a = ov[c], b = dv[c];
      const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&aw[k]));
        const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bw[k]));
        d = fmaf(fa.x, fb.x, d);
        d = fmaf(fa.y, fb.y, d);
      }
    }
    l = lse[(int64_t)head * n + i] * 1.4426950408889634f;
  }
  const int64_t at = (head * n_pad + (i & ~int64_t(63))) * 2 + (i & 63);
  ld[at] = -l;
  ld[at + 64] = -d;
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
  p.q = static_cast<const __nv_bfloat16*>(q);
  p.lse = lse;
  p.n = n;
  p.q_off = q_off;
  p.kv_len = kv_len;
  p.H = H;
  p.h = h;
  p.scale_log2 = 1.4426950408889634f / sqrtf(static_cast<float>(hd));
  auto run = [&](auto hd_tag) {
    constexpr int HD = decltype(hd_tag)::value;
    dim3 grid(static_cast<unsigned>(((n + BQ - 1) / BQ + 1) / 2), static_cast<unsigned>(H));  // query-tile pairs
    constexpr size_t smem = fwd_smem<HD>();
    static_assert(smem <= 232448, "attention fwd smem");
    SPK_CUDA(cudaFuncSetAttribute(attn_fwd_tc_k<HD>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attn_fwd_tc_k<HD><<<grid, 640, smem, s>>>(p);
    SPK_LAUNCH_CHECK();
  };
  switch (hd) {
    case 64: run(std::integral_constant<int, 64>{}); break;
    case 80: run(std::integral_constant<int, 80>{}); break;
    case 128: run(std::integral_constant<int, 128>{}); break;
    default: throw std::invalid_argument("attention tc: head_dim must be 64, 80 or 128");
  }
}

size_t attn_bwd_ws_delta_floats(int64_t n, int H) { return static_cast<size_t>(H) * ((n + 127) / 128 * 128) * 2; }

// Side stream of the calling thread's device for the dQ kernel: it runs concurrently
// with the dK/dV kernel (both only read the prep output and write disjoint results),
// so each fills the other's last-wave tail.
namespace {
struct SideStream {
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
};
SideStream& side_stream() {
  static thread_local SideStream per_dev[16];
  int dev = 0;
  SPK_CUDA(cudaGetDevice(&dev));
  SideStream& ss = per_dev[dev & 15];
  if (!ss.s) {
    SPK_CUDA(cudaStreamCreateWithFlags(&ss.s, cudaStreamNonBlocking));
    SPK_CUDA(cudaEventCreateWithFlags(&ss.fork, cudaEventDisableTiming));
    SPK_CUDA(cudaEventCreateWithFlags(&ss.join, cudaEventDisableTiming));
  }
  return ss;
}
}  // namespace

void attn_bwd_tc(bool dkv_overwrite, const void* q, const void* kv, const void* o, const void* dout, const float* lse, float* ws_delta,
                 float* ws_dq, void* dq, float* dkv, int64_t n, int64_t q_off, int64_t kv_len, int H, int hd,
                 cudaStream_t s) {
  const int h = H * hd;
  if ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(kv) | reinterpret_cast<uintptr_t>(dout) |
       reinterpret_cast<uintptr_t>(o) | reinterpret_cast<uintptr_t>(dq) | reinterpret_cast<uintptr_t>(dkv)) & 15)
    throw std::invalid_argument("attention: operands must be 16-byte aligned");
  const int64_t n_pad = (n + 127) / 128 * 128;  // the dQ kernel reads whole 128-row blocks
  {
    const unsigned blocks = static_cast<unsigned>((n_pad * H + 255) / 256);
    const auto* ob = static_cast<const __nv_bfloat16*>(o);
    const auto* db = static_cast<const __nv_bfloat16*>(dout);
    switch (hd) {
      case 64: attn_prep_k<64><<<blocks, 256, 0, s>>>(ob, db, lse, ws_delta, n, n_pad, H); break;
      case 80: attn_prep_k<80><<<blocks, 256, 0, s>>>(ob, db, lse, ws_delta, n, n_pad, H); break;
      case 128: attn_prep_k<128><<<blocks, 256, 0, s>>>(ob, db, lse, ws_delta, n, n_pad, H); break;
      default: throw std::invalid_argument("attention: unsupported head_dim");
    }
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
  a.dkv_store = dkv_overwrite ? 1 : 0;
  a.dq = static_cast<__nv_bfloat16*>(dq);
  {
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(2 * h), static_cast<cuuint64_t>(kv_len)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(2 * h) * 4};
    cuuint32_t box[2] = {static_cast<cuuint32_t>(hd), 128};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = tma_encode_fn()(&a.tdkv, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dkv, dims, strides, box, estr,
                                 CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                 CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    cuuint32_t box32[2] = {32, 128}, box16[2] = {16, 128};
    if (r == CUDA_SUCCESS)
      r = tma_encode_fn()(&a.tdkv32, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dkv, dims, strides, box32, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r == CUDA_SUCCESS)
      r = tma_encode_fn()(&a.tdkv16, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dkv, dims, strides, box16, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled (dkv) failed: " + std::to_string((int)r));
  }
  a.q = static_cast<const __nv_bfloat16*>(q);
  a.dout = static_cast<const __nv_bfloat16*>(dout);
  a.kv = static_cast<const __nv_bfloat16*>(kv);
  a.n = n;
  a.q_off = q_off;
  a.kv_len = kv_len;
  a.H = H;
  a.h = h;
  a.scale = 1.f / sqrtf(static_cast<float>(hd));
  a.scale_log2 = 1.4426950408889634f * a.scale;
  a.dbg = 0;
  a.trace = nullptr;
#if SPK_ATTN_PROFILING
  a.dbg = [] {
    const char* e = std::getenv("SP_ATTN_DBG");
    return e ? std::atoi(e) : 0;
  }();
  static unsigned long long* trace_buf = [] {
    unsigned long long* t = nullptr;
    if (std::getenv("SP_ATTN_TRACE")) SPK_CUDA(cudaMalloc(&t, 16 * 64 * sizeof(unsigned long long)));
    return t;
  }();
  a.trace = trace_buf;
  if (trace_buf) SPK_CUDA(cudaMemsetAsync(trace_buf, 0, 16 * 64 * sizeof(unsigned long long), s));
#endif
  AttnBwdParams b = a;  // dQ kernel: K/V in 64-row tiles (Q / dO go to TMEM from the raw rows)
  b.trace = nullptr;
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
      lc.blockDim = dim3(640);
      lc.dynamicSmemBytes = smem_dkv;
      lc.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeClusterDimension;
      at[0].val.clusterDim.x = 2;
      at[0].val.clusterDim.y = 1;
      at[0].val.clusterDim.z = 1;
      lc.attrs = at;
      lc.numAttrs = 1;
      static const bool concurrent = [] {
        const char* e = std::getenv("SP_ATTN_BWD_CONCURRENT");  // tuning: 0 = dQ after dK/dV in stream order
        return e ? std::atoi(e) != 0 : true;
      }();
      if (concurrent && !a.trace) {  // dQ first (long CTAs), on the side stream
        SideStream& ss = side_stream();
        SPK_CUDA(cudaEventRecord(ss.fork, s));
        SPK_CUDA(cudaStreamWaitEvent(ss.s, ss.fork, 0));
        dim3 g2c(static_cast<unsigned>((n + 127) / 128), static_cast<unsigned>(H));
        attn_bwd_dq_k<HD><<<g2c, 640, smem_dq, ss.s>>>(b);
        SPK_LAUNCH_CHECK();
        SPK_CUDA(cudaEventRecord(ss.join, ss.s));
        SPK_CUDA(cudaLaunchKernelEx(&lc, attn_bwd_dkv_k<HD>, a));
        SPK_CUDA(cudaStreamWaitEvent(s, ss.join, 0));
        return;
      }
      SPK_CUDA(cudaLaunchKernelEx(&lc, attn_bwd_dkv_k<HD>, a));
#if SPK_ATTN_PROFILING
      if (a.trace) {
        unsigned long long h_t[16 * 64];
        SPK_CUDA(cudaMemcpyAsync(h_t, a.trace, sizeof(h_t), cudaMemcpyDeviceToHost, s));
        SPK_CUDA(cudaStreamSynchronize(s));
        unsigned long long t0 = ~0ULL;
        for (unsigned long long v : h_t)
          if (v && v < t0) t0 = v;
        std::fprintf(stderr, "dkv trace (cycles from first stamp): it q_load g_issue dp_issue s_issue sm_qfull sm_s sm_dp sm_done\n");
        std::fprintf(stderr, "epilogue start %lld end %lld\n", (long long)(h_t[8 * 64] - t0), (long long)(h_t[9 * 64] - t0));
        for (int it = 0; it < 64; ++it) {
          std::fprintf(stderr, "%3d", it);
          for (int e = 0; e < 8; ++e)
            std::fprintf(stderr, " %8lld", h_t[e * 64 + it] ? (long long)(h_t[e * 64 + it] - t0) : -1LL);
          std::fprintf(stderr, "\n");
        }
      }
#endif
    }
    dim3 g2(static_cast<unsigned>((n + 127) / 128), static_cast<unsigned>(H));
    attn_bwd_dq_k<HD><<<g2, 640, smem_dq, s>>>(b);
    SPK_LAUNCH_CHECK();
  };
  switch (hd) {
    case 64: run(std::integral_constant<int, 64>{}); break;
    case 80: run(std::integral_constant<int, 80>{}); break;
    case 128: run(std::integral_constant<int, 128>{}); break;
    default: throw std::invalid_argument("attention tc: head_dim must be 64, 80 or 128");
  }
}

const void* module_anchor_attention_tc() { return reinterpret_cast<const void*>(&attn_fwd_tc_k<64>); }

}  // namespace spk
