#include <cstdlib>
// HBM-bound kernels of the per-stage transformer: embedding, LayerNorm/RMSNorm
// (fwd, recompute, bwd), GeLU/SwiGLU, RoPE, fused cross-entropy, AdamW, init.
// One CTA per row for the row reductions (warp-shuffle + smem reduce), grid
// sized to a multiple of the SM count for the streaming kernels.
#include <cmath>
#include <type_traits>

#include "cuda/common.cuh"
#include "cuda/ops.h"

namespace spk {
namespace {

constexpr int kRowThreads = 256;

int stream_grid(int64_t n, int threads) {
  int64_t blocks = (n + threads - 1) / threads;
  int64_t cap = static_cast<int64_t>(num_sms()) * 8;
  return static_cast<int>(blocks < cap ? (blocks > 0 ? blocks : 1) : cap);
}

// ------------------------------------------------------------------ embedding
template <typename T>
__global__ void embed_fwd_k(const int32_t* __restrict__ tok, const float* __restrict__ E,
                            const float* __restrict__ pos, int64_t pos0, T* __restrict__ x, int64_t n, int h) {
  const int64_t total = n * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / h, c = i % h;
    float v = E[(int64_t)tok[r] * h + c];
    if (pos) v += pos[(pos0 + r) * h + c];
    x[i] = from_f<T>(v);
  }
}

template <typename T>
__global__ void embed_bwd_k(const int32_t* __restrict__ tok, const T* __restrict__ dx, float* __restrict__ dE,
                            float* __restrict__ dpos, int64_t pos0, int64_t n, int h) {
  const int64_t total = n * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / h, c = i % h;
    const float g = to_f(dx[i]);
    atomicAdd(&dE[(int64_t)tok[r] * h + c], g);
    if (dpos) dpos[(pos0 + r) * h + c] += g;  // positions are unique within a launch
  }
}

// ------------------------------------------------------------------ norms
template <typename T, bool RMS>
__global__ void norm_fwd_k(const T* __restrict__ x, const float* __restrict__ g, T* __restrict__ y,
                           float* __restrict__ mean_out, float* __restrict__ rstd_out, int h, float eps) {
  __shared__ float scratch[32];
  const int64_t row = blockIdx.x;
  const T* xr = x + row * h;
  float mean = 0.f;
  if (!RMS) {
    float s = 0.f;
    for (int c = threadIdx.x; c < h; c += blockDim.x) s += to_f(xr[c]);
    mean = block_sum(s, scratch) / h;
  }
  float ss = 0.f;
  for (int c = threadIdx.x; c < h; c += blockDim.x) {
    const float d = to_f(xr[c]) - mean;
    ss += d * d;
  }
  const float rstd = rsqrtf(block_sum(ss, scratch) / h + eps);
  T* yr = y + row * h;
  for (int c = threadIdx.x; c < h; c += blockDim.x) yr[c] = from_f<T>((to_f(xr[c]) - mean) * rstd * g[c]);
  if (threadIdx.x == 0) {
    if (!RMS) mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

template <typename T, bool RMS>
__global__ void norm_apply_k(const T* __restrict__ x, const float* __restrict__ g, const float* __restrict__ mean,
                             const float* __restrict__ rstd, T* __restrict__ y, int64_t n, int h) {
  const int64_t total = n * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / h;
    const int c = static_cast<int>(i % h);
    const float mu = RMS ? 0.f : mean[r];
    y[i] = from_f<T>((to_f(x[i]) - mu) * rstd[r] * g[c]);
  }
}

// Rows are strided over the grid; each thread keeps partial dg for its
// columns in registers-by-loop (accumulated in a per-block smem row) and the
// block flushes once with atomics.
template <typename T, bool RMS>
__global__ void norm_bwd_k(const T* __restrict__ dy, const T* __restrict__ x, const float* __restrict__ g,
                           const float* __restrict__ mean, const float* __restrict__ rstd, const T* dres, T* dx,
                           float* __restrict__ dg, int64_t n, int h) {
  extern __shared__ float dg_part[];  // [h]
  __shared__ float scratch[32];
  for (int c = threadIdx.x; c < h; c += blockDim.x) dg_part[c] = 0.f;
  for (int64_t row = blockIdx.x; row < n; row += gridDim.x) {
    const T* xr = x + row * h;
    const T* dyr = dy + row * h;
    const float mu = RMS ? 0.f : mean[row];
    const float rs = rstd[row];
    float s1 = 0.f, s2 = 0.f;
    for (int c = threadIdx.x; c < h; c += blockDim.x) {
      const float xh = (to_f(xr[c]) - mu) * rs;
      const float dxh = to_f(dyr[c]) * g[c];
      s1 += dxh;
      s2 += dxh * xh;
      dg_part[c] += to_f(dyr[c]) * xh;
    }
    const float m1 = RMS ? 0.f : block_sum(s1, scratch) / h;
    const float m2 = block_sum(s2, scratch) / h;
    T* dxr = dx + row * h;
    const T* drr = dres ? dres + row * h : nullptr;
    for (int c = threadIdx.x; c < h; c += blockDim.x) {
      const float xh = (to_f(xr[c]) - mu) * rs;
      const float dxh = to_f(dyr[c]) * g[c];
      float v = rs * (dxh - m1 - xh * m2);
      if (drr) v += to_f(drr[c]);
      dxr[c] = from_f<T>(v);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < h; c += blockDim.x) atomicAdd(&dg[c], dg_part[c]);
}

// ------------------------------------------------------------------ activations
__device__ __forceinline__ float gelu_tanh(float u) {
  const float c = 0.7978845608028654f;
  return 0.5f * u * (1.f + tanhf(c * (u + 0.044715f * u * u * u)));
}
__device__ __forceinline__ float sigmoidf_(float u) { return 1.f / (1.f + expf(-u)); }

template <typename T>
__global__ void act_fwd_k(int family, const T* __restrict__ u, T* __restrict__ g, int64_t n, int F) {
  const int64_t total = n * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    if (family == 0) {
      g[i] = from_f<T>(gelu_tanh(to_f(u[i])));
    } else {
      const int64_t r = i / F, c = i % F;
      const float a = to_f(u[r * 2 * F + c]), b = to_f(u[r * 2 * F + F + c]);
      g[i] = from_f<T>(a * sigmoidf_(a) * b);
    }
  }
}

template <typename T>
__global__ void act_bwd_k(int family, const T* __restrict__ u, const T* dg, T* du, int64_t n, int F) {
  const int64_t total = n * F;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    if (family == 0) {
      du[i] = from_f<T>(to_f(dg[i]) * gelu_tanh_grad(to_f(u[i])));
    } else {
      const int64_t r = i / F, c = i % F;
      const float a = to_f(u[r * 2 * F + c]), b = to_f(u[r * 2 * F + F + c]);
      const float d = to_f(dg[i]);  // dg may alias du's first half row-by-row: read before write
      const float s = sigmoidf_(a);
      const float da = d * b * s * (1.f + a * (1.f - s));
      const float db = d * a * s;
      du[r * 2 * F + c] = from_f<T>(da);
      du[r * 2 * F + F + c] = from_f<T>(db);
    }
  }
}

// ------------------------------------------------------------------ RoPE
// Angles in double: positions reach 128K and fp32 sin/cos of large angles would
// dominate the fp32 validation-mode error budget.
template <typename T>
__global__ void rope_k(T* x, int64_t ld, int64_t n, int H, int hd, int64_t pos0, float theta, bool inverse) {
  const int half = hd / 2;
  const int64_t total = n * H * half;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (H * half);
    const int rem = static_cast<int>(i % (H * half));
    const int head = rem / half, j = rem % half;
    const double inv_freq = pow(static_cast<double>(theta), -2.0 * j / hd);
    double sn, cs;
    sincos(static_cast<double>(pos0 + r) * inv_freq, &sn, &cs);
    T* p = x + r * ld + head * hd;
    const double a = to_f(p[j]), b = to_f(p[j + half]);
    const double s = inverse ? -sn : sn;
    p[j] = from_f<T>(static_cast<float>(a * cs - b * s));
    p[j + half] = from_f<T>(static_cast<float>(a * s + b * cs));
  }
}

template <typename T>
__global__ void assemble_dqkv_k(const T* __restrict__ dq, const float* __restrict__ dkv, T* __restrict__ out, int64_t n,
                                int h) {
  const int64_t total = n * 3 * h;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / (3 * h);
    const int c = static_cast<int>(i % (3 * h));
    out[i] = c < h ? dq[r * h + c] : from_f<T>(dkv[r * 2 * h + (c - h)]);
  }
}

// ------------------------------------------------------------------ cross-entropy
template <typename T>
__global__ void ce_k(T* logits, int64_t ld, const int32_t* __restrict__ labels, int V, float scale, double* loss) {
  __shared__ float scratch[32];
  const int64_t row = blockIdx.x;
  T* lr = logits + row * ld;
  float mx = -INFINITY;
  for (int c = threadIdx.x; c < V; c += blockDim.x) mx = fmaxf(mx, to_f(lr[c]));
  mx = block_max(mx, scratch);
  float s = 0.f;
  for (int c = threadIdx.x; c < V; c += blockDim.x) s += expf(to_f(lr[c]) - mx);
  s = block_sum(s, scratch);
  const int lab = labels[row];
  const float lab_logit = to_f(lr[lab]);
  __syncthreads();
  const float inv = 1.f / s;
  for (int c = threadIdx.x; c < V; c += blockDim.x) {
    const float p = expf(to_f(lr[c]) - mx) * inv;
    lr[c] = from_f<T>((p - (c == lab ? 1.f : 0.f)) * scale);
  }
  for (int64_t c = V + threadIdx.x; c < ld; c += blockDim.x) lr[c] = from_f<T>(0.f);  // padded vocab columns
  if (threadIdx.x == 0) atomicAdd(loss, static_cast<double>(logf(s) + mx - lab_logit));
}

// ------------------------------------------------------------------ misc
template <typename T>
__global__ void cast_k(const float* __restrict__ src, T* __restrict__ dst, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    dst[i] = from_f<T>(src[i]);
}

__device__ __forceinline__ uint64_t splitmix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

__global__ void fill_normal_k(float* p, int64_t n, uint64_t seed, float stddev) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r = splitmix64(seed * 0x2545F4914F6CDD1DULL + static_cast<uint64_t>(i));
    const double u1 = (static_cast<double>(r >> 11) + 0.5) * (1.0 / 9007199254740992.0);
    const double u2 = static_cast<double>(splitmix64(r) >> 11) * (1.0 / 9007199254740992.0);
    p[i] = static_cast<float>(stddev * sqrt(-2.0 * log(u1)) * cos(6.283185307179586 * u2));
  }
}

__global__ void fill_const_k(float* p, int64_t n, float v) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) p[i] = v;
}

template <typename T>
__global__ void adamw_k(float* p, const float* __restrict__ g, float* m, float* v, T* pc, int64_t n, float lr, float b1,
                        float b2, float eps, float wd, const float* __restrict__ bc) {
  const float bc1 = bc[0], bc2 = bc[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float gi = g[i];
    const float mi = b1 * m[i] + (1.f - b1) * gi;
    const float vi = b2 * v[i] + (1.f - b2) * gi * gi;
    m[i] = mi;
    v[i] = vi;
    float pi = p[i];
    pi -= lr * ((mi / bc1) / (sqrtf(vi / bc2) + eps) + wd * pi);
    p[i] = pi;
    if (pc) pc[i] = from_f<T>(pi);
  }
}

// 4 parameters per thread per step (float4 loads / stores; ~30 bytes of traffic
// per parameter, HBM bound).
template <typename T>
__global__ void adamw_vec_k(float4* p, const float4* __restrict__ g, float4* m, float4* v, T* pc, int64_t n4, float lr,
                            float b1, float b2, float eps, float wd, const float* __restrict__ bc) {
  const float bc1 = bc[0], bc2 = bc[1];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    const float4 gi = g[i];
    float4 mi = m[i], vi = v[i], pi = p[i];
    float* mf = &mi.x;
    float* vf = &vi.x;
    float* pf = &pi.x;
    const float* gf = &gi.x;
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      mf[e] = b1 * mf[e] + (1.f - b1) * gf[e];
      vf[e] = b2 * vf[e] + (1.f - b2) * gf[e] * gf[e];
      pf[e] -= lr * ((mf[e] / bc1) / (sqrtf(vf[e] / bc2) + eps) + wd * pf[e]);
    }
    m[i] = mi;
    v[i] = vi;
    p[i] = pi;
    if (pc) {
#pragma unroll
      for (int e = 0; e < 4; ++e) pc[4 * i + e] = from_f<T>(pf[e]);
    }
  }
}

// ------------------------------------------------------------------ bf16 fast paths
// Rows of h = 256*NV bf16: one warp per row, each lane owns NV chunks of 8
// contiguous columns (16-byte loads/stores, fully coalesced), the row stays in
// registers between the statistics pass and the output pass.
struct alignas(16) Bf8 {
  __nv_bfloat162 v[4];
};
__device__ __forceinline__ void bf8_to_f(const Bf8& b, float (&f)[8]) {
#pragma unroll
  for (int e = 0; e < 4; ++e) {
    const float2 t = __bfloat1622float2(b.v[e]);
    f[2 * e] = t.x;
    f[2 * e + 1] = t.y;
  }
}
__device__ __forceinline__ Bf8 f_to_bf8(const float (&f)[8]) {
  Bf8 b;
#pragma unroll
  for (int e = 0; e < 4; ++e) b.v[e] = __floats2bfloat162_rn(f[2 * e], f[2 * e + 1]);
  return b;
}
__device__ __forceinline__ void ld_f8(const float* p, float (&f)[8]) {
  const float4 a = __ldg(reinterpret_cast<const float4*>(p)), b = __ldg(reinterpret_cast<const float4*>(p) + 1);
  f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w;
  f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
}

// 16-byte global -> shared copies that bypass registers (LDGSTS): the streaming norm kernels
// prefetch the next row's slice into shared memory while they work on the current one.
__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gsrc) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(static_cast<uint32_t>(__cvta_generic_to_shared(smem_dst))),
               "l"(gsrc)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NV, bool RMS>
__global__ void __launch_bounds__(256) norm_fwd_vec_k(const __nv_bfloat16* __restrict__ x, const float* __restrict__ g,
                                                      __nv_bfloat16* __restrict__ y, float* __restrict__ mean_out,
                                                      float* __restrict__ rstd_out, int64_t n, float eps) {
  constexpr int H = 256 * NV;
  const int lane = threadIdx.x & 31;
  const int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + threadIdx.x / 32;
  if (row >= n) return;
  const Bf8* xr = reinterpret_cast<const Bf8*>(x + row * H);
  Bf8 xv[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) xv[k] = xr[k * 32 + lane];
  float mean = 0.f;
  if (!RMS) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      float f[8];
      bf8_to_f(xv[k], f);
#pragma unroll
      for (int e = 0; e < 8; ++e) s += f[e];
    }
    mean = warp_sum(s) / H;
  }
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    float f[8];
    bf8_to_f(xv[k], f);
#pragma unroll
    for (int e = 0; e < 8; ++e) ss += (f[e] - mean) * (f[e] - mean);
  }
  const float rstd = rsqrtf(warp_sum(ss) / H + eps);
  Bf8* yr = reinterpret_cast<Bf8*>(y + row * H);
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    float f[8], gv[8];
    bf8_to_f(xv[k], f);
    ld_f8(g + (k * 32 + lane) * 8, gv);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = (f[e] - mean) * rstd * gv[e];
    yr[k * 32 + lane] = f_to_bf8(f);
  }
  if (lane == 0) {
    if (!RMS) mean_out[row] = mean;
    rstd_out[row] = rstd;
  }
}

// Rows of h >= 2048: G warps per row (G = 2 for h 2048-3072, 4 for h >= 4096), each caching
// a 1/G slice of the row and its fp32 gain slice (loaded once) in registers. The grid is
// persistent (2 CTAs per SM striding over rows) and every warp copies its slice of the NEXT row into
// shared memory (cp.async, no registers) before reducing the current one: the DRAM latency of
// row r+1 hides behind the reductions, barrier and stores of row r (one row per warp and no
// prefetch left the HBM pipe idle between waves: 0.52 of HBM). Each slice computes its own
// mean and centred sum of squares (two passes over registers); the G slices combine them in
// one shared-memory exchange (Chan: M2 = sum M2_g + (H/G) sum (mean_g - mean)^2).
template <int NV, int G>
struct RowSlice {
  static constexpr int H = 256 * NV, NS = NV / G, RB = 8 / G;  // vectors per lane, rows per CTA
};
template <int NV, int G, bool RMS>
__global__ void __launch_bounds__(256, 2) norm_fwd_rows_k(const __nv_bfloat16* __restrict__ x,
                                                          const float* __restrict__ g, __nv_bfloat16* __restrict__ y,
                                                          float* __restrict__ mean_out, float* __restrict__ rstd_out,
                                                          int64_t n, float eps) {
  using RS = RowSlice<NV, G>;
  constexpr int H = RS::H, NS = RS::NS;
  extern __shared__ float4 pf4[];  // [8 warps][NS * 32] Bf8: the next row's slice
  __shared__ float2 xch[2][RS::RB][G];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, rb = w / G, gi = w % G;
  Bf8* pf = reinterpret_cast<Bf8*>(pf4) + w * NS * 32;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * RS::RB;
  int64_t row = static_cast<int64_t>(blockIdx.x) * RS::RB + rb;
  auto slice = [&](int64_t r) { return reinterpret_cast<const Bf8*>(x + r * H) + gi * NS * 32; };
  auto prefetch = [&](int64_t r) {
    const Bf8* xr = slice(r);
#pragma unroll
    for (int k = 0; k < NS; ++k) cp_async16(pf + k * 32 + lane, xr + k * 32 + lane);
    cp_async_commit();
  };
  if (row < n) prefetch(row);
  // The warp's gain slice is the same for every row it handles: load it once (ncu on the
  // per-row version: L1/TEX throughput 78 %, half of it the fp32 gain re-read every row).
  float gk[NS][8];
#pragma unroll
  for (int k = 0; k < NS; ++k) ld_f8(g + gi * (H / G) + (k * 32 + lane) * 8, gk[k]);
  for (int par = 0; row < n; row += stride, par ^= 1) {
    // The slice is converted to fp32 once and kept in registers for the three passes (mean,
    // centred squares, output): converting per pass cost 2 of the ~5 instructions per element
    // of this issue-bound kernel.
    float f[NS][8];
    cp_async_wait_all();
#pragma unroll
    for (int k = 0; k < NS; ++k) bf8_to_f(pf[k * 32 + lane], f[k]);  // own lane's chunks: no barrier
    if (row + stride < n) prefetch(row + stride);
    // Slice statistics (mg = the slice's mean, ss = its centred sum of squares; RMSNorm: mg = 0).
    // G = 4 (h >= 4096, latency-bound): each lane's own mean and centred squares over its NS*8
    // values, then ONE butterfly merging (mean, M2) pairs of equal counts (Chan: M2 = M2a + M2b
    // + (mb - ma)^2 n/2) -- one shuffle chain per row instead of two. G = 2 (issue-bound): the
    // butterfly's extra arithmetic costs more than the chain it saves (h 2560: 24.6 vs 22.7 us),
    // so a sum chain, then the squares about the slice mean.
    float mg = 0.f, ss = 0.f;
    if (RMS) {
#pragma unroll
      for (int k = 0; k < NS; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) ss += f[k][e] * f[k][e];
      ss = warp_sum(ss);
    } else if constexpr (G >= 4) {
#pragma unroll
      for (int k = 0; k < NS; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) mg += f[k][e];
      mg *= 1.f / (NS * 8);
#pragma unroll
      for (int k = 0; k < NS; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) ss += (f[k][e] - mg) * (f[k][e] - mg);
      float half = NS * 4;  // n/2 of each merged half
#pragma unroll
      for (int o = 16; o > 0; o >>= 1, half *= 2.f) {
        const float om = __shfl_xor_sync(0xffffffffu, mg, o), os = __shfl_xor_sync(0xffffffffu, ss, o);
        const float dm = om - mg;
        ss = ss + os + dm * dm * half;
        mg = 0.5f * (mg + om);
      }
    } else {
#pragma unroll
      for (int k = 0; k < NS; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) mg += f[k][e];
      mg = warp_sum(mg) * (static_cast<float>(G) / H);
#pragma unroll
      for (int k = 0; k < NS; ++k)
#pragma unroll
        for (int e = 0; e < 8; ++e) ss += (f[k][e] - mg) * (f[k][e] - mg);
      ss = warp_sum(ss);
    }
    if (lane == 0) xch[par][rb][gi] = make_float2(mg, ss);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + rb), "r"(32 * G) : "memory");
    float mean = 0.f, m2 = 0.f;
#pragma unroll
    for (int q = 0; q < G; ++q) mean += xch[par][rb][q].x;
    mean *= 1.f / G;
#pragma unroll
    for (int q = 0; q < G; ++q) {
      const float2 o = xch[par][rb][q];
      m2 += o.y + (RMS ? 0.f : (o.x - mean) * (o.x - mean) * (H / G));
    }
    if (RMS) mean = 0.f;
    const float rstd = rsqrtf(m2 / H + eps);
    Bf8* yr = reinterpret_cast<Bf8*>(y + row * H) + gi * NS * 32;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      float o[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) o[e] = (f[k][e] - mean) * rstd * gk[k][e];
      yr[k * 32 + lane] = f_to_bf8(o);
    }
    if (lane == 0 && gi == 0) {
      if (!RMS) mean_out[row] = mean;
      rstd_out[row] = rstd;
    }
  }
}

// y = (x - mean) * rstd * g: no reduction, so a flat grid-stride loop over 16-byte chunks
// (the MLP activation's access pattern, ~0.9 of HBM) instead of one row per warp.
template <int NV, bool RMS>
__global__ void __launch_bounds__(256) norm_apply_vec_k(const __nv_bfloat16* __restrict__ x, const float* __restrict__ g,
                                                        const float* __restrict__ mean, const float* __restrict__ rstd,
                                                        __nv_bfloat16* __restrict__ y, int64_t n) {
  constexpr int PER_ROW = 32 * NV;  // 16-byte chunks per row
  const int64_t chunks = n * PER_ROW;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < chunks;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t row = i / PER_ROW;
    const int c = static_cast<int>(i - row * PER_ROW);
    const float mu = RMS ? 0.f : __ldg(mean + row), rs = __ldg(rstd + row);
    float f[8], gv[8];
    bf8_to_f(reinterpret_cast<const Bf8*>(x)[i], f);
    ld_f8(g + c * 8, gv);
#pragma unroll
    for (int e = 0; e < 8; ++e) f[e] = (f[e] - mu) * rs * gv[e];
    reinterpret_cast<Bf8*>(y)[i] = f_to_bf8(f);
  }
}

// dx = rstd (g*dy - mean(g*dy) - xhat mean(g*dy*xhat)) (+ dres); dg += dy*xhat.
// Warps stride over rows; each warp accumulates dg for its lane-owned columns in
// its own shared-memory row (no atomics, no bank conflicts), the block sums its
// 8 rows and adds them to dg once.
template <int NV, bool RMS>
__global__ void __launch_bounds__(256) norm_bwd_vec_k(const __nv_bfloat16* __restrict__ dy,
                                                      const __nv_bfloat16* __restrict__ x, const float* __restrict__ g,
                                                      const float* __restrict__ mean, const float* __restrict__ rstd,
                                                      const __nv_bfloat16* dres, __nv_bfloat16* dx,
                                                      float* __restrict__ dg, int64_t n) {
  constexpr int H = 256 * NV;
  extern __shared__ float4 sdg4[];  // [8 warps][H] fp32
  float* sdg = reinterpret_cast<float*>(sdg4);
  const int lane = threadIdx.x & 31, w = threadIdx.x / 32;
  float* my = sdg + w * H;
  for (int c = lane * 4; c < H; c += 128) *reinterpret_cast<float4*>(my + c) = make_float4(0.f, 0.f, 0.f, 0.f);
  __syncwarp();
  for (int64_t row = static_cast<int64_t>(blockIdx.x) * 8 + w; row < n; row += static_cast<int64_t>(gridDim.x) * 8) {
    const Bf8* xr = reinterpret_cast<const Bf8*>(x + row * H);
    const Bf8* dyr = reinterpret_cast<const Bf8*>(dy + row * H);
    const float mu = RMS ? 0.f : mean[row], rs = rstd[row];
    // hd up to 2560 keeps the row in registers between the passes; wider rows
    // re-read it (L1/L2 hits) instead of spilling.
    constexpr bool CACHE = NV <= 10;
    Bf8 xv[CACHE ? NV : 1], dv[CACHE ? NV : 1];
    if constexpr (CACHE) {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        xv[k] = xr[k * 32 + lane];
        dv[k] = dyr[k * 32 + lane];
      }
    }
    float s1 = 0.f, s2 = 0.f;
#pragma unroll(CACHE ? NV : 2)
    for (int k = 0; k < NV; ++k) {
      float f[8], d[8], gv[8];
      bf8_to_f(CACHE ? xv[CACHE ? k : 0] : xr[k * 32 + lane], f);
      bf8_to_f(CACHE ? dv[CACHE ? k : 0] : dyr[k * 32 + lane], d);
      ld_f8(g + (k * 32 + lane) * 8, gv);
      float* acc = my + (k * 32 + lane) * 8;
      float4 a0 = *reinterpret_cast<float4*>(acc), a1 = *reinterpret_cast<float4*>(acc + 4);
      float av[8] = {a0.x, a0.y, a0.z, a0.w, a1.x, a1.y, a1.z, a1.w};
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (f[e] - mu) * rs, dxh = d[e] * gv[e];
        s1 += dxh;
        s2 += dxh * xh;
        av[e] += d[e] * xh;
      }
      *reinterpret_cast<float4*>(acc) = make_float4(av[0], av[1], av[2], av[3]);
      *reinterpret_cast<float4*>(acc + 4) = make_float4(av[4], av[5], av[6], av[7]);
    }
    const float m1 = RMS ? 0.f : warp_sum(s1) / H;
    const float m2 = warp_sum(s2) / H;
    Bf8* dxr = reinterpret_cast<Bf8*>(dx + row * H);
    const Bf8* drr = dres ? reinterpret_cast<const Bf8*>(dres + row * H) : nullptr;
#pragma unroll(CACHE ? NV : 2)
    for (int k = 0; k < NV; ++k) {
      float f[8], d[8], gv[8], r[8];
      bf8_to_f(CACHE ? xv[CACHE ? k : 0] : xr[k * 32 + lane], f);
      bf8_to_f(CACHE ? dv[CACHE ? k : 0] : dyr[k * 32 + lane], d);
      ld_f8(g + (k * 32 + lane) * 8, gv);
      if (drr) bf8_to_f(drr[k * 32 + lane], r);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (f[e] - mu) * rs;
        f[e] = rs * (d[e] * gv[e] - m1 - xh * m2) + (drr ? r[e] : 0.f);
      }
      dxr[k * 32 + lane] = f_to_bf8(f);
    }
  }
  __syncthreads();
  for (int c = threadIdx.x; c < H; c += 256) {
    float s = 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) s += sdg[k * H + c];
    atomicAdd(&dg[c], s);
  }
}

// Backward of the same row layout (G warps per row, persistent grid, next row's x / dy slice
// prefetched during the current row; the residual gradient is loaded at the top of the row's
// iteration so its latency hides behind the two reductions). dg partials: one shared-memory
// row of H/G floats per warp (no atomics), summed over the CTA's rows and added once.
template <int NV, int G, bool RMS>
__global__ void __launch_bounds__(256, 2) norm_bwd_rows_k(const __nv_bfloat16* __restrict__ dy,
                                                          const __nv_bfloat16* __restrict__ x,
                                                          const float* __restrict__ g, const float* __restrict__ mean,
                                                          const float* __restrict__ rstd, const __nv_bfloat16* dres,
                                                          __nv_bfloat16* dx, float* __restrict__ dg, int64_t n) {
  using RS = RowSlice<NV, G>;
  constexpr int H = RS::H, NS = RS::NS, HS = H / G, SL = NS * 32;  // SL: 16-byte vectors per slice
  // per warp: x / dy slices double-buffered + the residual-gradient slice, all filled by
  // cp.async; reused for the dgain block reduction at the end
  extern __shared__ float4 sm4[];
  Bf8* pf = reinterpret_cast<Bf8*>(sm4) + (threadIdx.x >> 5) * 5 * SL;
  __shared__ float2 xch[2][RS::RB][G];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, rb = w / G, gi = w % G;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * RS::RB;
  int64_t row = static_cast<int64_t>(blockIdx.x) * RS::RB + rb;
  auto sl = [&](const __nv_bfloat16* base, int64_t r) { return reinterpret_cast<const Bf8*>(base + r * H) + gi * NS * 32; };
  auto prefetch_xdy = [&](int64_t r, int stg) {
    const Bf8 *xr = sl(x, r), *dyr = sl(dy, r);
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      cp_async16(pf + (2 * stg) * SL + k * 32 + lane, xr + k * 32 + lane);
      cp_async16(pf + (2 * stg + 1) * SL + k * 32 + lane, dyr + k * 32 + lane);
    }
    cp_async_commit();
  };
  // gain slice and dgain partials stay in registers across the warp's rows (per-row re-reads
  // of the fp32 gain and a shared-memory read-modify-write of the partials kept the per-row
  // kernel L1-bound)
  float gk[NS][8], dga[NS][8];
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    ld_f8(g + gi * HS + (k * 32 + lane) * 8, gk[k]);
#pragma unroll
    for (int e = 0; e < 8; ++e) dga[k][e] = 0.f;
  }
  if (row < n) prefetch_xdy(row, 0);
  for (int par = 0, stg = 0; row < n; row += stride, par ^= 1, stg ^= 1) {
    const bool more = row + stride < n;
    if (dres) {  // group: residual gradient of this row
      const Bf8* rr = sl(dres, row);
#pragma unroll
      for (int k = 0; k < NS; ++k) cp_async16(pf + 4 * SL + k * 32 + lane, rr + k * 32 + lane);
    }
    cp_async_commit();
    if (more) prefetch_xdy(row + stride, stg ^ 1);  // group: next row's x / dy
    if (more)
      cp_async_wait<2>();  // this row's x / dy landed (issued one iteration ago)
    else
      cp_async_wait<1>();
    const Bf8 *xs = pf + (2 * stg) * SL, *ds = xs + SL, *rs = pf + 4 * SL;
    const float mu = RMS ? 0.f : mean[row], rsd = rstd[row];
    float s1 = 0.f, s2 = 0.f;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      float f[8], d[8];
      bf8_to_f(xs[k * 32 + lane], f);
      bf8_to_f(ds[k * 32 + lane], d);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (f[e] - mu) * rsd, dxh = d[e] * gk[k][e];
        s1 += dxh;
        s2 += dxh * xh;
        dga[k][e] += d[e] * xh;
      }
    }
    s1 = RMS ? 0.f : warp_sum(s1);
    s2 = warp_sum(s2);
    if (lane == 0) xch[par][rb][gi] = make_float2(s1, s2);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + rb), "r"(32 * G) : "memory");
    float t1 = 0.f, t2 = 0.f;
#pragma unroll
    for (int q = 0; q < G; ++q) {
      t1 += xch[par][rb][q].x;
      t2 += xch[par][rb][q].y;
    }
    const float m1 = RMS ? 0.f : t1 / H, m2 = t2 / H;
    if (more)
      cp_async_wait<1>();  // the residual gradient landed
    else
      cp_async_wait<0>();
    Bf8* dxr = reinterpret_cast<Bf8*>(dx + row * H) + gi * NS * 32;
#pragma unroll
    for (int k = 0; k < NS; ++k) {
      float f[8], d[8], r[8];
      bf8_to_f(xs[k * 32 + lane], f);
      bf8_to_f(ds[k * 32 + lane], d);
      if (dres) bf8_to_f(rs[k * 32 + lane], r);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float xh = (f[e] - mu) * rsd;
        f[e] = rsd * (d[e] * gk[k][e] - m1 - xh * m2) + (dres ? r[e] : 0.f);
      }
      dxr[k * 32 + lane] = f_to_bf8(f);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  float* sdg = reinterpret_cast<float*>(sm4);  // [8 warps][H/G]
#pragma unroll
  for (int k = 0; k < NS; ++k) {
    float* dst = sdg + w * HS + (k * 32 + lane) * 8;
    *reinterpret_cast<float4*>(dst) = make_float4(dga[k][0], dga[k][1], dga[k][2], dga[k][3]);
    *reinterpret_cast<float4*>(dst + 4) = make_float4(dga[k][4], dga[k][5], dga[k][6], dga[k][7]);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < H; c += 256) {
    const int q = c / HS, cc = c - q * HS;
    float acc = 0.f;
#pragma unroll
    for (int r = 0; r < RS::RB; ++r) acc += sdg[(r * G + q) * HS + cc];
    atomicAdd(&dg[c], acc);
  }
}

// bf16 rows (ld % 8 == 0): 16-byte vectors and exp2 on the MUFU -- the scalar
// version above issued ~100 two-byte loads per thread per pass and ran at a
// quarter of HBM bandwidth. Columns >= V (vocabulary padding) are excluded from
// max / sum and written as 0.
__global__ void __launch_bounds__(512) ce_vec_k(__nv_bfloat16* logits, int64_t ld, const int32_t* __restrict__ labels,
                                                int V, float scale, double* loss) {
  __shared__ float scratch[32];
  const int64_t row = blockIdx.x;
  __nv_bfloat16* lr = logits + row * ld;
  Bf8* lv = reinterpret_cast<Bf8*>(lr);
  const int nv = static_cast<int>(ld / 8);
  constexpr float kLog2e = 1.4426950408889634f;
  float mx = -INFINITY;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    float f[8];
    bf8_to_f(lv[i], f);
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (i * 8 + e < V) mx = fmaxf(mx, f[e]);
  }
  mx = block_max(mx, scratch);
  const float nm = -mx * kLog2e;
  float s = 0.f;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    float f[8];
    bf8_to_f(lv[i], f);
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (i * 8 + e < V) s += exp2f(fmaf(f[e], kLog2e, nm));
  }
  s = block_sum(s, scratch);
  const int lab = labels[row];
  const float lab_logit = __bfloat162float(lr[lab]);
  __syncthreads();
  const float inv = scale / s;
  for (int i = threadIdx.x; i < nv; i += blockDim.x) {
    float f[8];
    bf8_to_f(lv[i], f);
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      const int c = i * 8 + e;
      f[e] = c < V ? exp2f(fmaf(f[e], kLog2e, nm)) * inv - (c == lab ? scale : 0.f) : 0.f;
    }
    lv[i] = f_to_bf8(f);
  }
  if (threadIdx.x == 0) atomicAdd(loss, static_cast<double>(logf(s) + mx - lab_logit));
}

__device__ __forceinline__ float gelu_f(float u) { return gelu_tanh(u); }

// bf16 production path: MUFU tanh (tanh.approx.f32, max rel. error ~2^-11, far
// below the bf16 output rounding). libm tanhf made these HBM-sized kernels
// issue-bound (~20 instructions per element). The fp32 validation path keeps tanhf.
__device__ __forceinline__ float gelu_fast(float u) {
  const float c = 0.7978845608028654f;
  return 0.5f * u * (1.f + tanh_fast(c * (u + 0.044715f * u * u * u)));
}
__device__ __forceinline__ float sigmoid_fast(float u) { return fmaf(0.5f, tanh_fast(0.5f * u), 0.5f); }

// GeLU (family 0) / SwiGLU (family 1) over 8-element vectors.
__global__ void act_fwd_vec_k(int family, const __nv_bfloat16* __restrict__ u, __nv_bfloat16* __restrict__ g,
                              int64_t n, int F) {
  const int64_t chunks = n * F / 8, per_row = F / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunks; i += (int64_t)gridDim.x * blockDim.x) {
    float a[8];
    if (family == 0) {
      bf8_to_f(reinterpret_cast<const Bf8*>(u)[i], a);
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] = gelu_fast(a[e]);
    } else {
      const int64_t r = i / per_row, c = i % per_row;
      float b[8];
      bf8_to_f(reinterpret_cast<const Bf8*>(u)[r * 2 * per_row + c], a);
      bf8_to_f(reinterpret_cast<const Bf8*>(u)[r * 2 * per_row + per_row + c], b);
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] = a[e] * sigmoid_fast(a[e]) * b[e];
    }
    reinterpret_cast<Bf8*>(g)[i] = f_to_bf8(a);
  }
}

__global__ void act_bwd_vec_k(int family, const __nv_bfloat16* __restrict__ u, const __nv_bfloat16* dg,
                              __nv_bfloat16* du, int64_t n, int F) {
  const int64_t chunks = n * F / 8, per_row = F / 8;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunks; i += (int64_t)gridDim.x * blockDim.x) {
    float d[8];
    bf8_to_f(reinterpret_cast<const Bf8*>(dg)[i], d);
    if (family == 0) {
      float a[8];
      bf8_to_f(reinterpret_cast<const Bf8*>(u)[i], a);
#pragma unroll
      for (int e = 0; e < 8; ++e) a[e] = d[e] * gelu_grad_fast(a[e]);
      reinterpret_cast<Bf8*>(du)[i] = f_to_bf8(a);
    } else {
      const int64_t r = i / per_row, c = i % per_row;
      float a[8], b[8];
      bf8_to_f(reinterpret_cast<const Bf8*>(u)[r * 2 * per_row + c], a);
      bf8_to_f(reinterpret_cast<const Bf8*>(u)[r * 2 * per_row + per_row + c], b);
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        const float s = sigmoid_fast(a[e]);
        const float da = d[e] * b[e] * s * (1.f + a[e] * (1.f - s)), db = d[e] * a[e] * s;
        a[e] = da;
        b[e] = db;
      }
      reinterpret_cast<Bf8*>(du)[r * 2 * per_row + c] = f_to_bf8(a);
      reinterpret_cast<Bf8*>(du)[r * 2 * per_row + per_row + c] = f_to_bf8(b);
    }
  }
}

// [dq | dk | dv] rows for the QKV dgrad / wgrad GEMMs: dq bf16 [n, h], dK/dV
// fp32 rows of the accumulator [n, 2h] -> bf16 [n, 3h]; 8 columns per thread.
__global__ void assemble_dqkv_vec_k(const __nv_bfloat16* __restrict__ dq, const float* __restrict__ dkv,
                                    __nv_bfloat16* __restrict__ out, int64_t n, int h) {
  const int64_t per_row = 3 * h / 8, chunks = n * per_row;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < chunks; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = i / per_row;
    const int c = static_cast<int>(i % per_row) * 8;
    if (c < h) {
      reinterpret_cast<Bf8*>(out)[i] = reinterpret_cast<const Bf8*>(dq + r * h + c)[0];
    } else {
      float f[8];
      const float* src = dkv + r * 2 * h + (c - h);
      const float4 a = *reinterpret_cast<const float4*>(src), b = *reinterpret_cast<const float4*>(src + 4);
      f[0] = a.x; f[1] = a.y; f[2] = a.z; f[3] = a.w; f[4] = b.x; f[5] = b.y; f[6] = b.z; f[7] = b.w;
      reinterpret_cast<Bf8*>(out)[i] = f_to_bf8(f);
    }
  }
}

// NV dispatch for the row kernels (h = 256 * NV); false = no fast path.
template <typename F>
bool dispatch_nv(int h, F&& f) {
  if (h % 256) return false;
  switch (h / 256) {
    case 1: f(std::integral_constant<int, 1>{}); return true;
    case 2: f(std::integral_constant<int, 2>{}); return true;
    case 4: f(std::integral_constant<int, 4>{}); return true;
    case 8: f(std::integral_constant<int, 8>{}); return true;
    case 10: f(std::integral_constant<int, 10>{}); return true;
    case 12: f(std::integral_constant<int, 12>{}); return true;
    case 16: f(std::integral_constant<int, 16>{}); return true;
    case 20: f(std::integral_constant<int, 20>{}); return true;
    default: return false;
  }
}

}  // namespace

#define SPK_DISPATCH(t, ...)                 \
  if ((t) == DType::kF32) {                  \
    using T = float;                         \
    __VA_ARGS__;                             \
  } else {                                   \
    using T = __nv_bfloat16;                 \
    __VA_ARGS__;                             \
  }

void embed_fwd(DType t, const int32_t* tok, const float* E, const float* pos, int64_t pos0, void* x, int64_t n, int h,
               cudaStream_t s) {
  SPK_DISPATCH(t, embed_fwd_k<T><<<stream_grid(n * h, 256), 256, 0, s>>>(tok, E, pos, pos0, (T*)x, n, h));
  SPK_LAUNCH_CHECK();
}

void embed_bwd(DType t, const int32_t* tok, const void* dx, float* dE, float* dpos, int64_t pos0, int64_t n, int h,
               cudaStream_t s) {
  SPK_DISPATCH(t, embed_bwd_k<T><<<stream_grid(n * h, 256), 256, 0, s>>>(tok, (const T*)dx, dE, dpos, pos0, n, h));
  SPK_LAUNCH_CHECK();
}

void norm_fwd(DType t, bool rms, const void* x, const float* g, void* y, float* mean, float* rstd, int64_t n, int h,
              float eps, cudaStream_t s) {
  if (n == 0) return;
  if (t == DType::kBF16 && dispatch_nv(h, [&](auto nv) {
        constexpr int NV = decltype(nv)::value;
        const auto* xb = static_cast<const __nv_bfloat16*>(x);
        auto* yb = static_cast<__nv_bfloat16*>(y);
        if constexpr (NV >= 8 && NV % 2 == 0) {
          constexpr int G = NV >= 16 ? 4 : 2;
          const int64_t blocks = (n + 8 / G - 1) / (8 / G);
          const unsigned grid = static_cast<unsigned>(std::min<int64_t>(blocks, 2 * num_sms()));
          const size_t pf = 8 * (NV / G) * 32 * 16;  // next-row slices, [8 warps][NS * 32] x 16 B
          if (rms)
            norm_fwd_rows_k<NV, G, true><<<grid, 256, pf, s>>>(xb, g, yb, mean, rstd, n, eps);
          else
            norm_fwd_rows_k<NV, G, false><<<grid, 256, pf, s>>>(xb, g, yb, mean, rstd, n, eps);
          return;
        }
        const unsigned grid = static_cast<unsigned>((n + 7) / 8);
        if (rms)
          norm_fwd_vec_k<NV, true><<<grid, 256, 0, s>>>(xb, g, yb, mean, rstd, n, eps);
        else
          norm_fwd_vec_k<NV, false><<<grid, 256, 0, s>>>(xb, g, yb, mean, rstd, n, eps);
      })) {
    SPK_LAUNCH_CHECK();
    return;
  }
  SPK_DISPATCH(t, {
    if (rms)
      norm_fwd_k<T, true><<<n, kRowThreads, 0, s>>>((const T*)x, g, (T*)y, mean, rstd, h, eps);
    else
      norm_fwd_k<T, false><<<n, kRowThreads, 0, s>>>((const T*)x, g, (T*)y, mean, rstd, h, eps);
  });
  SPK_LAUNCH_CHECK();
}

void norm_apply(DType t, bool rms, const void* x, const float* g, const float* mean, const float* rstd, void* y,
                int64_t n, int h, cudaStream_t s) {
  if (n == 0) return;
  if (t == DType::kBF16 && dispatch_nv(h, [&](auto nv) {
        constexpr int NV = decltype(nv)::value;
        const unsigned grid = static_cast<unsigned>(stream_grid(n * 32 * NV, 256));
        const auto* xb = static_cast<const __nv_bfloat16*>(x);
        auto* yb = static_cast<__nv_bfloat16*>(y);
        if (rms)
          norm_apply_vec_k<NV, true><<<grid, 256, 0, s>>>(xb, g, mean, rstd, yb, n);
        else
          norm_apply_vec_k<NV, false><<<grid, 256, 0, s>>>(xb, g, mean, rstd, yb, n);
      })) {
    SPK_LAUNCH_CHECK();
    return;
  }
  SPK_DISPATCH(t, {
    if (rms)
      norm_apply_k<T, true><<<stream_grid(n * h, 256), 256, 0, s>>>((const T*)x, g, mean, rstd, (T*)y, n, h);
    else
      norm_apply_k<T, false><<<stream_grid(n * h, 256), 256, 0, s>>>((const T*)x, g, mean, rstd, (T*)y, n, h);
  });
  SPK_LAUNCH_CHECK();
}

void norm_bwd(DType t, bool rms, const void* dy, const void* x, const float* g, const float* mean, const float* rstd,
              const void* dres, void* dx, float* dg, int64_t n, int h, cudaStream_t s) {
  if (n == 0) return;
  if (t == DType::kBF16 && dispatch_nv(h, [&](auto nv) {
        constexpr int NV = decltype(nv)::value;
        const size_t sm = sizeof(float) * 8 * 256 * NV;
        const int64_t blocks = (n + 7) / 8;
        const unsigned grid = static_cast<unsigned>(blocks < num_sms() ? blocks : num_sms());
        auto launch = [&](auto kern) {
          SPK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
          kern<<<grid, 256, sm, s>>>(static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x), g, mean,
                                     rstd, static_cast<const __nv_bfloat16*>(dres), static_cast<__nv_bfloat16*>(dx), dg, n);
        };
        if constexpr (NV >= 8 && NV % 2 == 0) {  // G warps per row, persistent, next row prefetched
          constexpr int G = NV >= 16 ? 4 : 2;
          const size_t sm2 = std::max<size_t>(8 * 5 * (NV / G) * 32 * 16, sizeof(float) * 8 * (256 * NV / G));
          const int64_t b2 = (n + 8 / G - 1) / (8 / G);
          const unsigned grid2 = static_cast<unsigned>(std::min<int64_t>(b2, 2 * num_sms()));
          auto launch2 = [&](auto kern) {
            SPK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm2));
            kern<<<grid2, 256, sm2, s>>>(static_cast<const __nv_bfloat16*>(dy), static_cast<const __nv_bfloat16*>(x), g,
                                        mean, rstd, static_cast<const __nv_bfloat16*>(dres),
                                        static_cast<__nv_bfloat16*>(dx), dg, n);
          };
          if (rms)
            launch2(norm_bwd_rows_k<NV, G, true>);
          else
            launch2(norm_bwd_rows_k<NV, G, false>);
          return;
        }
        if (rms)
          launch(norm_bwd_vec_k<NV, true>);
        else
          launch(norm_bwd_vec_k<NV, false>);
      })) {
    SPK_LAUNCH_CHECK();
    return;
  }
  const int grid = static_cast<int>(n < 2 * num_sms() ? n : 2 * num_sms());
  const size_t smem = sizeof(float) * h;
  SPK_DISPATCH(t, {
    if (rms) {
      if (smem > 48 * 1024) cudaFuncSetAttribute(norm_bwd_k<T, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      norm_bwd_k<T, true><<<grid, kRowThreads, smem, s>>>((const T*)dy, (const T*)x, g, mean, rstd, (const T*)dres,
                                                          (T*)dx, dg, n, h);
    } else {
      if (smem > 48 * 1024) cudaFuncSetAttribute(norm_bwd_k<T, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
      norm_bwd_k<T, false><<<grid, kRowThreads, smem, s>>>((const T*)dy, (const T*)x, g, mean, rstd, (const T*)dres,
                                                           (T*)dx, dg, n, h);
    }
  });
  SPK_LAUNCH_CHECK();
}

void act_fwd(DType t, int family, const void* u, void* g, int64_t n, int F, cudaStream_t s) {
  if (t == DType::kBF16 && F % 8 == 0) {
    act_fwd_vec_k<<<stream_grid(n * F / 8, 256), 256, 0, s>>>(family, static_cast<const __nv_bfloat16*>(u),
                                                               static_cast<__nv_bfloat16*>(g), n, F);
    SPK_LAUNCH_CHECK();
    return;
  }
  SPK_DISPATCH(t, act_fwd_k<T><<<stream_grid(n * F, 256), 256, 0, s>>>(family, (const T*)u, (T*)g, n, F));
  SPK_LAUNCH_CHECK();
}

void act_bwd(DType t, int family, const void* u, const void* dg, void* du, int64_t n, int F, cudaStream_t s) {
  if (t == DType::kBF16 && F % 8 == 0) {
    act_bwd_vec_k<<<stream_grid(n * F / 8, 256), 256, 0, s>>>(family, static_cast<const __nv_bfloat16*>(u),
                                                               static_cast<const __nv_bfloat16*>(dg),
                                                               static_cast<__nv_bfloat16*>(du), n, F);
    SPK_LAUNCH_CHECK();
    return;
  }
  SPK_DISPATCH(t, act_bwd_k<T><<<stream_grid(n * F, 256), 256, 0, s>>>(family, (const T*)u, (const T*)dg, (T*)du, n, F));
  SPK_LAUNCH_CHECK();
}

void rope(DType t, void* x, int64_t ld, int64_t n, int H, int hd, int64_t pos0, float theta, bool inverse,
          cudaStream_t s) {
  SPK_DISPATCH(t, rope_k<T><<<stream_grid(n * H * hd / 2, 256), 256, 0, s>>>((T*)x, ld, n, H, hd, pos0, theta, inverse));
  SPK_LAUNCH_CHECK();
}

void assemble_dqkv(DType t, const void* dq, const float* dkv, void* dqkv, int64_t n, int h, cudaStream_t s) {
  if (t == DType::kBF16 && h % 8 == 0) {
    assemble_dqkv_vec_k<<<stream_grid(n * 3 * h / 8, 256), 256, 0, s>>>(static_cast<const __nv_bfloat16*>(dq), dkv,
                                                                          static_cast<__nv_bfloat16*>(dqkv), n, h);
    SPK_LAUNCH_CHECK();
    return;
  }
  SPK_DISPATCH(t, assemble_dqkv_k<T><<<stream_grid(n * 3 * h, 256), 256, 0, s>>>((const T*)dq, dkv, (T*)dqkv, n, h));
  SPK_LAUNCH_CHECK();
}

void ce_fwd_bwd(DType t, void* logits, int64_t ld, const int32_t* labels, int64_t n, int V, float scale, double* loss,
                cudaStream_t s) {
  if (n == 0) return;
  if (t == DType::kBF16 && ld % 8 == 0 && (reinterpret_cast<uintptr_t>(logits) & 15) == 0) {
    ce_vec_k<<<n, 512, 0, s>>>(static_cast<__nv_bfloat16*>(logits), ld, labels, V, scale, loss);
    SPK_LAUNCH_CHECK();
    return;
  }
  SPK_DISPATCH(t, ce_k<T><<<n, 512, 0, s>>>((T*)logits, ld, labels, V, scale, loss));
  SPK_LAUNCH_CHECK();
}

void cast_from_f32(DType t, const float* src, void* dst, int64_t n, cudaStream_t s) {
  SPK_DISPATCH(t, cast_k<T><<<stream_grid(n, 256), 256, 0, s>>>(src, (T*)dst, n));
  SPK_LAUNCH_CHECK();
}

void fill_normal(float* p, int64_t n, uint64_t seed, float stddev, cudaStream_t s) {
  fill_normal_k<<<stream_grid(n, 256), 256, 0, s>>>(p, n, seed, stddev);
  SPK_LAUNCH_CHECK();
}

void fill_const(float* p, int64_t n, float v, cudaStream_t s) {
  fill_const_k<<<stream_grid(n, 256), 256, 0, s>>>(p, n, v);
  SPK_LAUNCH_CHECK();
}

void adamw(float* p, const float* g, float* m, float* v, void* pc, DType t, int64_t n, float lr, float b1, float b2,
           float eps, float wd, const float* bc, cudaStream_t s) {
  const auto al16 = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
  if (n % 4 == 0 && al16(p) && al16(g) && al16(m) && al16(v)) {
    SPK_DISPATCH(t, adamw_vec_k<T><<<stream_grid(n / 4, 256), 256, 0, s>>>(
                        reinterpret_cast<float4*>(p), reinterpret_cast<const float4*>(g), reinterpret_cast<float4*>(m),
                        reinterpret_cast<float4*>(v), (T*)pc, n / 4, lr, b1, b2, eps, wd, bc));
    SPK_LAUNCH_CHECK();
    return;
  }
  SPK_DISPATCH(t, adamw_k<T><<<stream_grid(n, 256), 256, 0, s>>>(p, g, m, v, (T*)pc, n, lr, b1, b2, eps, wd, bc));
  SPK_LAUNCH_CHECK();
}

const void* module_anchor_elementwise() { return reinterpret_cast<const void*>(&embed_fwd_k<float>); }

}  // namespace spk
