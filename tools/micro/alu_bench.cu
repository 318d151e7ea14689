// Throughput of the softmax building blocks on sm_100a: MUFU.EX2, the FMA-pipe
// exp2 polynomial, F2FP (bf16x2 pack), FFMA2. 4 or 16 warps per SM, cycles per
// warp-instruction per SMSP.
#include <cstdio>
#include <cstdint>
#include <cuda_bf16.h>
__device__ __forceinline__ float ex2(float x) { float y; asm volatile("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x)); return y; }
template <int KIND>
__global__ void k(int iters, float* out, unsigned long long* cyc) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3f - i * 0.1f;
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (KIND == 0) a[i] = ex2(a[i]) - 1.0f;
      if (KIND == 1) {
        __nv_bfloat162 v = __floats2bfloat162_rn(a[i], a[(i + 1) & 7]);
        acc += *reinterpret_cast<uint32_t*>(&v);
        a[i] += 1e-7f;
      }
      if (KIND == 2) a[i] = fmaf(a[i], 0.999f, 1e-4f);
      if (KIND == 3) {  // one MUFU.EX2 + one F2FP per element: shared pipe => ~8 + 3.5 cycles
        a[i] = ex2(a[i]) - 1.0f;
        __nv_bfloat162 v = __floats2bfloat162_rn(a[i], a[(i + 3) & 7]);
        acc += *reinterpret_cast<uint32_t*>(&v);
      }
      if (KIND == 5) {  // packed f16x2 exp2: two elements per lane-instruction
        uint32_t h, y;
        asm volatile("cvt.rn.f16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(h));
        acc += y;
        a[i] += 1e-7f;
      }
      if (KIND == 6) {  // packed bf16x2 exp2
        uint32_t h, y;
        asm volatile("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(a[i]), "f"(a[(i + 1) & 7]));
        asm volatile("ex2.approx.ftz.bf16x2 %0, %1;" : "=r"(y) : "r"(h));
        acc += y;
        a[i] += 1e-7f;
      }
      if (KIND == 7) {  // ex2 f16x2 alone (input chain through the result)
        uint32_t y;
        asm volatile("ex2.approx.f16x2 %0, %1;" : "=r"(y) : "r"(acc + i));
        acc ^= y;
      }
      if (KIND == 4) {  // PRMT-based bf16x2 pack with round-half-up (integer pipe)
        const uint32_t x0 = __float_as_uint(a[i]) + 0x8000u, x1 = __float_as_uint(a[(i + 1) & 7]) + 0x8000u;
        uint32_t v;
        asm("prmt.b32 %0, %1, %2, 0x7632;" : "=r"(v) : "r"(x0), "r"(x1));
        acc += v;
        a[i] += 1e-7f;
      }
    }
  }
  unsigned long long t1 = clock64();
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s + acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  float* o; unsigned long long* c; cudaMalloc(&o, 148 * 1024 * 4); cudaMalloc(&c, 148 * 8);
  const char* nm[] = {"MUFU.EX2", "F2FP pack", "FFMA", "EX2+F2FP", "PRMT pack", "cvt+ex2 f16x2", "cvt+ex2 bf16x2", "ex2 f16x2"};
  for (int kind = 0; kind < 8; ++kind)
    for (int warps : {4, 8, 16, 32}) {
      const int iters = 2048;
      if (kind == 0) k<0><<<148, warps * 32>>>(iters, o, c);
      if (kind == 1) k<1><<<148, warps * 32>>>(iters, o, c);
      if (kind == 2) k<2><<<148, warps * 32>>>(iters, o, c);
      if (kind == 3) k<3><<<148, warps * 32>>>(iters, o, c);
      if (kind == 4) k<4><<<148, warps * 32>>>(iters, o, c);
      if (kind == 5) k<5><<<148, warps * 32>>>(iters, o, c);
      if (kind == 6) k<6><<<148, warps * 32>>>(iters, o, c);
      if (kind == 7) k<7><<<148, warps * 32>>>(iters, o, c);
      unsigned long long h; cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
      const double inst_per_smsp = (double)iters * 8 * warps / 4;
      printf("%-10s %2d warps: %.2f cycles per warp-instruction per SMSP (%.1f lanes/clk/SM)\n", nm[kind], warps,
             h / inst_per_smsp, 128.0 * inst_per_smsp / h);
    }
  return 0;
}
