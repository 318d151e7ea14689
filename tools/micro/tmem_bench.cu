// Microbenchmarks of the tcgen05 datapath on sm_100a (B200): TMEM load
// bandwidth (tcgen05.ld 32x32b.x32 from 4 or 8 warps) and MMA issue rates for
// the attention shapes (SS 128x64x16, TS 128x80x16, SS 128x128x16).
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I../../paper_2406_03488_b200/csrc tmem_bench.cu -o tmem_bench -lcuda
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#include "cuda/tc_common.cuh"
using namespace spk;

__global__ void __launch_bounds__(384, 1) ld_bench(int iters, int nwarps, unsigned long long* out, uint32_t* sink) {
  __shared__ uint32_t slot;
  __shared__ uint64_t bar;
  const int warp = threadIdx.x / 32;
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  uint32_t acc = 0;
  unsigned long long t0 = clock64();
  if (warp < nwarps) {
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    for (int i = 0; i < iters; ++i) {
      uint32_t r[32];
      tc::tmem_ld32(tmem + lane_base + ((i * 32 + (warp >> 2) * 256) & 511), r);
      tc::tmem_ld_wait();
#pragma unroll
      for (int k = 0; k < 32; ++k) acc += r[k];
    }
  }
  __syncthreads();
  unsigned long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 0x12345) sink[threadIdx.x] = acc;
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

// MMA rate: one warp issues `iters` MMAs of the given kind back to back; the
// commit at the end is waited on; cycles / iters = cycles per MMA.
template <int KIND>
__global__ void __launch_bounds__(384, 1) mma_bench(int iters, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ uint64_t bar, bar2[3];
  __shared__ int stop_flag;
  const int warp = threadIdx.x / 32;
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
  if (threadIdx.x == 0) {
    stop_flag = 0;
    tc::mbar_init(&bar, 1);
    for (int i = 0; i < 3; ++i) tc::mbar_init(&bar2[i], 1);
    tc::mbar_arrive(&bar2[1]);  // complete phase 0 so KIND 11 waits on a finished phase
    tc::fence_mbar_init();
  }
  if (warp == 0) tc::tmem_alloc(&slot, 512);
  tc::tc_fence_before();
  __syncthreads();
  tc::tc_fence_after();
  const uint32_t tmem = slot;
  if (warp == 1) {
    const uint32_t a = tc::smem_u32(base), b = tc::smem_u32(base + 65536);
    const uint64_t ad = tc::smem_desc(a, 16, 1024, tc::kSwizzle128B), bd = tc::smem_desc(b, 16, 1024, tc::kSwizzle128B);
    const uint64_t bmn = tc::smem_desc(b, 16384, 1024, tc::kSwizzle128B);
    unsigned long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      if (KIND == 0) tc::mma_bf16_ss_w(tmem, ad, bd, tc::idesc_bf16(128, 64, false, false), 1);
      if (KIND == 1) tc::mma_bf16_ts_w(tmem + 256, tmem, bmn, tc::idesc_bf16(128, 80, false, true), 1);
      if (KIND == 2) tc::mma_bf16_ss_w(tmem, ad, bd, tc::idesc_bf16(128, 128, false, false), 1);
      if (KIND == 3) tc::mma_bf16_ss_w(tmem, ad, bd, tc::idesc_bf16(128, 256, false, false), 1);
      if (KIND == 4) tc::mma_bf16_ts_w(tmem + 256, tmem, bmn, tc::idesc_bf16(128, 256, false, true), 1);
      if (KIND == 7) tc::mma_bf16_ts_w(tmem + 256, tmem, bd, tc::idesc_bf16(128, 64, false, false), 1);
      if (KIND == 8) tc::mma_bf16_ts_w(tmem + 256, tmem, bd, tc::idesc_bf16(128, 32, false, false), 1);
      if (KIND == 9) tc::mma_bf16_ts_w(tmem + 256, tmem, bd, tc::idesc_bf16(128, 16, false, false), 1);
      if (KIND == 10) tc::mma_bf16_ss_w(tmem + 256, ad, bd, tc::idesc_bf16(128, 32, false, false), 1);
      // fused-backward dQ^T = K^T dS^T shapes: B = dS^T tile, MN-major (N = queries)
      if (KIND == 14)
        tc::mma_bf16_ts_w(tmem + 256, tmem, tc::smem_desc(b + (i & 7) * 1024, 4096, 512, tc::kSwizzle64B),
                          tc::idesc_bf16(128, 32, false, true), 1);
      if (KIND == 15)
        tc::mma_bf16_ts_w(tmem + 256, tmem, tc::smem_desc(b + (i & 7) * 2048, 8192, 1024, tc::kSwizzle128B),
                          tc::idesc_bf16(128, 64, false, true), 1);
      if (KIND == 16)  // dV / dK of a 32-query block: N = 80, B MN-major 32-row tile
        tc::mma_bf16_ts_w(tmem + 256, tmem, tc::smem_desc(b + (i & 1) * 2048, 4096, 1024, tc::kSwizzle128B),
                          tc::idesc_bf16(128, 80, false, true), 1);
      if (KIND == 11) {  // wait-free group: 5 MMAs + commit + a TRYWAIT on an already-complete barrier
        for (int kk = 0; kk < 5; ++kk) tc::mma_bf16_ts_w(tmem + 256, tmem + 8 * kk, bd, tc::idesc_bf16(128, 64, false, false), 1);
        tc::mma_commit_w(&bar2[0]);
        tc::mbar_wait_w(&bar2[1], 0);  // phase 0 already completed
      }
      if (KIND == 5 || KIND == 6 || KIND == 12 || KIND == 13) {  // one dK/dV iteration: S^T (5 TS N=64), dP^T (5 TS N=64), dV+dK (8 TS N=80)
        const uint32_t is = tc::idesc_bf16(128, 64, false, false), ig = tc::idesc_bf16(128, 80, false, true);
        for (int kk = 0; kk < 5; ++kk) tc::mma_bf16_ts_w(tmem + (i % 3) * 64, tmem + 432 + 8 * kk, bd + 2 * kk, is, kk > 0);
        if (KIND == 6) tc::mma_commit_w(&bar2[0]);
        for (int kk = 0; kk < 5; ++kk) tc::mma_bf16_ts_w(tmem + 192, tmem + 472 + 8 * kk, bd + 2 * kk, is, kk > 0);
        if (KIND == 6) tc::mma_commit_w(&bar2[1]);
        for (int kk = 0; kk < 4; ++kk) {
          tc::mma_bf16_ts_w(tmem + 256, tmem + (i % 3) * 64 + 8 * kk, bmn + 128 * kk, ig, 1);
          tc::mma_bf16_ts_w(tmem + 352, tmem + (i % 3) * 64 + 16 + 8 * kk, bmn + 128 * kk, ig, 1);
        }
        if (KIND == 6) tc::mma_commit_w(&bar2[2]);
      }
    }
    tc::mma_commit_w(&bar);
    tc::mbar_wait(&bar, 0);
    unsigned long long t1 = clock64();
    if (threadIdx.x == 32) out[blockIdx.x] = t1 - t0;
    if (threadIdx.x == 32) stop_flag = 1;
  } else if (warp >= 4 && (KIND == 12 || KIND == 13)) {  // softmax-like TMEM traffic on columns [0, 192)
    const uint32_t lane_base = static_cast<uint32_t>((warp & 3) * 32) << 16;
    uint32_t acc = 0;
    int i = 0;
    while (!*(volatile int*)&stop_flag) {
      uint32_t r[32];
      tc::tmem_ld32(tmem + lane_base + ((i & 3) * 32), r);
      tc::tmem_ld_wait();
      if (KIND == 13) {
        uint32_t w[16];
        for (int k = 0; k < 16; ++k) w[k] = r[k] + r[k + 16];
        tc::tmem_st16(tmem + lane_base + 128 + (i & 3) * 16, w);
        tc::tmem_st_wait();
      }
      for (int k = 0; k < 32; ++k) acc += r[k];
      ++i;
    }
    if (acc == 0x1234567) out[1] = acc;
  }
  tc::tc_fence_before();
  __syncthreads();
  if (warp == 0) tc::tmem_dealloc(tmem, 512);
}

int main() {
  unsigned long long* d;
  uint32_t* sink;
  cudaMalloc(&d, 148 * 8);
  cudaMalloc(&sink, 4096);
  unsigned long long h[148];
  const int iters = 4096;
  for (int nw : {1, 4, 8}) {
    ld_bench<<<148, 384>>>(iters, nw, d, sink);
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = (double)h[0] / iters;
    printf("tcgen05.ld 32x32b.x32, %d warps: %.1f cycles per round -> %.1f B/cycle per SM\n", nw, cyc,
           nw * 4096.0 / cyc);
  }
  const char* names[] = {"SS 128x64x16", "TS 128x80x16 (A tmem, B MN-major)", "SS 128x128x16", "SS 128x256x16",
                         "TS 128x256x16", "dKV iteration (18 TS MMAs)", "dKV iteration + 3 commits", "TS 128x64x16",
                         "TS 128x32x16", "TS 128x16x16", "SS 128x32x16", "5xTS N64 + commit + completed wait",
                         "dKV iteration + 8 warps tcgen05.ld", "dKV iteration + 8 warps ld+st",
                         "TS 128x32x16 B MN-major SW64", "TS 128x64x16 B MN-major SW128", "TS 128x80x16 B MN 32-row"};
  const double fma[] = {128 * 64 * 16, 128 * 80 * 16, 128 * 128 * 16, 128 * 256 * 16, 128 * 256 * 16,
                        4.0 * 128 * 64 * 80, 4.0 * 128 * 64 * 80, 128 * 64 * 16, 128 * 32 * 16, 128 * 16 * 16,
                        128 * 32 * 16, 5.0 * 128 * 64 * 16, 4.0 * 128 * 64 * 80, 4.0 * 128 * 64 * 80,
                        128 * 32 * 16, 128 * 64 * 16, 128 * 80 * 16};
  for (int k = 0; k < 17; ++k) {
    void (*f)(int, unsigned long long*) = k == 0 ? mma_bench<0> : k == 1 ? mma_bench<1> : k == 2 ? mma_bench<2>
                                          : k == 3 ? mma_bench<3> : k == 4 ? mma_bench<4> : k == 5 ? mma_bench<5>
                                          : k == 6 ? mma_bench<6> : k == 7 ? mma_bench<7> : k == 8 ? mma_bench<8>
                                          : k == 9 ? mma_bench<9> : k == 10 ? mma_bench<10> : k == 11 ? mma_bench<11>
                                          : k == 12 ? mma_bench<12> : k == 13 ? mma_bench<13>
                                          : k == 14 ? mma_bench<14> : k == 15 ? mma_bench<15> : mma_bench<16>;
    const bool grp = k == 5 || k == 6 || k == 11 || k == 12 || k == 13;
    cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, 140000);
    f<<<148, 384, 140000>>>(grp ? iters / 8 : iters, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(h, d, sizeof(h), cudaMemcpyDeviceToHost);
    double cyc = (double)h[0] / (grp ? iters / 8 : iters);
    printf("%-36s %6.1f cycles/MMA  -> %.0f FMA/cycle/SM (%s)\n", names[k], cyc, fma[k] / cyc, cudaGetErrorString(e));
  }
  return 0;
}
