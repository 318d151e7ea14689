// L2 reduction throughput on sm_100a: how fast can 148 SMs add fp32 partial
// sums into a global accumulator that stays L2-resident? (Sizing the dQ
// reduction of a fused attention backward: one [64 x hd] fp32 partial per
// (key block, query block) pair.)
//   0: red.global.add.f32, one warp = 128 contiguous bytes per instruction
//   1: red.global.add.v4.f32, one warp = 512 contiguous bytes per instruction
//   2: cp.reduce.async.bulk (TMA bulk add.f32) of a 20 KB SMEM tile
//   3: plain st.global.v4 (reference point: write bandwidth to L2)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_bench red_bench.cu
#include <cstdint>
#include <cstdio>

constexpr int TILE_FLOATS = 64 * 80;  // one [64 q x 80] fp32 partial (20 KB)

template <int KIND>
__global__ void __launch_bounds__(256) red_k(float* acc, int64_t acc_tiles, int iters) {
  extern __shared__ __align__(128) float stile[];
  for (int i = threadIdx.x; i < TILE_FLOATS; i += blockDim.x) stile[i] = 1e-6f * i;
  __syncthreads();
  uint32_t seed = blockIdx.x * 2654435761u;
  for (int it = 0; it < iters; ++it) {
    seed = seed * 1664525u + 1013904223u;
    float* dst = acc + static_cast<int64_t>((seed >> 8) % acc_tiles) * TILE_FLOATS;
    if (KIND == 0) {
      for (int i = threadIdx.x; i < TILE_FLOATS; i += blockDim.x)
        asm volatile("red.global.add.f32 [%0], %1;" ::"l"(dst + i), "f"(stile[i]) : "memory");
    } else if (KIND == 1) {
      for (int i = threadIdx.x * 4; i < TILE_FLOATS; i += blockDim.x * 4)
        asm volatile("red.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + i), "f"(stile[i]), "f"(stile[i + 1]),
                     "f"(stile[i + 2]), "f"(stile[i + 3])
                     : "memory");
    } else if (KIND == 2) {
      if (threadIdx.x == 0) {
        asm volatile(
            "cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
            "r"(static_cast<uint32_t>(__cvta_generic_to_shared(stile))), "r"(TILE_FLOATS * 4)
            : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        asm volatile("cp.async.bulk.wait_group.read 4;" ::: "memory");
      }
    } else {
      for (int i = threadIdx.x * 4; i < TILE_FLOATS; i += blockDim.x * 4)
        *reinterpret_cast<float4*>(dst + i) = *reinterpret_cast<float4*>(stile + i);
    }
  }
  if (KIND == 2 && threadIdx.x == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int KIND>
void run(const char* name, float* acc, int64_t tiles, int ctas, int threads) {
  const int iters = 400;
  cudaFuncSetAttribute(red_k<KIND>, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_FLOATS * 4);
  red_k<KIND><<<ctas, threads, TILE_FLOATS * 4>>>(acc, tiles, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  red_k<KIND><<<ctas, threads, TILE_FLOATS * 4>>>(acc, tiles, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double bytes = static_cast<double>(ctas) * iters * TILE_FLOATS * 4;
  printf("%-44s ctas %4d x %3d thr: %8.1f GB/s of fp32 partials (%s)\n", name, ctas, threads, bytes / ms / 1e6,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const int64_t tiles = (48ll << 20) / (TILE_FLOATS * 4);  // 48 MB accumulator: L2-resident
  float* acc;
  cudaMalloc(&acc, tiles * TILE_FLOATS * 4);
  cudaMemset(acc, 0, tiles * TILE_FLOATS * 4);
  for (int per_sm : {1, 2}) {
    const int ctas = 148 * per_sm;
    run<0>("red.global.add.f32 (128 B / warp-instr)", acc, tiles, ctas, 128);
    run<1>("red.global.add.v4.f32 (512 B / warp-instr)", acc, tiles, ctas, 128);
    run<2>("cp.reduce.async.bulk add.f32 (20 KB tile)", acc, tiles, ctas, 32);
    run<3>("st.global.v4 (write, no reduction)", acc, tiles, ctas, 128);
  }
  return 0;
}
