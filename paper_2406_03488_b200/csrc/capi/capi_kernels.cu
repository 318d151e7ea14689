// extern "C" kernel-level entry points (tests, microbenchmarks, bench roofline).
#include "capi/capi_common.hpp"
#include "cuda/common.cuh"
#include "cuda/ops.h"
#include "seqpipe_b200.h"

namespace {
spk::DType dt(int32_t d) {
  if (d != SP_DTYPE_F32 && d != SP_DTYPE_BF16) throw std::invalid_argument("dtype must be SP_DTYPE_F32 or SP_DTYPE_BF16");
  return d == SP_DTYPE_F32 ? spk::DType::kF32 : spk::DType::kBF16;
}

template <typename F>
int cuda_guard(F&& f) {
  try {
    f();
    return SP_OK;
  } catch (const spk::CudaError& e) {
    spc::set_error(e.what());
    return SP_ERR_CUDA;
  } catch (...) {
    return spc::map_exception();
  }
}
}  // namespace

extern "C" {

int sp_gemm(int32_t dtype, int32_t impl, const void* A, int32_t a_kmajor, const void* B, int32_t b_kmajor, void* C,
            int32_t c_f32, int32_t accumulate, int64_t M, int64_t N, int64_t K, void* stream) {
  return cuda_guard([&] {
    spk::GemmArgs g;
    g.M = M;
    g.N = N;
    g.K = K;
    g.ab = dt(dtype);
    g.A = A;
    g.a_kmajor = a_kmajor != 0;
    g.lda = a_kmajor ? K : M;
    g.B = B;
    g.b_kmajor = b_kmajor != 0;
    g.ldb = b_kmajor ? K : N;
    g.C = C;
    g.ldc = N;
    g.c = c_f32 ? spk::DType::kF32 : g.ab;
    if (accumulate) {
      if (!c_f32) throw std::invalid_argument("accumulate requires an fp32 C");
      g.epi = spk::Epi::kAccumF32;
    }
    if (impl == spk::kGemmTcgen05 && !spk::gemm_tc_supported(g))
      throw std::invalid_argument("tcgen05 GEMM does not support these operands");
    spk::gemm(g, static_cast<cudaStream_t>(stream), impl);
  });
}

int sp_attention_fwd(int32_t dtype, int32_t impl, const void* q, const void* kv, void* o, float* lse, int64_t n,
                     int64_t q_off, int64_t kv_len, int32_t heads, int32_t head_dim, void* stream) {
  return cuda_guard([&] {
    spk::attn_fwd(dt(dtype), impl, q, kv, o, lse, n, q_off, kv_len, heads, head_dim, static_cast<cudaStream_t>(stream));
  });
}

int sp_attention_bwd(int32_t dtype, int32_t impl, const void* q, const void* kv, const void* o, const void* dout,
                     const float* lse, void* dq, float* dkv_acc, int64_t n, int64_t q_off, int64_t kv_len, int32_t heads,
                     int32_t head_dim, void* stream) {
  return cuda_guard([&] {
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    // Workspace cached per device and grown on demand (a per-call cudaMallocAsync /
    // cudaFreeAsync pair returns memory to the driver at every sync and distorts timing).
    static thread_local float* ws_buf[64] = {};
    static thread_local size_t ws_cap[64] = {};
    int dev = 0;
    SPK_CUDA(cudaGetDevice(&dev));
    const size_t floats = spk::attn_bwd_ws_delta_floats(n, heads) + static_cast<size_t>(n) * heads * head_dim;
    if (dev < 0 || dev >= 64) throw std::invalid_argument("device ordinal out of range");
    if (ws_cap[dev] < floats) {
      if (ws_buf[dev]) SPK_CUDA(cudaFree(ws_buf[dev]));
      SPK_CUDA(cudaMalloc(&ws_buf[dev], floats * sizeof(float)));
      ws_cap[dev] = floats;
    }
    float* ws = ws_buf[dev];
    spk::attn_bwd(dt(dtype), impl, q, kv, o, dout, lse, ws, ws + spk::attn_bwd_ws_delta_floats(n, heads), dq, dkv_acc, n, q_off,
                  kv_len, heads, head_dim, s);
  });
}

int sp_norm_fwd(int32_t dtype, int32_t rms, const void* x, const float* g, void* y, float* mean, float* rstd,
                int64_t n, int32_t h, float eps, void* stream) {
  return cuda_guard([&] {
    spk::norm_fwd(dt(dtype), rms != 0, x, g, y, mean, rstd, n, h, eps, static_cast<cudaStream_t>(stream));
  });
}

int sp_norm_bwd(int32_t dtype, int32_t rms, const void* dy, const void* x, const float* g, const float* mean,
                const float* rstd, const void* dres, void* dx, float* dg, int64_t n, int32_t h, void* stream) {
  return cuda_guard([&] {
    spk::norm_bwd(dt(dtype), rms != 0, dy, x, g, mean, rstd, dres, dx, dg, n, h, static_cast<cudaStream_t>(stream));
  });
}

int sp_act_fwd(int32_t dtype, int32_t family, const void* u, void* out, int64_t n, int32_t F, void* stream) {
  return cuda_guard([&] { spk::act_fwd(dt(dtype), family, u, out, n, F, static_cast<cudaStream_t>(stream)); });
}

int sp_act_bwd(int32_t dtype, int32_t family, const void* u, const void* dout, void* du, int64_t n, int32_t F,
               void* stream) {
  return cuda_guard([&] { spk::act_bwd(dt(dtype), family, u, dout, du, n, F, static_cast<cudaStream_t>(stream)); });
}

int sp_device_synchronize(int32_t cuda_device) {
  return cuda_guard([&] {
    SPK_CUDA(cudaSetDevice(cuda_device));
    SPK_CUDA(cudaDeviceSynchronize());
  });
}

int sp_cuda_device_count(int32_t* n) {
  return cuda_guard([&] {
    int c = 0;
    cudaError_t e = cudaGetDeviceCount(&c);
    *n = e == cudaSuccess ? c : 0;
  });
}

}  // extern "C"
