// GPU-resident launcher core: the computation-wise partition and the per-device
// op tables are produced by device kernels, so a stage's whole schedule can be
// materialised (and captured into a CUDA graph) without host planning work.
//
// cwp: same double-precision bisection as the reference
// (/root/reference/proj/core/src/partition.cpp:100-207), written with explicit
// round-to-nearest intrinsics so no FMA contraction can change a bit.
// Op tables: closed form of the gpipe / 1f1b / seq1f1b device orders
// (schedule.cpp:68-126), identical to seqpipe::op_at on the host.
#include <cuda.h>

#include <mutex>
#include <set>
#include <vector>

#include "capi/capi_common.hpp"
#include "cuda/common.cuh"
#include "seqpipe/partition.hpp"
#include "seqpipe/schedule.hpp"
#include "cuda/ops.h"
#include "seqpipe_b200.h"

namespace spk {
namespace {

constexpr int kMaxSegments = 256;

struct CwpIn {
  int k;
  int64_t n;
  double layers, hidden, params;
};

__device__ void cwp_lengths(const CwpIn& c, double target, double* x) {
  const double a = __dmul_rn(__dmul_rn(2.0, c.layers), c.hidden);
  double prefix = 0.0;
  for (int i = 0; i < c.k; ++i) {
    const double b = __dadd_rn(__dmul_rn(2.0, c.params), __dmul_rn(a, prefix));
    double xi;
    if (a == 0.0) {
      xi = __ddiv_rn(target, b);
    } else {
      const double disc = __dadd_rn(__dmul_rn(b, b), __dmul_rn(__dmul_rn(4.0, a), target));
      xi = __ddiv_rn(__dadd_rn(-b, __dsqrt_rn(disc)), __dmul_rn(2.0, a));
    }
    x[i] = xi;
    prefix = __dadd_rn(prefix, xi);
  }
}

// Single-thread kernel: the solve is latency-bound and tiny (k <= 256).
__global__ void cwp_kernel(CwpIn c, int64_t* out, int* status) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  double x[kMaxSegments];
  const double nd = static_cast<double>(c.n);
  double lo = 0.0;
  const double hi0 = __dadd_rn(__dmul_rn(__dmul_rn(2.0, nd), c.params),
                               __dmul_rn(__dmul_rn(__dmul_rn(__dmul_rn(2.0, c.layers), nd), nd), c.hidden));
  double hi = hi0, mid = hi0;
  for (int it = 0; it < 200; ++it) {
    mid = __dmul_rn(0.5, __dadd_rn(lo, hi));
    cwp_lengths(c, mid, x);
    double total = 0.0;
    for (int i = 0; i < c.k; ++i) total = __dadd_rn(total, x[i]);
    if (fabs(__dadd_rn(total, -nd)) <= __dmul_rn(1e-6, nd)) break;
    if (total < nd)
      lo = mid;
    else
      hi = mid;
  }
  cwp_lengths(c, mid, x);
  // Largest-remainder rounding, ties to the earliest segment (stable order).
  int64_t len[kMaxSegments];
  double rem[kMaxSegments];
  int order[kMaxSegments];
  int64_t assigned = 0;
  for (int i = 0; i < c.k; ++i) {
    const double cl = x[i] > 0.0 ? x[i] : 0.0;
    len[i] = static_cast<int64_t>(floor(cl));
    rem[i] = __dadd_rn(cl, -static_cast<double>(len[i]));
    assigned += len[i];
    order[i] = i;
  }
  for (int i = 1; i < c.k; ++i) {  // stable insertion sort by remainder, descending
    const int v = order[i];
    int j = i - 1;
    while (j >= 0 && rem[order[j]] < rem[v]) {
      order[j + 1] = order[j];
      --j;
    }
    order[j + 1] = v;
  }
  int64_t left = c.n - assigned;
  int64_t turn = 0;
  for (; left > 0; --left, ++turn) len[order[turn % c.k]] += 1;
  while (left < 0) {
    const int victim = order[c.k - 1 - (turn % c.k)];
    if (len[victim] > 0) {
      len[victim] -= 1;
      ++left;
    }
    ++turn;
  }
  for (int i = 0; i < c.k; ++i) {
    while (len[i] < 1) {
      int big = 0;
      for (int j = 1; j < c.k; ++j)
        if (len[j] > len[big]) big = j;
      if (len[big] <= 1) {
        *status = 1;
        return;
      }
      len[big] -= 1;
      len[i] += 1;
    }
  }
  for (int i = 0; i < c.k; ++i) out[i] = len[i];
  *status = 0;
}

struct OpShape {
  int P, M, k;
  int seq_level, gpipe, bwd_kind;
};

// One thread per (device, position): the closed-form op table.
__global__ void op_table_kernel(OpShape s, sp_task* out) {
  const int per_dev = 2 * s.M * s.k;
  const int64_t total = static_cast<int64_t>(per_dev) * s.P;
  for (int64_t g = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; g < total; g += (int64_t)gridDim.x * blockDim.x) {
    const int d = static_cast<int>(g / per_dev) + 1;
    const int j = static_cast<int>(g % per_dev);
    const int U = s.seq_level ? s.M * s.k : s.M;
    const int per_unit = s.seq_level ? 1 : s.k;
    int w = U;
    if (!s.gpipe && s.M > s.P) w = s.seq_level ? s.P - d - 1 + s.k : s.P - d;
    if (w > U) w = U;
    const int u = j / per_unit, q = j % per_unit;
    bool fwd;
    int idx;
    if (u < w) {
      fwd = true;
      idx = u;
    } else if (u < 2 * U - w) {
      const int r = u - w;
      fwd = (r % 2) == 0;
      idx = fwd ? w + r / 2 : r / 2;
    } else {
      fwd = false;
      idx = u - U;
    }
    sp_task t;
    t.kind = fwd ? SP_TASK_F : s.bwd_kind;
    if (s.seq_level) {
      t.micro_batch = idx / s.k + 1;
      t.segment = fwd ? idx % s.k + 1 : s.k - idx % s.k;
    } else {
      t.micro_batch = idx + 1;
      t.segment = fwd ? q + 1 : s.k - q;
    }
    t.stage = d;
    t.device = d;
    out[g] = t;
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    SPK_CUDA(cudaGetDevice(&prev));
    SPK_CUDA(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

std::vector<int64_t> device_cwp(const seqpipe::ScenarioConfig& cfg, int dev) {
  if (cfg.seq_len < cfg.segments) throw std::invalid_argument("seq_len must be >= segments");
  if (std::int64_t(cfg.layers) * cfg.hidden_dim == 0 && cfg.param_count == 0)
    throw std::domain_error("cannot balance segments under an all-zero cost model");
  if (cfg.segments > kMaxSegments) throw std::invalid_argument("device cwp supports at most 256 segments");
  if (cfg.segments == 1) return {cfg.seq_len};
  DeviceGuard g(dev);
  CwpIn in{cfg.segments, cfg.seq_len, static_cast<double>(cfg.layers), static_cast<double>(cfg.hidden_dim),
           static_cast<double>(cfg.param_count)};
  int64_t* d_out = nullptr;
  int* d_status = nullptr;
  SPK_CUDA(cudaMalloc(&d_out, sizeof(int64_t) * cfg.segments));
  SPK_CUDA(cudaMalloc(&d_status, sizeof(int)));
  cwp_kernel<<<1, 32>>>(in, d_out, d_status);
  std::vector<int64_t> out(static_cast<size_t>(cfg.segments));
  int status = 0;
  cudaError_t e1 = cudaMemcpy(out.data(), d_out, sizeof(int64_t) * cfg.segments, cudaMemcpyDeviceToHost);
  cudaError_t e2 = cudaMemcpy(&status, d_status, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(d_out);
  cudaFree(d_status);
  SPK_CUDA(e1);
  SPK_CUDA(e2);
  if (status) throw std::logic_error("cannot repair degenerate partition");
  return out;
}

std::vector<sp_task> device_op_table(const seqpipe::ScenarioConfig& cfg, seqpipe::ScheduleKind kind, int dev) {
  using seqpipe::ScheduleKind;
  cfg.validate();
  if (seqpipe::is_interleaved(kind) || seqpipe::is_zero_bubble(kind))
    throw seqpipe::UnsupportedScheduleError("device op tables cover gpipe, 1f1b and seq1f1b");
  if (cfg.stages_per_device != 1)
    throw seqpipe::UnsupportedScheduleError(std::string(seqpipe::schedule_kind_name(kind)) +
                                            " requires stages_per_device == 1");
  DeviceGuard g(dev);
  OpShape s{cfg.pipeline_size, cfg.micro_batches, cfg.segments, seqpipe::is_sequence_level(kind) ? 1 : 0,
            kind == ScheduleKind::kGPipe ? 1 : 0, SP_TASK_B};
  const int64_t total = static_cast<int64_t>(2) * cfg.micro_batches * cfg.segments * cfg.pipeline_size;
  sp_task* d_out = nullptr;
  SPK_CUDA(cudaMalloc(&d_out, sizeof(sp_task) * total));
  const int blocks = static_cast<int>((total + 255) / 256 < 1024 ? (total + 255) / 256 : 1024);
  op_table_kernel<<<blocks, 256>>>(s, d_out);
  std::vector<sp_task> out(static_cast<size_t>(total));
  cudaError_t e1 = cudaGetLastError();
  cudaError_t e2 = cudaMemcpy(out.data(), d_out, sizeof(sp_task) * total, cudaMemcpyDeviceToHost);
  cudaFree(d_out);
  SPK_CUDA(e1);
  SPK_CUDA(e2);
  return out;
}

namespace {

template <typename F>
F driver_fn(const char* name) {
  void* f = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint(name, &f, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
    throw CudaError(std::string("driver entry point unavailable: ") + name);
  return reinterpret_cast<F>(f);
}

void preload_module_of(const void* anchor) {
  using GetLibrary = CUresult (*)(CUlibrary*, CUkernel);
  using KernelCount = CUresult (*)(unsigned int*, CUlibrary);
  using Enumerate = CUresult (*)(CUkernel*, unsigned int, CUlibrary);
  using GetFunction = CUresult (*)(CUfunction*, CUkernel);
  static const auto get_library = driver_fn<GetLibrary>("cuKernelGetLibrary");
  static const auto kernel_count = driver_fn<KernelCount>("cuLibraryGetKernelCount");
  static const auto enumerate = driver_fn<Enumerate>("cuLibraryEnumerateKernels");
  static const auto get_function = driver_fn<GetFunction>("cuKernelGetFunction");
  cudaKernel_t k = nullptr;
  SPK_CUDA(cudaGetKernel(&k, anchor));
  CUlibrary lib = nullptr;
  unsigned int n = 0;
  auto ok = [](CUresult r, const char* what) {
    if (r != CUDA_SUCCESS) throw CudaError(std::string(what) + " failed: " + std::to_string(static_cast<int>(r)));
  };
  ok(get_library(&lib, reinterpret_cast<CUkernel>(k)), "cuKernelGetLibrary");
  ok(kernel_count(&n, lib), "cuLibraryGetKernelCount");
  std::vector<CUkernel> ks(n);
  ok(enumerate(ks.data(), n, lib), "cuLibraryEnumerateKernels");
  for (CUkernel kk : ks) {
    CUfunction f = nullptr;
    ok(get_function(&f, kk), "cuKernelGetFunction");  // loads it into the current context
  }
}

}  // namespace

void preload_kernels() {
  static std::mutex mu;
  static std::set<int> done;  // devices whose context holds every kernel
  int dev = 0;
  SPK_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  if (done.count(dev)) return;
  for (const void* a : {module_anchor_attention_simt(), module_anchor_attention_tc(), module_anchor_elementwise(),
                        module_anchor_gemm_simt(), module_anchor_gemm_tcgen05(),
                        reinterpret_cast<const void*>(&cwp_kernel)})
    preload_module_of(a);
  done.insert(dev);
}

}  // namespace spk

extern "C" int sp_device_partition(const sp_scenario* cfg, int32_t mode, int32_t cuda_device, int64_t* lengths_out) {
  SP_GUARD({
    auto c = spc::from_c(cfg);
    std::vector<int64_t> len;
    if (mode == SP_PART_CWP) {
      len = spk::device_cwp(c, cuda_device);
    } else if (mode == SP_PART_EVEN) {
      len = seqpipe::even_partition(c).lengths;  // integer split: no device work worth a launch
    } else {
      throw std::invalid_argument("device partition supports even and cwp");
    }
    seqpipe::make_partition(len, c);  // same validation as the host path
    std::copy(len.begin(), len.end(), lengths_out);
  });
}

extern "C" int sp_device_schedule_ops(const sp_scenario* cfg, int32_t kind, int32_t cuda_device, sp_task* ops,
                                      int64_t* counts) {
  SP_GUARD({
    auto c = spc::from_c(cfg);
    auto table = spk::device_op_table(c, spc::kind_from_c(kind), cuda_device);
    const int64_t per = 2LL * c.micro_batches * c.segments;
    for (int d = 0; d < c.pipeline_size; ++d) counts[d] = per;
    std::copy(table.begin(), table.end(), ops);
  });
}
