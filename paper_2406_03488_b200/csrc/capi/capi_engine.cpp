// extern "C" boundary of the execution engine (include/seqpipe_b200.h, sp_engine_*).
#include <cuda_runtime.h>
#include <nccl.h>

#include <cstring>
#include <vector>

#include "capi/capi_common.hpp"
#include "engine/comm_plan.hpp"
#include "engine/engine.hpp"
#include "seqpipe/json_io.hpp"
#include "seqpipe/render.hpp"
#include "seqpipe_b200.h"

struct sp_engine {
  std::unique_ptr<spe::Engine> impl;
};

struct sp_local_hub {
  std::shared_ptr<spe::LocalHub> impl;
};

namespace {

template <typename F>
int eguard(F&& f) {
  try {
    f();
    return SP_OK;
  } catch (const spk::CudaError& e) {
    spc::set_error(e.what());
    return SP_ERR_CUDA;
  } catch (const std::runtime_error& e) {
    const std::string w = e.what();
    if (w.rfind("NCCL", 0) == 0) {
      spc::set_error(w);
      return SP_ERR_NCCL;
    }
    return spc::map_exception();
  } catch (...) {
    return spc::map_exception();
  }
}

spe::ModelCfg model_from_c(const sp_model* m) {
  if (!m) throw std::invalid_argument("null model");
  spe::ModelCfg c;
  if (m->family != SP_MODEL_GPT && m->family != SP_MODEL_LLAMA) throw std::invalid_argument("unknown model family");
  if (m->dtype != SP_DTYPE_F32 && m->dtype != SP_DTYPE_BF16) throw std::invalid_argument("unknown dtype");
  c.family = m->family;
  c.dt = m->dtype == SP_DTYPE_F32 ? spk::DType::kF32 : spk::DType::kBF16;
  c.V = m->vocab;
  c.Vpad = (m->vocab + 127) / 128 * 128;
  c.h = m->hidden;
  c.L = m->layers;
  c.H = m->heads;
  c.hd = m->head_dim;
  c.F = m->ffn;
  c.Fup = m->family == SP_MODEL_LLAMA ? 2 * m->ffn : m->ffn;
  c.max_seq = m->max_seq;
  c.seed = m->seed;
  c.init_std = m->init_std;
  c.eps = m->norm_eps;
  c.theta = m->rope_theta;
  c.lr = m->lr;
  c.b1 = m->beta1;
  c.b2 = m->beta2;
  c.adam_eps = m->adam_eps;
  c.wd = m->weight_decay;
  c.flags = m->flags;
  if (c.V < 2 || c.h < 1 || c.L < 1 || c.H < 1 || c.hd < 1 || c.F < 1) throw std::invalid_argument("invalid model shape");
  if (c.h % 64 || c.F % 64) throw std::invalid_argument("hidden and ffn must be multiples of 64");
  if (c.hd % 8 || c.hd > 128) throw std::invalid_argument("head_dim must be a multiple of 8 and <= 128");
  return c;
}

spe::Engine& E(sp_engine* e) {
  if (!e || !e->impl) throw std::invalid_argument("null engine");
  return *e->impl;
}

}  // namespace

extern "C" {

int sp_engine_create(const sp_scenario* cfg, int32_t schedule_kind, const int64_t* lengths, const sp_model* model,
                     int32_t rank, int32_t world_size, int32_t cuda_device, sp_engine** out) {
  return eguard([&] {
    auto c = spc::from_c(cfg);
    auto part = spc::partition_from_c(c, lengths, c.segments);
    auto eng = std::make_unique<sp_engine>();
    eng->impl = std::make_unique<spe::Engine>(c, spc::kind_from_c(schedule_kind), part.lengths, model_from_c(model),
                                              rank, world_size, cuda_device);
    *out = eng.release();
  });
}

int sp_comm_plan(const sp_scenario* cfg, int32_t schedule_kind, const int64_t* lengths, int32_t device, int64_t hidden,
                 sp_comm_op* out, int64_t* n) {
  return eguard([&] {
    auto c = spc::from_c(cfg);
    auto part = spc::partition_from_c(c, lengths, c.segments);
    if (device < 1 || device > c.pipeline_size) throw std::out_of_range("device out of range");
    auto sch = seqpipe::generate(c, spc::kind_from_c(schedule_kind), part);
    auto plan = spe::comm_plan(sch, part.lengths, device, hidden);
    if (out) {
      if (*n < static_cast<int64_t>(plan.size())) throw spc::SpStatusError(SP_ERR_BUFFER_TOO_SMALL, "buffer too small");
      std::copy(plan.begin(), plan.end(), out);
    }
    *n = static_cast<int64_t>(plan.size());
  });
}

int sp_plan_memory(const sp_scenario* cfg, int32_t schedule_kind, const int64_t* lengths, const sp_model* model,
                   int32_t stage, double* live_peak_bytes, double* arena_bytes, double* dkv_bytes) {
  return eguard([&] {
    auto c = spc::from_c(cfg);
    auto part = spc::partition_from_c(c, lengths, c.segments);
    auto mc = model_from_c(model);
    if (stage < 1 || stage > c.total_stages()) throw std::out_of_range("stage out of range");
    if (mc.L % c.total_stages()) throw std::invalid_argument("model layers must divide evenly over the pipeline stages");
    auto sch = seqpipe::generate(c, spc::kind_from_c(schedule_kind), part);
    const int dev = (stage - 1) % c.pipeline_size;
    auto plan = spe::plan_stage_memory(mc, c, part.lengths, sch.device_orders[static_cast<size_t>(dev)], stage);
    if (live_peak_bytes) *live_peak_bytes = static_cast<double>(plan.live_peak);
    if (arena_bytes) *arena_bytes = static_cast<double>(plan.size());
    if (dkv_bytes) *dkv_bytes = static_cast<double>(mc.L / c.total_stages()) * c.seq_len * 2 * mc.h * 4;
  });
}

int sp_engine_destroy(sp_engine* eng) {
  return eguard([&] { delete eng; });
}

int sp_nccl_unique_id(uint8_t* out, size_t len) {
  return eguard([&] {
    ncclUniqueId id;
    if (len < sizeof(id)) throw std::invalid_argument("buffer smaller than NCCL_UNIQUE_ID_BYTES");
    ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL: ") + ncclGetErrorString(r));
    std::memcpy(out, &id, sizeof(id));
  });
}

int sp_engine_comm_init(sp_engine* eng, const uint8_t* const* ids, int32_t n_ids) {
  return eguard([&] {
    std::vector<std::string> v;
    for (int i = 0; i < n_ids; ++i) v.emplace_back(reinterpret_cast<const char*>(ids[i]), sizeof(ncclUniqueId));
    E(eng).comm_init(v);
  });
}

int sp_engine_ipc_export(sp_engine* eng, uint8_t* out, size_t* len) {
  return eguard([&] {
    if (!len) throw std::invalid_argument("null length");
    const std::string b = E(eng).ipc_export();
    if (out) {
      if (*len < b.size()) {
        *len = b.size();
        throw spc::SpStatusError(SP_ERR_BUFFER_TOO_SMALL, "ipc blob needs " + std::to_string(b.size()) + " bytes");
      }
      std::memcpy(out, b.data(), b.size());
    }
    *len = b.size();
  });
}

int sp_engine_ipc_connect(sp_engine* eng, const uint8_t* const* blobs, const size_t* lens, int32_t n) {
  return eguard([&] {
    if (n < 0 || (n > 0 && (!blobs || !lens))) throw std::invalid_argument("null blobs");
    std::vector<std::string> v;
    for (int32_t i = 0; i < n; ++i) v.emplace_back(reinterpret_cast<const char*>(blobs[i]), lens[i]);
    E(eng).ipc_connect(v);
  });
}

int sp_engine_comm_channels(sp_engine* eng, int32_t* n) {
  return eguard([&] { *n = E(eng).comm_channels(); });
}

int sp_local_hub_create(int32_t world_size, double watchdog_seconds, sp_local_hub** out) {
  return eguard([&] {
    if (!out) throw std::invalid_argument("null output");
    auto h = std::make_unique<sp_local_hub>();
    h->impl = spe::make_local_hub(world_size, watchdog_seconds > 0 ? watchdog_seconds : 600.0);
    *out = h.release();
  });
}

int sp_local_hub_destroy(sp_local_hub* hub) {
  delete hub;
  return SP_OK;
}

int sp_engine_attach_local(sp_engine* eng, sp_local_hub* hub) {
  return eguard([&] {
    if (!hub || !hub->impl) throw std::invalid_argument("null hub");
    E(eng).attach_local(hub->impl);
  });
}

int sp_engine_enable_graph(sp_engine* eng, int32_t on) {
  return eguard([&] { E(eng).enable_graph(on != 0); });
}

int sp_engine_set_flags(sp_engine* eng, int32_t flags) {
  return eguard([&] { E(eng).set_flags(flags); });
}

int sp_engine_step(sp_engine* eng, const int32_t* tokens, int32_t tokens_on_device, sp_step_report* report) {
  return eguard([&] { E(eng).step(tokens, tokens_on_device != 0, report); });
}

int sp_engine_op_log(sp_engine* eng, sp_task* ops, int64_t* counts) {
  return eguard([&] {
    auto by_dev = E(eng).op_log_by_device();
    size_t off = 0;
    for (size_t d = 0; d < by_dev.size(); ++d) {
      counts[d] = static_cast<int64_t>(by_dev[d].size());
      if (ops)
        for (const auto& t : by_dev[d]) ops[off++] = spc::to_c(t);
    }
  });
}

int sp_engine_timeline(sp_engine* eng, double* start_ms, double* end_ms, int64_t* n) {
  return eguard([&] {
    const auto& a = E(eng).t_start();
    const auto& b = E(eng).t_end();
    if (!start_ms || *n < static_cast<int64_t>(a.size())) {
      *n = static_cast<int64_t>(a.size());
      return;
    }
    std::copy(a.begin(), a.end(), start_ms);
    std::copy(b.begin(), b.end(), end_ms);
    *n = static_cast<int64_t>(a.size());
  });
}

int sp_engine_report_json(sp_engine* eng, int32_t indent, int64_t memory_downsample, char* buf, size_t* len) {
  return eguard([&] {
    const std::string text = seqpipe::report_to_json(E(eng).measured_report(), indent,
                                                     static_cast<std::size_t>(memory_downsample < 0 ? 0 : memory_downsample));
    if (!len) throw std::invalid_argument("null length");
    const size_t need = text.size() + 1;
    if (!buf || *len < need) {
      *len = need;
      if (buf) throw std::length_error("buffer too small");
      return;
    }
    std::memcpy(buf, text.c_str(), need);
    *len = need;
  });
}

int sp_engine_render_gantt(sp_engine* eng, int32_t format, int32_t width, char* buf, size_t* len) {
  return eguard([&] {
    if (format != SP_RENDER_ASCII && format != SP_RENDER_SVG) throw std::invalid_argument("unknown render format");
    const seqpipe::SimReport rep = E(eng).measured_report();
    const std::string text =
        format == SP_RENDER_SVG ? seqpipe::render_svg_gantt(rep) : seqpipe::render_ascii_gantt(rep, width);
    if (!len) throw std::invalid_argument("null length");
    const size_t need = text.size() + 1;
    if (!buf || *len < need) {
      *len = need;
      if (buf) throw std::length_error("buffer too small");
      return;
    }
    std::memcpy(buf, text.c_str(), need);
    *len = need;
  });
}

int sp_engine_param_count(sp_engine* eng, int64_t* n) {
  return eguard([&] { *n = static_cast<int64_t>(E(eng).all_params().size()); });
}

int sp_engine_param_info(sp_engine* eng, int64_t idx, char* name, size_t name_len, int64_t* numel, int32_t* rows,
                         int32_t* cols) {
  return eguard([&] {
    auto all = E(eng).all_params();
    if (idx < 0 || idx >= static_cast<int64_t>(all.size())) throw std::out_of_range("param index out of range");
    const spe::Param& p = all[static_cast<size_t>(idx)].second;
    if (name && name_len) {
      std::strncpy(name, p.name.c_str(), name_len - 1);
      name[name_len - 1] = 0;
    }
    const int32_t r = p.rows;  // lm_head reports its padded row count (vocab rounded up to 128)
    if (numel) *numel = static_cast<int64_t>(r) * p.cols;
    if (rows) *rows = r;
    if (cols) *cols = p.cols;
  });
}

static void copy_param(sp_engine* eng, const char* name, float* host, int64_t numel, bool grad, bool write) {
  spe::Param p;
  spe::Stage* st = E(eng).stage_for_param(name ? name : "", &p);
  if (!st) throw std::invalid_argument(std::string("unknown parameter '") + (name ? name : "") + "'");
  if (numel > p.numel) throw std::invalid_argument("numel exceeds parameter size");
  SPK_CUDA(cudaSetDevice(E(eng).device()));
  SPK_CUDA(cudaDeviceSynchronize());
  float* dev = (grad ? st->grads() : st->master()) + p.off;
  if (write) {
    SPK_CUDA(cudaMemcpy(dev, host, sizeof(float) * numel, cudaMemcpyHostToDevice));
    st->sync_compute();
  } else {
    SPK_CUDA(cudaMemcpy(host, dev, sizeof(float) * numel, cudaMemcpyDeviceToHost));
  }
}

int sp_engine_read_param(sp_engine* eng, const char* name, float* out, int64_t numel) {
  return eguard([&] { copy_param(eng, name, out, numel, false, false); });
}
int sp_engine_read_grad(sp_engine* eng, const char* name, float* out, int64_t numel) {
  return eguard([&] { copy_param(eng, name, out, numel, true, false); });
}
int sp_engine_write_param(sp_engine* eng, const char* name, const float* in, int64_t numel) {
  return eguard([&] { copy_param(eng, name, const_cast<float*>(in), numel, false, true); });
}

int sp_engine_memory(sp_engine* eng, double* allocated_bytes, double* device_free_bytes) {
  return eguard([&] {
    SPK_CUDA(cudaSetDevice(E(eng).device()));
    size_t fr = 0, tot = 0;
    SPK_CUDA(cudaMemGetInfo(&fr, &tot));
    if (allocated_bytes) *allocated_bytes = static_cast<double>(tot - fr);
    if (device_free_bytes) *device_free_bytes = static_cast<double>(fr);
  });
}

}  // extern "C"
