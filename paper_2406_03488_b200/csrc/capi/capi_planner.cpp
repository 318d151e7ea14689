// extern "C" boundary for the planner (include/seqpipe_b200.h). Exceptions never
// cross it: every entry point maps the seqpipe exception type to an SP_ERR_*
// code and stores the message for sp_last_error().
#include <cstring>
#include <string>

#include "capi_common.hpp"
#include "seqpipe/cost.hpp"
#include "seqpipe/partition.hpp"
#include "seqpipe/scenario.hpp"
#include "seqpipe/schedule.hpp"
#include "seqpipe/json_io.hpp"
#include "seqpipe/render.hpp"
#include "seqpipe/sim.hpp"
#include "seqpipe/validate.hpp"
#include "seqpipe_b200.h"

namespace spc {

thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }

int map_exception() {
  try {
    throw;
  } catch (const seqpipe::UnsupportedScheduleError& e) {
    set_error(e.what());
    return SP_ERR_UNSUPPORTED;
  } catch (const seqpipe::DeadlockError& e) {
    set_error(e.what());
    return SP_ERR_DEADLOCK;
  } catch (const seqpipe::MissingDependencyError& e) {
    set_error(e.what());
    return SP_ERR_MISSING_DEPENDENCY;
  } catch (const SpStatusError& e) {
    set_error(e.what());
    return e.code;
  } catch (const std::out_of_range& e) {
    set_error(e.what());
    return SP_ERR_OUT_OF_RANGE;
  } catch (const std::invalid_argument& e) {
    set_error(e.what());
    return SP_ERR_INVALID_ARGUMENT;
  } catch (const std::domain_error& e) {
    set_error(e.what());
    return SP_ERR_DOMAIN;
  } catch (const std::overflow_error& e) {
    set_error(e.what());
    return SP_ERR_OVERFLOW;
  } catch (const std::logic_error& e) {
    set_error(e.what());
    return SP_ERR_LOGIC;
  } catch (const std::exception& e) {
    set_error(e.what());
    return SP_ERR_RUNTIME;
  } catch (...) {
    set_error("unknown exception");
    return SP_ERR_RUNTIME;
  }
}

seqpipe::Rational from_c(const sp_rational& r) { return seqpipe::Rational(r.num, r.den); }
sp_rational to_c(const seqpipe::Rational& r) { return sp_rational{r.numerator(), r.denominator()}; }

seqpipe::ScenarioConfig from_c(const sp_scenario* c) {
  if (!c) throw std::invalid_argument("null scenario");
  seqpipe::ScenarioConfig s;
  s.pipeline_size = c->pipeline_size;
  s.stages_per_device = c->stages_per_device;
  s.micro_batches = c->micro_batches;
  s.segments = c->segments;
  s.seq_len = c->seq_len;
  s.layers = c->layers;
  s.hidden_dim = c->hidden_dim;
  s.param_count = c->param_count;
  s.backward_ratio = from_c(c->backward_ratio);
  s.bw_input_ratio = from_c(c->bw_input_ratio);
  s.bw_weight_ratio = from_c(c->bw_weight_ratio);
  s.comm_latency = from_c(c->comm_latency);
  s.activation_cost_per_token = from_c(c->activation_cost_per_token);
  s.time_per_flop = from_c(c->time_per_flop);
  s.cost_model = c->cost_model == SP_COST_UNIFORM ? seqpipe::CostModel::kUniform : seqpipe::CostModel::kFlops;
  s.uniform_forward = from_c(c->uniform_forward);
  return s;
}

void to_c(const seqpipe::ScenarioConfig& s, sp_scenario* c) {
  c->pipeline_size = s.pipeline_size;
  c->stages_per_device = s.stages_per_device;
  c->micro_batches = s.micro_batches;
  c->segments = s.segments;
  c->seq_len = s.seq_len;
  c->layers = s.layers;
  c->hidden_dim = s.hidden_dim;
  c->param_count = s.param_count;
  c->backward_ratio = to_c(s.backward_ratio);
  c->bw_input_ratio = to_c(s.bw_input_ratio);
  c->bw_weight_ratio = to_c(s.bw_weight_ratio);
  c->comm_latency = to_c(s.comm_latency);
  c->activation_cost_per_token = to_c(s.activation_cost_per_token);
  c->time_per_flop = to_c(s.time_per_flop);
  c->cost_model = s.cost_model == seqpipe::CostModel::kUniform ? SP_COST_UNIFORM : SP_COST_FLOPS;
  c->uniform_forward = to_c(s.uniform_forward);
}

seqpipe::Task from_c(const sp_task& t) {
  if (t.kind < 0 || t.kind > 3) throw std::invalid_argument("task kind out of range");
  return seqpipe::Task{static_cast<seqpipe::TaskKind>(t.kind), t.micro_batch, t.segment, t.stage, t.device};
}
sp_task to_c(const seqpipe::Task& t) {
  return sp_task{static_cast<int32_t>(t.kind), t.micro_batch, t.segment, t.stage, t.device};
}

seqpipe::ScheduleKind kind_from_c(int32_t k) {
  if (k < 0 || k > 6) throw std::invalid_argument("schedule kind out of range");
  return static_cast<seqpipe::ScheduleKind>(k);
}

seqpipe::SequencePartition partition_from_c(const seqpipe::ScenarioConfig& cfg, const int64_t* lengths, int k) {
  if (!lengths || k < 1) throw std::invalid_argument("null/empty partition");
  return seqpipe::make_partition(std::vector<std::int64_t>(lengths, lengths + k), cfg);
}

seqpipe::Schedule schedule_from_c(const seqpipe::ScenarioConfig& cfg, int32_t kind, const sp_task* ops,
                                  const int64_t* counts) {
  if (!counts) throw std::invalid_argument("null counts");
  seqpipe::Schedule s;
  s.config = cfg;
  s.kind = kind_from_c(kind);
  std::size_t off = 0;
  for (int d = 0; d < cfg.pipeline_size; ++d) {
    if (counts[d] < 0) throw std::invalid_argument("negative op count");
    std::vector<seqpipe::Task> o;
    for (int64_t i = 0; i < counts[d]; ++i) o.push_back(from_c(ops[off + static_cast<std::size_t>(i)]));
    off += static_cast<std::size_t>(counts[d]);
    s.device_orders.push_back(std::move(o));
  }
  return s;
}

void schedule_to_c(const seqpipe::Schedule& s, sp_task* ops, int64_t* counts) {
  std::size_t off = 0;
  for (std::size_t d = 0; d < s.device_orders.size(); ++d) {
    counts[d] = static_cast<int64_t>(s.device_orders[d].size());
    if (ops)
      for (const seqpipe::Task& t : s.device_orders[d]) ops[off++] = to_c(t);
  }
}

int write_text(const std::string& text, char* buf, size_t* len) {
  if (!len) throw std::invalid_argument("null length");
  const size_t need = text.size() + 1;
  if (!buf || *len < need) {
    *len = need;
    if (!buf) return SP_OK;
    set_error("buffer too small");
    return SP_ERR_BUFFER_TOO_SMALL;
  }
  std::memcpy(buf, text.c_str(), need);
  *len = need;
  return SP_OK;
}

std::string violations_text(const std::vector<seqpipe::Violation>& vs) {
  std::string out;
  for (const auto& v : vs) out += v.code + "\t" + std::to_string(v.device) + "\t" + v.detail + "\n";
  return out;
}

}  // namespace spc

using namespace spc;

extern "C" {

const char* sp_last_error(void) { return g_last_error.c_str(); }
const char* sp_version(void) { return "seqpipe_b200 0.1 (sm_100a)"; }

void sp_scenario_default(sp_scenario* out) {
  if (out) to_c(seqpipe::ScenarioConfig{}, out);
}

int sp_scenario_validate(const sp_scenario* cfg) {
  SP_GUARD(from_c(cfg).validate());
}

int sp_preset_scenario(const char* name, sp_scenario* out) {
  SP_GUARD(to_c(seqpipe::preset_scenario(name ? name : ""), out));
}

int sp_apply_override(sp_scenario* cfg, const char* key, const char* value) {
  SP_GUARD({
    seqpipe::ScenarioConfig s = from_c(cfg);
    seqpipe::apply_scenario_override(s, key ? key : "", value ? value : "");
    to_c(s, cfg);
  });
}

int sp_parse_scenario_text(const char* text, sp_scenario* out) {
  SP_GUARD(to_c(seqpipe::parse_scenario_text(text ? text : ""), out));
}

int sp_scenario_to_text(const sp_scenario* cfg, char* buf, size_t* len) {
  try {
    return write_text(seqpipe::scenario_to_text(from_c(cfg)), buf, len);
  } catch (...) {
    return map_exception();
  }
}

int sp_segment_flops(const sp_scenario* cfg, int64_t prefix_before, int64_t length, int64_t* hi, uint64_t* lo) {
  SP_GUARD({
    seqpipe::detail::Int128 v = seqpipe::segment_flops(from_c(cfg), prefix_before, length);
    *hi = static_cast<int64_t>(v >> 64);
    *lo = static_cast<uint64_t>(v);
  });
}

int sp_forward_cost(const sp_scenario* cfg, const int64_t* lengths, int32_t k, int32_t segment, sp_rational* out) {
  SP_GUARD({
    auto c = from_c(cfg);
    *out = to_c(seqpipe::forward_cost(c, partition_from_c(c, lengths, k), segment));
  });
}

int sp_task_cost(const sp_scenario* cfg, const int64_t* lengths, int32_t k, const sp_task* task, sp_rational* out) {
  SP_GUARD({
    auto c = from_c(cfg);
    *out = to_c(seqpipe::task_cost(c, partition_from_c(c, lengths, k), from_c(*task)));
  });
}

int sp_partition(const sp_scenario* cfg, int32_t mode, int64_t* lengths_out, sp_rational* imbalance_out) {
  SP_GUARD({
    if (mode < 0 || mode > 2) throw std::invalid_argument("partition mode out of range");
    auto p = seqpipe::partition_for(from_c(cfg), static_cast<seqpipe::PartitionMode>(mode));
    std::copy(p.lengths.begin(), p.lengths.end(), lengths_out);
    if (imbalance_out) *imbalance_out = to_c(p.imbalance);
  });
}

int sp_even_partition(int64_t n, int32_t k, const sp_scenario* cfg, int64_t* lengths_out, sp_rational* imbalance_out) {
  SP_GUARD({
    auto p = seqpipe::even_partition(n, k, from_c(cfg));
    std::copy(p.lengths.begin(), p.lengths.end(), lengths_out);
    if (imbalance_out) *imbalance_out = to_c(p.imbalance);
  });
}

int sp_make_partition(const sp_scenario* cfg, const int64_t* lengths, int32_t k, sp_rational* imbalance_out) {
  SP_GUARD({
    auto p = partition_from_c(from_c(cfg), lengths, k);
    if (imbalance_out) *imbalance_out = to_c(p.imbalance);
  });
}

int sp_balance_report(const sp_scenario* cfg, const int64_t* lengths, int32_t k, sp_rational* costs,
                      sp_rational* imbalance_out) {
  SP_GUARD({
    auto c = from_c(cfg);
    auto r = seqpipe::balance_report(partition_from_c(c, lengths, k), c);
    for (std::size_t i = 0; i < r.segment_costs.size(); ++i) costs[i] = to_c(r.segment_costs[i]);
    if (imbalance_out) *imbalance_out = to_c(r.imbalance);
  });
}

int sp_warmup(int32_t formula, int32_t P, int32_t a, int32_t k, int32_t device, int32_t* out) {
  SP_GUARD({
    switch (formula) {
      case 0: *out = seqpipe::warmup_1f1b(P, a, device); break;
      case 1: *out = seqpipe::warmup_seq1f1b(P, a, k, device); break;
      case 2: *out = seqpipe::warmup_1f1b_interleaved(P, a, device); break;
      case 3: *out = seqpipe::warmup_seq1f1b_interleaved(P, a, k, device); break;
      default: throw std::invalid_argument("warm-up formula out of range");
    }
  });
}

int sp_schedule_ops(const sp_scenario* cfg, int32_t kind, const int64_t* lengths, sp_task* ops, int64_t* counts) {
  SP_GUARD({
    auto c = from_c(cfg);
    c.validate();
    auto s = seqpipe::generate(c, kind_from_c(kind), partition_from_c(c, lengths, c.segments));
    schedule_to_c(s, ops, counts);
  });
}

int sp_dependencies(const sp_task* task, const sp_scenario* cfg, sp_task* out, int32_t* n_out) {
  SP_GUARD({
    auto d = seqpipe::dependencies(from_c(*task), from_c(cfg));
    for (std::size_t i = 0; i < d.size(); ++i) out[i] = to_c(d[i]);
    *n_out = static_cast<int32_t>(d.size());
  });
}

int sp_simulate(const sp_scenario* cfg, int32_t kind, const int64_t* lengths, const sp_task* ops, const int64_t* counts,
                sp_task_timing* timings, sp_device_report* devices, sp_sim_summary* summary) {
  SP_GUARD({
    auto c = from_c(cfg);
    auto part = partition_from_c(c, lengths, c.segments);
    auto rep = seqpipe::simulate(schedule_from_c(c, kind, ops, counts), part);
    if (timings) {
      std::size_t off = 0;
      for (const auto& tt : rep.task_times)
        for (const auto& t : tt) timings[off++] = sp_task_timing{to_c(t.task), to_c(t.start), to_c(t.end)};
    }
    if (devices) {
      for (std::size_t d = 0; d < rep.devices.size(); ++d) {
        const auto& r = rep.devices[d];
        sp_device_report& o = devices[d];
        o.device = r.device;
        o.warmup_forward_tasks = r.warmup_forward_tasks;
        o.peak_allocations = r.peak_allocations;
        o.first_start = to_c(r.first_start);
        o.last_end = to_c(r.last_end);
        o.busy = to_c(r.busy);
        o.idle = to_c(r.idle);
        o.bubble_ratio = to_c(r.bubble_ratio);
        o.idle_in_makespan = to_c(r.idle_in_makespan);
        o.bubble_ratio_in_makespan = to_c(r.bubble_ratio_in_makespan);
        o.peak_memory = to_c(r.peak_memory);
        o.memory_series_len = static_cast<int64_t>(r.memory_series.size());
      }
    }
    if (summary) {
      summary->makespan = to_c(rep.makespan);
      summary->aggregate_bubble_ratio = to_c(rep.aggregate_bubble_ratio);
      summary->aggregate_bubble_ratio_in_makespan = to_c(rep.aggregate_bubble_ratio_in_makespan);
      summary->max_peak_memory = to_c(rep.max_peak_memory);
      summary->modeled_throughput = to_c(rep.modeled_throughput);
    }
  });
}

int sp_simulate_memory_series(const sp_scenario* cfg, int32_t kind, const int64_t* lengths, const sp_task* ops,
                              const int64_t* counts, int32_t device, sp_rational* series, int64_t* len) {
  try {
    auto c = from_c(cfg);
    auto part = partition_from_c(c, lengths, c.segments);
    auto rep = seqpipe::simulate(schedule_from_c(c, kind, ops, counts), part);
    if (device < 1 || device > c.pipeline_size) throw std::out_of_range("device index out of range");
    const auto& ms = rep.devices[static_cast<std::size_t>(device - 1)].memory_series;
    const int64_t need = static_cast<int64_t>(ms.size());
    if (!series || *len < need) {
      *len = need;
      if (!series) return SP_OK;
      set_error("buffer too small");
      return SP_ERR_BUFFER_TOO_SMALL;
    }
    for (std::size_t i = 0; i < ms.size(); ++i) {
      series[2 * i] = to_c(ms[i].first);
      series[2 * i + 1] = to_c(ms[i].second);
    }
    *len = need;
    return SP_OK;
  } catch (...) {
    return map_exception();
  }
}

int sp_check_schedule(const sp_scenario* cfg, int32_t kind, const sp_task* ops, const int64_t* counts, char* buf,
                      size_t* len, int32_t* n_violations) {
  try {
    auto v = seqpipe::check_schedule(schedule_from_c(from_c(cfg), kind, ops, counts));
    if (n_violations) *n_violations = static_cast<int32_t>(v.size());
    return write_text(violations_text(v), buf, len);
  } catch (...) {
    return map_exception();
  }
}

int sp_check_warmup_formulas(const sp_scenario* cfg, int32_t kind, const sp_task* ops, const int64_t* counts, char* buf,
                             size_t* len, int32_t* n_violations) {
  try {
    auto v = seqpipe::check_warmup_formulas(schedule_from_c(from_c(cfg), kind, ops, counts));
    if (n_violations) *n_violations = static_cast<int32_t>(v.size());
    return write_text(violations_text(v), buf, len);
  } catch (...) {
    return map_exception();
  }
}


int sp_schedule_to_json(const sp_scenario* cfg, int32_t kind, const sp_task* ops, const int64_t* counts, int32_t indent,
                        char* buf, size_t* len) {
  try {
    const auto c = from_c(cfg);
    return write_text(seqpipe::schedule_to_json(schedule_from_c(c, kind, ops, counts), indent), buf, len);
  } catch (...) {
    return map_exception();
  }
}

int sp_schedule_from_json(const char* text, sp_scenario* cfg_out, int32_t* kind_out, sp_task* ops, int64_t* counts,
                          int32_t max_devices) {
  SP_GUARD({
    if (!text || !cfg_out || !kind_out || !counts) throw std::invalid_argument("null argument");
    const seqpipe::Schedule s = seqpipe::schedule_from_json(text);
    if (static_cast<int32_t>(s.device_orders.size()) > max_devices)
      throw std::out_of_range("schedule has more devices than max_devices");
    to_c(s.config, cfg_out);
    *kind_out = static_cast<int32_t>(s.kind);
    std::size_t off = 0;
    for (std::size_t d = 0; d < s.device_orders.size(); ++d) {
      counts[d] = static_cast<int64_t>(s.device_orders[d].size());
      if (ops)
        for (const auto& t : s.device_orders[d]) ops[off++] = to_c(t);
    }
  });
}

int sp_report_to_json(const sp_scenario* cfg, int32_t kind, const int64_t* lengths, const sp_task* ops,
                      const int64_t* counts, int32_t indent, int64_t memory_downsample, char* buf, size_t* len) {
  try {
    const auto c = from_c(cfg);
    const auto rep = seqpipe::simulate(schedule_from_c(c, kind, ops, counts), partition_from_c(c, lengths, c.segments));
    return write_text(seqpipe::report_to_json(rep, indent, static_cast<std::size_t>(memory_downsample < 0 ? 0 : memory_downsample)),
                      buf, len);
  } catch (...) {
    return map_exception();
  }
}

int sp_render_gantt(const sp_scenario* cfg, int32_t kind, const int64_t* lengths, const sp_task* ops,
                    const int64_t* counts, int32_t format, int32_t width, char* buf, size_t* len) {
  try {
    const auto c = from_c(cfg);
    const auto rep = seqpipe::simulate(schedule_from_c(c, kind, ops, counts), partition_from_c(c, lengths, c.segments));
    if (format != SP_RENDER_ASCII && format != SP_RENDER_SVG) throw std::invalid_argument("unknown render format");
    return write_text(format == SP_RENDER_SVG ? seqpipe::render_svg_gantt(rep) : seqpipe::render_ascii_gantt(rep, width),
                      buf, len);
  } catch (...) {
    return map_exception();
  }
}

int sp_compare_csv(int32_t n, const sp_scenario* cfgs, const int32_t* kinds, const int64_t* const* lengths,
                   const sp_task* const* ops, const int64_t* const* counts, int32_t allow_mixed, char* buf,
                   size_t* len) {
  try {
    if (n < 0 || (n > 0 && (!cfgs || !kinds || !lengths || !ops || !counts))) throw std::invalid_argument("null input");
    std::vector<seqpipe::SimReport> reps;
    reps.reserve(static_cast<std::size_t>(n));
    for (int32_t i = 0; i < n; ++i) {
      const auto c = from_c(&cfgs[i]);
      reps.push_back(seqpipe::simulate(schedule_from_c(c, kinds[i], ops[i], counts[i]),
                                       partition_from_c(c, lengths[i], c.segments)));
    }
    return write_text(seqpipe::compare(reps, allow_mixed != 0).to_csv(), buf, len);
  } catch (...) {
    return map_exception();
  }
}

}  // extern "C"
