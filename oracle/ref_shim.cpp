// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// extern "C" shim over the UNMODIFIED reference seqpipe core, compiled from
// its own sources in /root/reference/proj/core/src by oracle/build_ref.sh into
// oracle/_ref/libseqpipe_ref.so. It exposes the reference's planner through the
// same C structs as include/seqpipe_b200.h (prefix ref_ instead of sp_) so
// tests can diff the engine's planner against the reference byte for byte.
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
// reference legs may load it.
#include <chrono>
#include <cstring>
#include <string>
#include <vector>

#include "seqpipe/cost.hpp"
#include "seqpipe/json_io.hpp"
#include "seqpipe/render.hpp"
#include "seqpipe/partition.hpp"
#include "seqpipe/poq.hpp"
#include "seqpipe/scenario.hpp"
#include "seqpipe/schedule.hpp"
#include "seqpipe/sim.hpp"
#include "seqpipe/validate.hpp"
#include "seqpipe_b200.h"  // C structs only

using namespace seqpipe;

namespace {

thread_local std::string g_err;

int fail(int code, const char* what) {
  g_err = what;
  return code;
}

#define REF_GUARD(...)                                                          \
  try {                                                                         \
    __VA_ARGS__;                                                                \
    return 0;                                                                   \
  } catch (const UnsupportedScheduleError& e) {                                 \
    return fail(SP_ERR_UNSUPPORTED, e.what());                                  \
  } catch (const DeadlockError& e) {                                            \
    return fail(SP_ERR_DEADLOCK, e.what());                                     \
  } catch (const MissingDependencyError& e) {                                   \
    return fail(SP_ERR_MISSING_DEPENDENCY, e.what());                           \
  } catch (const std::out_of_range& e) {                                        \
    return fail(SP_ERR_OUT_OF_RANGE, e.what());                                 \
  } catch (const std::invalid_argument& e) {                                    \
    return fail(SP_ERR_INVALID_ARGUMENT, e.what());                             \
  } catch (const std::domain_error& e) {                                        \
    return fail(SP_ERR_DOMAIN, e.what());                                       \
  } catch (const std::overflow_error& e) {                                      \
    return fail(SP_ERR_OVERFLOW, e.what());                                     \
  } catch (const std::logic_error& e) {                                         \
    return fail(SP_ERR_LOGIC, e.what());                                        \
  } catch (const std::exception& e) {                                           \
    return fail(SP_ERR_RUNTIME, e.what());                                      \
  }

Rational R(const sp_rational& r) { return Rational(r.num, r.den); }
sp_rational C(const Rational& r) { return sp_rational{r.numerator(), r.denominator()}; }

ScenarioConfig cfg_of(const sp_scenario* c) {
  ScenarioConfig s;
  s.pipeline_size = c->pipeline_size;
  s.stages_per_device = c->stages_per_device;
  s.micro_batches = c->micro_batches;
  s.segments = c->segments;
  s.seq_len = c->seq_len;
  s.layers = c->layers;
  s.hidden_dim = c->hidden_dim;
  s.param_count = c->param_count;
  s.backward_ratio = R(c->backward_ratio);
  s.bw_input_ratio = R(c->bw_input_ratio);
  s.bw_weight_ratio = R(c->bw_weight_ratio);
  s.comm_latency = R(c->comm_latency);
  s.activation_cost_per_token = R(c->activation_cost_per_token);
  s.time_per_flop = R(c->time_per_flop);
  s.cost_model = c->cost_model == SP_COST_UNIFORM ? CostModel::kUniform : CostModel::kFlops;
  s.uniform_forward = R(c->uniform_forward);
  return s;
}

void cfg_to(const ScenarioConfig& s, sp_scenario* c) {
  c->pipeline_size = s.pipeline_size;
  c->stages_per_device = s.stages_per_device;
  c->micro_batches = s.micro_batches;
  c->segments = s.segments;
  c->seq_len = s.seq_len;
  c->layers = s.layers;
  c->hidden_dim = s.hidden_dim;
  c->param_count = s.param_count;
  c->backward_ratio = C(s.backward_ratio);
  c->bw_input_ratio = C(s.bw_input_ratio);
  c->bw_weight_ratio = C(s.bw_weight_ratio);
  c->comm_latency = C(s.comm_latency);
  c->activation_cost_per_token = C(s.activation_cost_per_token);
  c->time_per_flop = C(s.time_per_flop);
  c->cost_model = s.cost_model == CostModel::kUniform ? SP_COST_UNIFORM : SP_COST_FLOPS;
  c->uniform_forward = C(s.uniform_forward);
}

Task task_of(const sp_task& t) {
  return Task{static_cast<TaskKind>(t.kind), t.micro_batch, t.segment, t.stage, t.device};
}
sp_task task_to(const Task& t) {
  return sp_task{static_cast<int32_t>(t.kind), t.micro_batch, t.segment, t.stage, t.device};
}

SequencePartition part_of(const ScenarioConfig& c, const int64_t* len) {
  return make_partition(std::vector<std::int64_t>(len, len + c.segments), c);
}

Schedule sched_of(const ScenarioConfig& c, int32_t kind, const sp_task* ops, const int64_t* counts) {
  Schedule s;
  s.config = c;
  s.kind = static_cast<ScheduleKind>(kind);
  std::size_t off = 0;
  for (int d = 0; d < c.pipeline_size; ++d) {
    std::vector<Task> o;
    for (int64_t i = 0; i < counts[d]; ++i) o.push_back(task_of(ops[off + static_cast<std::size_t>(i)]));
    off += static_cast<std::size_t>(counts[d]);
    s.device_orders.push_back(std::move(o));
  }
  return s;
}

int text_out(const std::string& t, char* buf, size_t* len) {
  if (!buf || *len < t.size() + 1) {
    *len = t.size() + 1;
    return buf ? fail(SP_ERR_BUFFER_TOO_SMALL, "buffer too small") : 0;
  }
  std::memcpy(buf, t.c_str(), t.size() + 1);
  *len = t.size() + 1;
  return 0;
}

std::string vtext(const std::vector<Violation>& vs) {
  std::string out;
  for (const auto& v : vs) out += v.code + "\t" + std::to_string(v.device) + "\t" + v.detail + "\n";
  return out;
}

}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

int ref_preset_scenario(const char* name, sp_scenario* out) { REF_GUARD(cfg_to(preset_scenario(name), out)); }

int ref_parse_scenario_text(const char* text, sp_scenario* out) { REF_GUARD(cfg_to(parse_scenario_text(text), out)); }

int ref_apply_override(sp_scenario* c, const char* key, const char* value) {
  REF_GUARD({
    ScenarioConfig s = cfg_of(c);
    apply_scenario_override(s, key, value);
    cfg_to(s, c);
  });
}

int ref_scenario_validate(const sp_scenario* c) { REF_GUARD(cfg_of(c).validate()); }

int ref_scenario_to_text(const sp_scenario* c, char* buf, size_t* len) {
  try {
    return text_out(scenario_to_text(cfg_of(c)), buf, len);
  } catch (const std::exception& e) {
    return fail(SP_ERR_RUNTIME, e.what());
  }
}

int ref_partition(const sp_scenario* c, int32_t mode, int64_t* out, sp_rational* imb) {
  REF_GUARD({
    auto p = partition_for(cfg_of(c), static_cast<PartitionMode>(mode));
    std::copy(p.lengths.begin(), p.lengths.end(), out);
    if (imb) *imb = C(p.imbalance);
  });
}

int ref_make_partition(const sp_scenario* c, const int64_t* len, int32_t k, sp_rational* imb) {
  REF_GUARD({
    auto p = make_partition(std::vector<std::int64_t>(len, len + k), cfg_of(c));
    if (imb) *imb = C(p.imbalance);
  });
}

int ref_balance_report(const sp_scenario* c, const int64_t* len, int32_t k, sp_rational* costs, sp_rational* imb) {
  REF_GUARD({
    auto cfg = cfg_of(c);
    auto r = balance_report(make_partition(std::vector<std::int64_t>(len, len + k), cfg), cfg);
    for (std::size_t i = 0; i < r.segment_costs.size(); ++i) costs[i] = C(r.segment_costs[i]);
    if (imb) *imb = C(r.imbalance);
  });
}

int ref_segment_flops(const sp_scenario* c, int64_t before, int64_t n, int64_t* hi, uint64_t* lo) {
  REF_GUARD({
    detail::Int128 v = segment_flops(cfg_of(c), before, n);
    *hi = static_cast<int64_t>(v >> 64);
    *lo = static_cast<uint64_t>(v);
  });
}

int ref_task_cost(const sp_scenario* c, const int64_t* len, const sp_task* t, sp_rational* out) {
  REF_GUARD({
    auto cfg = cfg_of(c);
    *out = C(task_cost(cfg, part_of(cfg, len), task_of(*t)));
  });
}

int ref_warmup(int32_t formula, int32_t P, int32_t a, int32_t k, int32_t device, int32_t* out) {
  REF_GUARD({
    switch (formula) {
      case 0: *out = warmup_1f1b(P, a, device); break;
      case 1: *out = warmup_seq1f1b(P, a, k, device); break;
      case 2: *out = warmup_1f1b_interleaved(P, a, device); break;
      default: *out = warmup_seq1f1b_interleaved(P, a, k, device); break;
    }
  });
}

int ref_schedule_ops(const sp_scenario* c, int32_t kind, const int64_t* len, sp_task* ops, int64_t* counts) {
  REF_GUARD({
    auto cfg = cfg_of(c);
    Schedule s = generate(cfg, static_cast<ScheduleKind>(kind), part_of(cfg, len));
    std::size_t off = 0;
    for (std::size_t d = 0; d < s.device_orders.size(); ++d) {
      counts[d] = static_cast<int64_t>(s.device_orders[d].size());
      if (ops)
        for (const Task& t : s.device_orders[d]) ops[off++] = task_to(t);
    }
  });
}

int ref_dependencies(const sp_task* t, const sp_scenario* c, sp_task* out, int32_t* n) {
  REF_GUARD({
    auto d = dependencies(task_of(*t), cfg_of(c));
    for (std::size_t i = 0; i < d.size(); ++i) out[i] = task_to(d[i]);
    *n = static_cast<int32_t>(d.size());
  });
}

int ref_simulate(const sp_scenario* c, int32_t kind, const int64_t* len, const sp_task* ops, const int64_t* counts,
                 sp_task_timing* timings, sp_device_report* devs, sp_sim_summary* sum) {
  REF_GUARD({
    auto cfg = cfg_of(c);
    SimReport r = simulate(sched_of(cfg, kind, ops, counts), part_of(cfg, len));
    if (timings) {
      std::size_t off = 0;
      for (const auto& tt : r.task_times)
        for (const auto& t : tt) timings[off++] = sp_task_timing{task_to(t.task), C(t.start), C(t.end)};
    }
    if (devs)
      for (std::size_t d = 0; d < r.devices.size(); ++d) {
        const DeviceReport& x = r.devices[d];
        devs[d] = sp_device_report{x.device,      x.warmup_forward_tasks, x.peak_allocations, C(x.first_start),
                                   C(x.last_end), C(x.busy),              C(x.idle),          C(x.bubble_ratio),
                                   C(x.idle_in_makespan), C(x.bubble_ratio_in_makespan), C(x.peak_memory),
                                   static_cast<int64_t>(x.memory_series.size())};
      }
    if (sum)
      *sum = sp_sim_summary{C(r.makespan), C(r.aggregate_bubble_ratio), C(r.aggregate_bubble_ratio_in_makespan),
                            C(r.max_peak_memory), C(r.modeled_throughput)};
  });
}

int ref_check_schedule(const sp_scenario* c, int32_t kind, const sp_task* ops, const int64_t* counts, char* buf,
                       size_t* len, int32_t* nv) {
  try {
    auto v = check_schedule(sched_of(cfg_of(c), kind, ops, counts));
    *nv = static_cast<int32_t>(v.size());
    return text_out(vtext(v), buf, len);
  } catch (const std::exception& e) {
    return fail(SP_ERR_RUNTIME, e.what());
  }
}

int ref_check_warmup_formulas(const sp_scenario* c, int32_t kind, const sp_task* ops, const int64_t* counts, char* buf,
                              size_t* len, int32_t* nv) {
  try {
    auto v = check_warmup_formulas(sched_of(cfg_of(c), kind, ops, counts));
    *nv = static_cast<int32_t>(v.size());
    return text_out(vtext(v), buf, len);
  } catch (const std::invalid_argument& e) {
    return fail(SP_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::exception& e) {
    return fail(SP_ERR_RUNTIME, e.what());
  }
}

// POQ driver for the queue KATs: push (m,s) pairs, then pop n times.
int ref_poq_run(const int32_t* ops, int32_t n_ops, int32_t* pops_out, int32_t* n_pops) {
  // ops: triples (op, m, s) with op 0 = push, 1 = pop.
  REF_GUARD({
    PartiallyOrderedQueue q;
    int32_t np = 0;
    for (int32_t i = 0; i < n_ops; ++i) {
      if (ops[3 * i] == 0) {
        q.push(ops[3 * i + 1], ops[3 * i + 2]);
      } else {
        auto [m, s] = q.pop();
        pops_out[2 * np] = m;
        pops_out[2 * np + 1] = s;
        ++np;
      }
    }
    *n_pops = np;
  });
}

// Planner timing for the CPU baseline: cwp_partition + generate + simulate +
// check_schedule, best of `reps` (nanoseconds). Single-threaded, as the reference.
int ref_time_planner(const sp_scenario* c, int32_t kind, int32_t mode, int32_t reps, double* best_ns) {
  REF_GUARD({
    auto cfg = cfg_of(c);
    double best = 1e300;
    for (int r = 0; r < reps; ++r) {
      auto t0 = std::chrono::steady_clock::now();
      auto p = partition_for(cfg, static_cast<PartitionMode>(mode));
      Schedule s = generate(cfg, static_cast<ScheduleKind>(kind), p);
      SimReport rep = simulate(s, p);
      auto v = check_schedule(s);
      auto t1 = std::chrono::steady_clock::now();
      if (!v.empty() || rep.makespan.is_zero()) throw std::logic_error("reference planner produced an invalid schedule");
      best = std::min(best, std::chrono::duration<double, std::nano>(t1 - t0).count());
    }
    *best_ns = best;
  });
}

int ref_schedule_to_json(const sp_scenario* c, int32_t kind, const sp_task* ops, const int64_t* counts, int32_t indent,
                         char* buf, size_t* len) {
  try {
    return text_out(schedule_to_json(sched_of(cfg_of(c), kind, ops, counts), indent), buf, len);
  } catch (const std::exception& e) {
    return fail(SP_ERR_RUNTIME, e.what());
  }
}

// dump(parse(text)) through the reference: the canonical-form round trip.
int ref_schedule_json_roundtrip(const char* text, int32_t indent, char* buf, size_t* len) {
  try {
    return text_out(schedule_to_json(schedule_from_json(text), indent), buf, len);
  } catch (const std::exception& e) {
    return fail(SP_ERR_INVALID_ARGUMENT, e.what());
  }
}

int ref_report_to_json(const sp_scenario* c, int32_t kind, const int64_t* lengths, const sp_task* ops,
                       const int64_t* counts, int32_t indent, int64_t downsample, char* buf, size_t* len) {
  try {
    auto cfg = cfg_of(c);
    SimReport r = simulate(sched_of(cfg, kind, ops, counts), part_of(cfg, lengths));
    return text_out(report_to_json(r, indent, static_cast<std::size_t>(downsample < 0 ? 0 : downsample)), buf, len);
  } catch (const std::exception& e) {
    return fail(SP_ERR_RUNTIME, e.what());
  }
}

int ref_render_gantt(const sp_scenario* c, int32_t kind, const int64_t* lengths, const sp_task* ops,
                     const int64_t* counts, int32_t format, int32_t width, char* buf, size_t* len) {
  try {
    auto cfg = cfg_of(c);
    SimReport r = simulate(sched_of(cfg, kind, ops, counts), part_of(cfg, lengths));
    return text_out(format == 1 ? render_svg_gantt(r) : render_ascii_gantt(r, width), buf, len);
  } catch (const std::exception& e) {
    return fail(SP_ERR_RUNTIME, e.what());
  }
}

int ref_compare_csv(int32_t n, const sp_scenario* cs, const int32_t* kinds, const int64_t* const* lengths,
                    const sp_task* const* ops, const int64_t* const* counts, int32_t allow_mixed, char* buf,
                    size_t* len) {
  try {
    std::vector<SimReport> reps;
    for (int32_t i = 0; i < n; ++i) {
      auto cfg = cfg_of(&cs[i]);
      reps.push_back(simulate(sched_of(cfg, kinds[i], ops[i], counts[i]), part_of(cfg, lengths[i])));
    }
    return text_out(compare(reps, allow_mixed != 0).to_csv(), buf, len);
  } catch (const std::invalid_argument& e) {
    return fail(SP_ERR_INVALID_ARGUMENT, e.what());
  } catch (const std::exception& e) {
    return fail(SP_ERR_RUNTIME, e.what());
  }
}

}  // extern "C"
