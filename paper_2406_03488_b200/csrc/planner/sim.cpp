// Host planner, part 3: dependency model and the modeled (exact rational)
// execution. Reference behaviour: /root/reference/proj/core/src/sim.cpp:14-317.
// Start times are a pure function of dependency end times and the device's
// previous end, so the event loop below gives the reference's times exactly
// regardless of the order devices are visited in.
#include <algorithm>
#include <array>
#include <map>
#include <sstream>

#include "seqpipe/cost.hpp"
#include "seqpipe/sim.hpp"

namespace seqpipe {

std::vector<Task> dependencies(const Task& t, const ScenarioConfig& cfg) {
  return timing_dependencies(t, cfg, false);
}

std::vector<Task> timing_dependencies(const Task& t, const ScenarioConfig& cfg, bool batch_atomic) {
  // Legality edges (sim.cpp:14-44); with batch_atomic the cross-stage edge
  // binds to the neighbour's last task of the unit (sim.cpp:54-88).
  const int P = cfg.pipeline_size, V = cfg.total_stages(), k = cfg.segments;
  std::vector<Task> deps;
  switch (t.kind) {
    case TaskKind::kForward:
      if (t.stage > 1) deps.push_back(make_task(TaskKind::kForward, t.micro_batch, batch_atomic ? k : t.segment, t.stage - 1, P));
      if (t.segment > 1) deps.push_back(make_task(TaskKind::kForward, t.micro_batch, t.segment - 1, t.stage, P));
      break;
    case TaskKind::kFusedBackward:
    case TaskKind::kInputGrad:
      if (t.stage < V) deps.push_back(make_task(t.kind, t.micro_batch, batch_atomic ? 1 : t.segment, t.stage + 1, P));
      if (t.segment < k) deps.push_back(make_task(t.kind, t.micro_batch, t.segment + 1, t.stage, P));
      deps.push_back(make_task(TaskKind::kForward, t.micro_batch, t.segment, t.stage, P));
      break;
    case TaskKind::kWeightGrad:
      deps.push_back(make_task(TaskKind::kInputGrad, t.micro_batch, t.segment, t.stage, P));
      break;
  }
  return deps;
}

namespace {

struct Index {
  int M, k, V;
  std::size_t size() const { return 4u * static_cast<std::size_t>(M) * k * V; }
  bool valid(const Task& t) const {
    return t.micro_batch >= 1 && t.micro_batch <= M && t.segment >= 1 && t.segment <= k && t.stage >= 1 && t.stage <= V;
  }
  std::size_t of(const Task& t) const {
    return ((static_cast<std::size_t>(t.kind) * M + (t.micro_batch - 1)) * k + (t.segment - 1)) * V + (t.stage - 1);
  }
};

std::string show(const Task& t) {
  std::ostringstream o;
  o << task_kind_name(t.kind) << "(m=" << t.micro_batch << ",s=" << t.segment << ",stage=" << t.stage << ")";
  return o.str();
}

}  // namespace

SimReport simulate(const Schedule& sch, const SequencePartition& part) {
  const ScenarioConfig& cfg = sch.config;
  cfg.validate();
  if (part.segment_count() != cfg.segments || part.total != cfg.seq_len)
    throw std::invalid_argument("partition does not match the scenario");
  const int P = cfg.pipeline_size;
  if (static_cast<int>(sch.device_orders.size()) != P)
    throw std::invalid_argument("schedule device count does not match pipeline_size");

  const Index ix{cfg.micro_batches, cfg.segments, cfg.total_stages()};
  std::vector<char> present(ix.size(), 0), done(ix.size(), 0);
  std::vector<Rational> finish(ix.size());
  for (const auto& order : sch.device_orders)
    for (const Task& t : order) {
      if (!ix.valid(t)) throw std::invalid_argument("task out of range: " + show(t));
      present[ix.of(t)] = 1;
    }

  // Resolve durations and timing edges once.
  const bool batch_atomic = !is_sequence_level(sch.kind);
  struct Edge {
    std::size_t id;
    bool remote;
  };
  std::vector<std::vector<Rational>> dur(static_cast<std::size_t>(P));
  std::vector<std::vector<std::vector<Edge>>> edges(static_cast<std::size_t>(P));
  std::size_t remaining = 0;
  for (int d = 0; d < P; ++d) {
    for (const Task& t : sch.device_orders[static_cast<std::size_t>(d)]) {
      dur[static_cast<std::size_t>(d)].push_back(task_cost(cfg, part, t));
      std::vector<Edge> e;
      for (const Task& dep : timing_dependencies(t, cfg, batch_atomic)) {
        if (!present[ix.of(dep)]) throw MissingDependencyError("schedule is missing " + show(dep) + ", required by " + show(t));
        e.push_back({ix.of(dep), dep.device != t.device});
      }
      edges[static_cast<std::size_t>(d)].push_back(std::move(e));
      ++remaining;
    }
  }

  SimReport rep;
  rep.kind = sch.kind;
  rep.config = cfg;
  rep.partition_lengths = part.lengths;
  rep.task_times.resize(static_cast<std::size_t>(P));
  std::vector<std::size_t> next(static_cast<std::size_t>(P), 0);
  std::vector<Rational> free_at(static_cast<std::size_t>(P), Rational(0));
  while (remaining) {
    bool moved = false;
    for (int d = 0; d < P; ++d) {
      const auto& order = sch.device_orders[static_cast<std::size_t>(d)];
      std::size_t& c = next[static_cast<std::size_t>(d)];
      for (; c < order.size(); ++c) {
        Rational start = free_at[static_cast<std::size_t>(d)];
        bool ready = true;
        for (const Edge& e : edges[static_cast<std::size_t>(d)][c]) {
          if (!done[e.id]) {
            ready = false;
            break;
          }
          start = std::max(start, e.remote ? finish[e.id] + cfg.comm_latency : finish[e.id]);
        }
        if (!ready) break;
        const Rational end = start + dur[static_cast<std::size_t>(d)][c];
        free_at[static_cast<std::size_t>(d)] = end;
        done[ix.of(order[c])] = 1;
        finish[ix.of(order[c])] = end;
        rep.task_times[static_cast<std::size_t>(d)].push_back({order[c], start, end});
        --remaining;
        moved = true;
      }
    }
    if (!moved) {
      std::ostringstream o;
      o << "deadlock: no runnable task; blocked front tasks:";
      for (int d = 0; d < P; ++d) {
        const auto& order = sch.device_orders[static_cast<std::size_t>(d)];
        const std::size_t c = next[static_cast<std::size_t>(d)];
        if (c >= order.size()) continue;
        o << " device " << d + 1 << " waits on " << show(order[c]) << " needing";
        for (const Task& dep : timing_dependencies(order[c], cfg, batch_atomic))
          if (!done[ix.of(dep)]) o << ' ' << show(dep);
        o << ';';
      }
      throw DeadlockError(o.str());
    }
  }

  // Per-device aggregates (sim.cpp:234-274).
  for (const auto& tt : rep.task_times)
    for (const TaskTiming& t : tt) rep.makespan = std::max(rep.makespan, t.end);
  Rational idle_sum{0}, window_sum{0}, idle_mk_sum{0};
  for (int d = 0; d < P; ++d) {
    const auto& tt = rep.task_times[static_cast<std::size_t>(d)];
    DeviceReport dr;
    dr.device = d + 1;
    if (!tt.empty()) {
      dr.first_start = tt.front().start;
      dr.last_end = tt.back().end;
      for (const TaskTiming& t : tt) dr.busy += t.end - t.start;
      const Rational window = dr.last_end - dr.first_start;
      dr.idle = window - dr.busy;
      dr.bubble_ratio = window.is_zero() ? Rational(0) : dr.idle / window;
      dr.idle_in_makespan = rep.makespan - dr.busy;
      dr.bubble_ratio_in_makespan = rep.makespan.is_zero() ? Rational(0) : dr.idle_in_makespan / rep.makespan;
      idle_sum += dr.idle;
      window_sum += window;
      idle_mk_sum += dr.idle_in_makespan;
      while (dr.warmup_forward_tasks < static_cast<int>(tt.size()) &&
             tt[static_cast<std::size_t>(dr.warmup_forward_tasks)].task.kind == TaskKind::kForward)
        ++dr.warmup_forward_tasks;
    }
    rep.devices.push_back(std::move(dr));
  }
  rep.aggregate_bubble_ratio = window_sum.is_zero() ? Rational(0) : idle_sum / window_sum;
  rep.aggregate_bubble_ratio_in_makespan =
      rep.makespan.is_zero() ? Rational(0) : idle_mk_sum / (Rational(P) * rep.makespan);

  // Activation residency (sim.cpp:276-311): +act*n_s at F end, -act*n_s at the
  // end of the freeing task (B, or W for the zero-bubble kinds). Same-time
  // events are merged before the level is sampled.
  const TaskKind frees = is_zero_bubble(sch.kind) ? TaskKind::kWeightGrad : TaskKind::kFusedBackward;
  for (int d = 0; d < P; ++d) {
    std::map<Rational, std::pair<Rational, std::int64_t>> ev;
    for (const TaskTiming& t : rep.task_times[static_cast<std::size_t>(d)]) {
      const Rational amt = cfg.activation_cost_per_token * Rational(part.lengths[static_cast<std::size_t>(t.task.segment - 1)]);
      if (t.task.kind == TaskKind::kForward) {
        ev[t.end].first += amt;
        ev[t.end].second += 1;
      } else if (t.task.kind == frees) {
        ev[t.end].first -= amt;
        ev[t.end].second -= 1;
      }
    }
    DeviceReport& dr = rep.devices[static_cast<std::size_t>(d)];
    Rational level{0};
    std::int64_t live = 0;
    dr.memory_series.emplace_back(Rational(0), Rational(0));
    for (const auto& [time, delta] : ev) {
      level += delta.first;
      live += delta.second;
      if (level.is_negative()) throw std::logic_error("negative activation residency on device " + std::to_string(d + 1));
      dr.peak_memory = std::max(dr.peak_memory, level);
      dr.peak_allocations = std::max(dr.peak_allocations, live);
      dr.memory_series.emplace_back(time, level);
    }
    rep.max_peak_memory = std::max(rep.max_peak_memory, dr.peak_memory);
  }
  rep.modeled_throughput =
      rep.makespan.is_zero() ? Rational(0) : Rational(std::int64_t(cfg.micro_batches) * cfg.seq_len) / rep.makespan;
  return rep;
}

std::vector<std::pair<int, int>> replay_order(const Schedule& sch) {
  const ScenarioConfig& cfg = sch.config;
  const int P = cfg.pipeline_size;
  const Index ix{cfg.micro_batches, cfg.segments, cfg.total_stages()};
  std::vector<char> done(ix.size(), 0);
  std::vector<std::size_t> next(static_cast<std::size_t>(P), 0);
  std::size_t remaining = 0;
  for (const auto& o : sch.device_orders) remaining += o.size();
  std::vector<std::pair<int, int>> out;
  out.reserve(remaining);
  while (remaining) {
    bool moved = false;
    for (int d = 0; d < P; ++d) {
      const auto& order = sch.device_orders[static_cast<std::size_t>(d)];
      std::size_t& c = next[static_cast<std::size_t>(d)];
      for (; c < order.size(); ++c) {
        bool ready = true;
        for (const Task& dep : dependencies(order[c], cfg))
          if (!ix.valid(dep) || !done[ix.of(dep)]) ready = false;
        if (!ready) break;
        done[ix.of(order[c])] = 1;
        out.emplace_back(d, static_cast<int>(c));
        --remaining;
        moved = true;
      }
    }
    if (!moved) throw DeadlockError("replay_order: schedule cannot complete (dependency cycle across device orders)");
  }
  return out;
}

ComparisonTable compare(const std::vector<SimReport>& reports, bool allow_mixed) {
  if (reports.size() < 2) throw std::invalid_argument("compare needs at least two reports");
  const ScenarioConfig& base = reports.front().config;
  const bool same_workload = std::all_of(reports.begin(), reports.end(), [&](const SimReport& r) {
    return r.config.seq_len == base.seq_len && r.config.micro_batches == base.micro_batches;
  });
  if (!allow_mixed && !same_workload)
    throw std::invalid_argument(
        "reports cover different workloads (seq_len/micro_batches); pass allow_mixed to override");
  ComparisonTable table;
  table.rows.reserve(reports.size());
  for (const SimReport& r : reports)
    table.rows.push_back(ComparisonRow{schedule_kind_name(r.kind), r.config, r.makespan, r.aggregate_bubble_ratio,
                                       r.max_peak_memory, r.modeled_throughput});
  return table;
}

std::string ComparisonTable::to_csv() const {
  std::string csv =
      "kind,pipeline_size,stages_per_device,micro_batches,segments,seq_len,"
      "makespan,bubble_ratio,max_peak_memory,throughput,"
      "makespan_vs_first,bubble_vs_first,memory_vs_first,throughput_vs_first\n";
  if (rows.empty()) return csv;
  const ComparisonRow& first = rows.front();
  auto metrics = [](const ComparisonRow& r) {
    return std::array<const Rational*, 4>{&r.makespan, &r.bubble_ratio, &r.max_peak_memory, &r.throughput};
  };
  const auto base = metrics(first);
  for (const ComparisonRow& r : rows) {
    const ScenarioConfig& c = r.config;
    csv += r.kind;
    for (long long v : {static_cast<long long>(c.pipeline_size), static_cast<long long>(c.stages_per_device),
                        static_cast<long long>(c.micro_batches), static_cast<long long>(c.segments),
                        static_cast<long long>(c.seq_len)})
      csv += ',' + std::to_string(v);
    const auto m = metrics(r);
    for (const Rational* v : m) csv += ',' + format_decimal(*v, 6);
    for (std::size_t i = 0; i < m.size(); ++i)
      csv += ',' + (base[i]->is_zero() ? std::string() : format_decimal(*m[i] / *base[i], 6));
    csv += '\n';
  }
  return csv;
}

}  // namespace seqpipe
