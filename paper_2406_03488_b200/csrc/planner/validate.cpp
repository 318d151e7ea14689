// Host planner, part 4: the legality checker run against every op table the
// engine executes. Same checks, codes and violation order as the reference
// (/root/reference/proj/core/src/validate.cpp:85-325); the dependency rules are
// restated here independently of sim.cpp so the two cross-check each other.
#include <algorithm>
#include <map>
#include <sstream>
#include <tuple>

#include "seqpipe/validate.hpp"

namespace seqpipe {

std::string violations_to_string(const std::vector<Violation>& vs) {
  std::ostringstream o;
  for (const Violation& v : vs) {
    o << v.code;
    if (v.device > 0) o << " [device " << v.device << "]";
    o << ": " << v.detail << '\n';
  }
  return o.str();
}

namespace {

using Key = std::tuple<int, int, int, int>;  // kind, m, s, stage
Key key(const Task& t) { return {static_cast<int>(t.kind), t.micro_batch, t.segment, t.stage}; }

std::string name(const Task& t) {
  std::ostringstream o;
  o << task_kind_name(t.kind) << "(m=" << t.micro_batch << ",s=" << t.segment << ",stage=" << t.stage << ")";
  return o.str();
}

// What must have run before `t` (independent restatement of the data flow):
// forward <- upstream stage's forward of the same sub-sequence, and the
// previous sub-sequence at this stage (its K/V are this one's prefix);
// backward <- downstream stage's backward, the next sub-sequence's backward
// here (it accumulates into this prefix's dK/dV), and its own forward;
// weight grad <- its input grad.
std::vector<Task> prereqs(const Task& t, int k, int V, int P) {
  std::vector<Task> r;
  if (t.kind == TaskKind::kWeightGrad) {
    r.push_back(make_task(TaskKind::kInputGrad, t.micro_batch, t.segment, t.stage, P));
  } else if (t.kind == TaskKind::kForward) {
    if (t.stage != 1) r.push_back(make_task(TaskKind::kForward, t.micro_batch, t.segment, t.stage - 1, P));
    if (t.segment != 1) r.push_back(make_task(TaskKind::kForward, t.micro_batch, t.segment - 1, t.stage, P));
  } else {
    if (t.stage != V) r.push_back(make_task(t.kind, t.micro_batch, t.segment, t.stage + 1, P));
    if (t.segment != k) r.push_back(make_task(t.kind, t.micro_batch, t.segment + 1, t.stage, P));
    r.push_back(make_task(TaskKind::kForward, t.micro_batch, t.segment, t.stage, P));
  }
  return r;
}

}  // namespace

std::vector<Violation> check_schedule(const Schedule& sch) {
  std::vector<Violation> out;
  const ScenarioConfig& cfg = sch.config;
  const int P = cfg.pipeline_size, k = cfg.segments, M = cfg.micro_batches, V = cfg.total_stages();
  if (static_cast<int>(sch.device_orders.size()) != P) {
    out.push_back({"device_count", 0,
                   "schedule holds " + std::to_string(sch.device_orders.size()) + " device lists, config says " +
                       std::to_string(P)});
    return out;
  }

  // (1) range + placement, counting occurrences.
  std::map<Key, int> seen;
  bool in_range = true;
  for (int d = 1; d <= P; ++d) {
    for (const Task& t : sch.device_orders[static_cast<std::size_t>(d - 1)]) {
      if (t.micro_batch < 1 || t.micro_batch > M || t.segment < 1 || t.segment > k || t.stage < 1 || t.stage > V) {
        out.push_back({"task_out_of_range", d, name(t)});
        in_range = false;
        continue;
      }
      const int owner = (t.stage - 1) % P + 1;
      if (t.device != owner)
        out.push_back({"wrong_device_field", d,
                       name(t) + " carries device " + std::to_string(t.device) + ", stage map says " + std::to_string(owner)});
      if (owner != d) out.push_back({"misplaced_task", d, name(t) + " belongs to device " + std::to_string(owner)});
      ++seen[key(t)];
    }
  }
  if (!in_range) return out;

  auto count = [&](TaskKind kd, int m, int s, int v) {
    auto it = seen.find({static_cast<int>(kd), m, s, v});
    return it == seen.end() ? 0 : it->second;
  };

  // (2) completeness: one F and either one B or one I+W pair per (m, s, stage).
  bool complete = true;
  for (int m = 1; m <= M; ++m)
    for (int s = 1; s <= k; ++s)
      for (int v = 1; v <= V; ++v) {
        const int dev = (v - 1) % P + 1;
        const std::string at = "(m=" + std::to_string(m) + ",s=" + std::to_string(s) + ",stage=" + std::to_string(v) + ")";
        const int f = count(TaskKind::kForward, m, s, v), b = count(TaskKind::kFusedBackward, m, s, v);
        const int i = count(TaskKind::kInputGrad, m, s, v), w = count(TaskKind::kWeightGrad, m, s, v);
        if (f != 1) {
          out.push_back({"completeness", dev, "expected exactly one forward for " + at + ", found " + std::to_string(f)});
          complete = false;
        }
        if (!((b == 1 && i == 0 && w == 0) || (b == 0 && i == 1 && w == 1))) {
          out.push_back({"completeness", dev,
                         "backward units for " + at + " are B=" + std::to_string(b) + " I=" + std::to_string(i) +
                             " W=" + std::to_string(w) + "; expected one fused backward or one input+weight pair"});
          complete = false;
        }
      }

  // (3) every stage accumulates M*k gradient units.
  for (int v = 1; v <= V; ++v) {
    int units = 0;
    for (int m = 1; m <= M; ++m)
      for (int s = 1; s <= k; ++s)
        if (count(TaskKind::kFusedBackward, m, s, v) > 0 || count(TaskKind::kWeightGrad, m, s, v) > 0) ++units;
    if (units != M * k)
      out.push_back({"accumulation_count", (v - 1) % P + 1,
                     "stage " + std::to_string(v) + " accumulates " + std::to_string(units) + " gradient units, expected " +
                         std::to_string(M * k)});
  }

  // (4) per (micro-batch, stage): forwards ascend over segments, backwards descend.
  for (int d = 1; d <= P; ++d) {
    std::map<std::pair<int, int>, int> last_f, last_b;
    for (const Task& t : sch.device_orders[static_cast<std::size_t>(d - 1)]) {
      const std::pair<int, int> mk{t.micro_batch, t.stage};
      if (t.kind == TaskKind::kForward) {
        auto [it, fresh] = last_f.try_emplace(mk, t.segment);
        if (fresh) continue;
        if (t.segment <= it->second)
          out.push_back({"forward_segment_order", d, name(t) + " does not ascend over segment " + std::to_string(it->second)});
        it->second = t.segment;
      } else if (t.kind == TaskKind::kFusedBackward || t.kind == TaskKind::kInputGrad) {
        auto [it, fresh] = last_b.try_emplace(mk, t.segment);
        if (fresh) continue;
        if (t.segment >= it->second)
          out.push_back({"backward_segment_order", d, name(t) + " does not descend under segment " + std::to_string(it->second)});
        it->second = t.segment;
      }
    }
  }

  // (5) zero-cost replay under the checker's dependency rules.
  if (complete) {
    std::map<Key, bool> ran;
    for (const auto& kv : seen) ran[kv.first] = false;
    std::vector<std::size_t> pos(static_cast<std::size_t>(P), 0);
    std::size_t left = 0;
    for (const auto& o : sch.device_orders) left += o.size();
    auto satisfied = [&](const Task& pre) {
      auto it = ran.find(key(pre));
      return it != ran.end() && it->second;
    };
    while (left) {
      bool moved = false;
      for (int d = 1; d <= P; ++d) {
        const auto& order = sch.device_orders[static_cast<std::size_t>(d - 1)];
        std::size_t& c = pos[static_cast<std::size_t>(d - 1)];
        while (c < order.size()) {
          const std::vector<Task> need = prereqs(order[c], k, V, P);
          if (!std::all_of(need.begin(), need.end(), satisfied)) break;
          ran[key(order[c])] = true;
          ++c;
          --left;
          moved = true;
        }
      }
      if (moved) continue;
      for (int d = 1; d <= P; ++d) {
        const auto& order = sch.device_orders[static_cast<std::size_t>(d - 1)];
        const std::size_t c = pos[static_cast<std::size_t>(d - 1)];
        if (c >= order.size()) continue;
        std::ostringstream o;
        o << "task[" << c << "] " << name(order[c]) << " blocked on";
        for (const Task& pre : prereqs(order[c], k, V, P))
          if (!satisfied(pre)) o << ' ' << name(pre);
        out.push_back({"order_deadlock", d, o.str()});
      }
      break;
    }
  }
  return out;
}

std::vector<Violation> check_warmup_formulas(const Schedule& sch) {  // ref validate.cpp:260-325
  const ScenarioConfig& cfg = sch.config;
  const ScheduleKind kind = sch.kind;
  if (kind != ScheduleKind::kOneFOneB && kind != ScheduleKind::kOneFOneBInterleaved && kind != ScheduleKind::kSeq1F1B &&
      kind != ScheduleKind::kSeq1F1BInterleaved)
    throw std::invalid_argument("warm-up formulas apply to the 1F1B-family kinds only");
  if (cfg.micro_batches <= cfg.pipeline_size)
    throw std::invalid_argument("warm-up formulas require micro_batches > pipeline_size");
  const bool seq = is_sequence_level(kind);
  const int per_unit = seq ? 1 : cfg.segments;
  const int units = cfg.micro_batches * cfg.segments * cfg.stages_per_device / per_unit;
  std::vector<Violation> out;
  for (int d = 1; d <= cfg.pipeline_size; ++d) {
    const auto& order = sch.device_orders[static_cast<std::size_t>(d - 1)];
    auto first_bwd = std::find_if(order.begin(), order.end(), [](const Task& t) { return t.kind != TaskKind::kForward; });
    const int fwd = static_cast<int>(first_bwd - order.begin());
    int expect = 0;
    switch (kind) {
      case ScheduleKind::kOneFOneB: expect = warmup_1f1b(cfg.pipeline_size, cfg.micro_batches, d); break;
      case ScheduleKind::kSeq1F1B: expect = warmup_seq1f1b(cfg.pipeline_size, cfg.micro_batches, cfg.segments, d); break;
      case ScheduleKind::kOneFOneBInterleaved: expect = warmup_1f1b_interleaved(cfg.pipeline_size, cfg.stages_per_device, d); break;
      default: expect = warmup_seq1f1b_interleaved(cfg.pipeline_size, cfg.stages_per_device, cfg.segments, d); break;
    }
    expect = std::min(expect, units);
    if (first_bwd == order.end() || fwd % per_unit != 0) {
      out.push_back({"warmup_count", d, "device order has no steady backward or a ragged warm-up block"});
      continue;
    }
    const int flat = expect + (expect < units ? 1 : 0);  // the first steady F precedes the first B
    if (fwd / per_unit != flat)
      out.push_back({"warmup_count", d,
                     "observed " + std::to_string(fwd / per_unit) + " forward units before the first backward, formula expects " +
                         std::to_string(flat) + " (warm-up " + std::to_string(expect) + " + 1 steady forward)"});
  }
  return out;
}

// Pairs in device-order position order of the dependent, prerequisites in prereqs() order
// (the reference's enumeration, validate.cpp:510-528, so seeded picks select the same pairs).
std::vector<DependencyPair> dependency_order_pairs(const Schedule& sch) {
  const ScenarioConfig& cfg = sch.config;
  std::vector<DependencyPair> pairs;
  for (int d = 1; d <= cfg.pipeline_size && d <= static_cast<int>(sch.device_orders.size()); ++d) {
    const auto& order = sch.device_orders[static_cast<size_t>(d - 1)];
    std::map<Key, size_t> at;
    for (size_t i = 0; i < order.size(); ++i) at[key(order[i])] = i;
    for (size_t i = 0; i < order.size(); ++i)
      for (const Task& pre : prereqs(order[i], cfg.segments, cfg.total_stages(), cfg.pipeline_size)) {
        if (pre.device != d) continue;
        const auto it = at.find(key(pre));
        if (it != at.end()) pairs.push_back({d, it->second, i});
      }
  }
  return pairs;
}

Schedule swap_order_pair(const Schedule& sch, const DependencyPair& pair) {
  Schedule out = sch;
  auto& order = out.device_orders.at(static_cast<size_t>(pair.device - 1));
  std::swap(order.at(pair.prerequisite_index), order.at(pair.dependent_index));
  return out;
}

}  // namespace seqpipe
