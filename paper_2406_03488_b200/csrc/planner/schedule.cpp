// Host planner, part 2: schedule generation (reference behaviour:
// /root/reference/proj/core/src/schedule.cpp:38-349).
//
// Non-interleaved kinds use the closed-form op table (op_at). It is the same
// function the GPU launcher kernel evaluates (csrc/cuda/launcher.cu), so the
// host and device tables agree by construction; tests pin both against the
// compiled reference generate().
#include <algorithm>
#include <cctype>
#include <string>

#include "seqpipe/cost.hpp"
#include "seqpipe/schedule.hpp"
#include "seqpipe/sim.hpp"

namespace seqpipe {

const char* schedule_kind_name(ScheduleKind kind) {
  switch (kind) {
    case ScheduleKind::kGPipe: return "gpipe";
    case ScheduleKind::kOneFOneB: return "1f1b";
    case ScheduleKind::kOneFOneBInterleaved: return "1f1b-i";
    case ScheduleKind::kSeq1F1B: return "seq1f1b";
    case ScheduleKind::kSeq1F1BInterleaved: return "seq1f1b-i";
    case ScheduleKind::kZB1P: return "zb1p";
    case ScheduleKind::kSeqZB1P: return "seqzb1p";
  }
  return "?";
}

ScheduleKind parse_schedule_kind(std::string_view name) {
  std::string low;
  for (char c : name) low += static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  for (ScheduleKind k : kAllScheduleKinds)
    if (low == schedule_kind_name(k)) return k;
  throw std::invalid_argument("unknown schedule kind '" + std::string(name) + "'");
}

namespace {
void check_device(int pipeline_size, int device) {
  if (device < 1 || device > pipeline_size) throw std::out_of_range("device index out of range");
}
}  // namespace

// PAPER Eq. 1 (schedule.cpp:38-42): P - i when saturated, else every micro-batch.
int warmup_1f1b(int P, int M, int device) {
  check_device(P, device);
  return M > P ? P - device : M;
}
// PAPER Eq. 4 (schedule.cpp:44-48): k - 1 extra sub-sequence units over 1F1B.
int warmup_seq1f1b(int P, int M, int k, int device) {
  check_device(P, device);
  return M > P ? P - device - 1 + k : M;
}
// PAPER Eq. 5 (schedule.cpp:50-53).
int warmup_1f1b_interleaved(int P, int nv, int device) {
  check_device(P, device);
  return 2 * (P - device) + (nv - 1) * P;
}
// PAPER Eq. 6 (schedule.cpp:55-58).
int warmup_seq1f1b_interleaved(int P, int nv, int k, int device) {
  check_device(P, device);
  return 2 * (P - device) + (nv - 1) * P + k - 1;
}

bool operator==(const Schedule& a, const Schedule& b) {
  return a.config == b.config && a.kind == b.kind && a.device_orders == b.device_orders;
}

// ------------------------------------------------------------------ closed form

OpTableShape op_table_shape(const ScenarioConfig& cfg, ScheduleKind kind) {
  OpTableShape s;
  s.pipeline_size = cfg.pipeline_size;
  s.micro_batches = cfg.micro_batches;
  s.segments = cfg.segments;
  s.seq_level = is_sequence_level(kind);
  s.gpipe = kind == ScheduleKind::kGPipe;
  s.backward_kind = static_cast<int>(is_zero_bubble(kind) ? TaskKind::kInputGrad : TaskKind::kFusedBackward);
  return s;
}

int ops_per_device(const OpTableShape& s) { return 2 * s.micro_batches * s.segments; }

// Position j (0-based) of device d's order. Units are sub-sequences
// (seq-level) or whole micro-batches of k tasks (batch-level). The device
// runs w warm-up forward units, then alternates F, B for U - w units, then
// drains; the partially-ordered queue always pops micro-batches in order and
// segments last-to-first, which is what makes the O(1) form exact (the
// warm-up is >= k-1 units, so a micro-batch is fully queued before its first
// pop). Reference semantics: schedule.cpp:68-126.
Task op_at(const OpTableShape& s, int d, int j) {
  const int P = s.pipeline_size, M = s.micro_batches, k = s.segments;
  const int U = s.seq_level ? M * k : M;
  const int per_unit = s.seq_level ? 1 : k;
  int w = U;
  if (!s.gpipe && M > P) w = s.seq_level ? P - d - 1 + k : P - d;
  w = std::min(w, U);
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
  Task t;
  t.kind = fwd ? TaskKind::kForward : static_cast<TaskKind>(s.backward_kind);
  if (s.seq_level) {
    t.micro_batch = idx / k + 1;
    t.segment = fwd ? idx % k + 1 : k - idx % k;
  } else {
    t.micro_batch = idx + 1;
    t.segment = fwd ? q + 1 : k - q;
  }
  t.stage = d;
  t.device = d;
  return t;
}

namespace {

std::vector<Task> closed_form_order(const ScenarioConfig& cfg, ScheduleKind kind, int device) {
  const OpTableShape s = op_table_shape(cfg, kind);
  const int n = ops_per_device(s);
  std::vector<Task> order(static_cast<std::size_t>(n));
  for (int j = 0; j < n; ++j) order[static_cast<std::size_t>(j)] = op_at(s, device, j);
  return order;
}

// ------------------------------------------------------------------ interleaved
// Units visit every stage chunk in windows of P units: forwards ascend over
// chunks, backwards descend (ref schedule.cpp:128-215; the rotation is every P
// *units*).
struct ChunkUnit {
  int m, s, chunk;  // s == 0: whole micro-batch
};

std::vector<ChunkUnit> windowed(const std::vector<std::pair<int, int>>& flat, int P, int chunks, bool down) {
  std::vector<ChunkUnit> out;
  for (std::size_t w0 = 0; w0 < flat.size(); w0 += static_cast<std::size_t>(P)) {
    const std::size_t w1 = std::min(flat.size(), w0 + static_cast<std::size_t>(P));
    for (int c = 0; c < chunks; ++c)
      for (std::size_t u = w0; u < w1; ++u) out.push_back({flat[u].first, flat[u].second, down ? chunks - 1 - c : c});
  }
  return out;
}

std::vector<Task> interleaved_order(const ScenarioConfig& cfg, ScheduleKind kind, int device) {
  const int P = cfg.pipeline_size, M = cfg.micro_batches, k = cfg.segments, nv = cfg.stages_per_device;
  const bool seq = is_sequence_level(kind);
  std::vector<std::pair<int, int>> fflat, bflat;
  for (int m = 1; m <= M; ++m) {
    if (!seq) {
      fflat.emplace_back(m, 0);
      bflat.emplace_back(m, 0);
      continue;
    }
    for (int s = 1; s <= k; ++s) fflat.emplace_back(m, s);
    for (int s = k; s >= 1; --s) bflat.emplace_back(m, s);
  }
  const std::vector<ChunkUnit> fs = windowed(fflat, P, nv, false), bs = windowed(bflat, P, nv, true);
  const int total = static_cast<int>(fs.size());
  int w = seq ? warmup_seq1f1b_interleaved(P, nv, k, device) : warmup_1f1b_interleaved(P, nv, device);
  w = std::min(w, total);

  std::vector<Task> order;
  auto emit = [&](const ChunkUnit& u, bool fwd) {
    const int stage = device + u.chunk * P;
    const TaskKind kk = fwd ? TaskKind::kForward : TaskKind::kFusedBackward;
    if (seq) {
      order.push_back(make_task(kk, u.m, u.s, stage, P));
    } else {
      for (int i = 1; i <= k; ++i) order.push_back(make_task(kk, u.m, fwd ? i : k + 1 - i, stage, P));
    }
  };
  int fi = 0, bi = 0;
  while (fi < w) emit(fs[static_cast<std::size_t>(fi++)], true);
  while (fi < total) {
    emit(fs[static_cast<std::size_t>(fi++)], true);
    emit(bs[static_cast<std::size_t>(bi++)], false);
  }
  while (bi < total) emit(bs[static_cast<std::size_t>(bi++)], false);
  return order;
}

// ------------------------------------------------------------------ zero bubble
// Weight-gradient placement (ref schedule.cpp:217-309): simulate the F/I
// skeleton, then drop each W (ordered by its I's completion, then position)
// into the earliest idle gap where it fits (first fit within a gap), and
// append the rest back-to-back after the skeleton.
Schedule place_weight_grads(Schedule base, const SequencePartition& part) {
  const ScenarioConfig& cfg = base.config;
  const SimReport rep = simulate(base, part);
  for (std::size_t d = 0; d < base.device_orders.size(); ++d) {
    const std::vector<TaskTiming>& tt = rep.task_times[d];
    if (tt.empty()) continue;
    struct Pending {
      Rational ready, dur;
      Task task;
      std::size_t pos;
      bool done;
    };
    std::vector<Pending> pend;
    for (std::size_t i = 0; i < tt.size(); ++i) {
      if (tt[i].task.kind != TaskKind::kInputGrad) continue;
      Task w = tt[i].task;
      w.kind = TaskKind::kWeightGrad;
      pend.push_back({tt[i].end, task_cost(cfg, part, w), w, i, false});
    }
    std::stable_sort(pend.begin(), pend.end(), [](const Pending& a, const Pending& b) {
      return a.ready != b.ready ? a.ready < b.ready : a.pos < b.pos;
    });
    std::vector<std::pair<Rational, Task>> slots;
    for (const TaskTiming& t : tt) slots.emplace_back(t.start, t.task);
    for (std::size_t i = 1; i < tt.size(); ++i) {
      if (!(tt[i].start > tt[i - 1].end)) continue;
      Rational cur = tt[i - 1].end;
      const Rational gap_end = tt[i].start;
      for (bool placed = true; placed;) {
        placed = false;
        for (Pending& p : pend) {
          if (p.done) continue;
          const Rational st = std::max(cur, p.ready);
          if (st + p.dur > gap_end) continue;
          p.done = placed = true;
          slots.emplace_back(st, p.task);
          cur = st + p.dur;
          break;
        }
      }
    }
    Rational tail = tt.back().end;
    for (Pending& p : pend) {
      if (p.done) continue;
      const Rational st = std::max(tail, p.ready);
      slots.emplace_back(st, p.task);
      tail = st + p.dur;
    }
    std::stable_sort(slots.begin(), slots.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    std::vector<Task>& out = base.device_orders[d];
    out.clear();
    for (const auto& s : slots) out.push_back(s.second);
  }
  return base;
}

}  // namespace

Schedule generate(const ScenarioConfig& cfg, ScheduleKind kind, const SequencePartition& part) {
  cfg.validate();
  if (part.segment_count() != cfg.segments || part.total != cfg.seq_len)
    throw std::invalid_argument("partition does not match the scenario (segments/seq_len)");
  if (is_interleaved(kind)) {
    if (cfg.stages_per_device < 2)
      throw UnsupportedScheduleError(std::string(schedule_kind_name(kind)) + " requires stages_per_device >= 2");
    if (kind == ScheduleKind::kSeq1F1BInterleaved && cfg.segments > cfg.pipeline_size)
      throw UnsupportedScheduleError("seq1f1b-i requires segments <= pipeline_size (warm-up formula infeasible)");
  } else if (cfg.stages_per_device != 1) {
    throw UnsupportedScheduleError(std::string(schedule_kind_name(kind)) + " requires stages_per_device == 1");
  }
  Schedule sch;
  sch.config = cfg;
  sch.kind = kind;
  for (int d = 1; d <= cfg.pipeline_size; ++d)
    sch.device_orders.push_back(is_interleaved(kind) ? interleaved_order(cfg, kind, d) : closed_form_order(cfg, kind, d));
  if (is_zero_bubble(kind)) sch = place_weight_grads(std::move(sch), part);
  return sch;
}

}  // namespace seqpipe
