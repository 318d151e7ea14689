// Dependency model + modeled execution (reference: core/include/seqpipe/sim.hpp:21-99,
// core/src/sim.cpp:14-367). The engine (seqpipe/engine.hpp) executes the same op
// tables for real; its measured report reuses the metric definitions below.
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "seqpipe/partition.hpp"
#include "seqpipe/rational.hpp"
#include "seqpipe/scenario.hpp"
#include "seqpipe/schedule.hpp"
#include "seqpipe/task.hpp"

namespace seqpipe {

// F(m,s,v) <- F(m,s,v-1) [pipeline], F(m,s-1,v) [causal: KV prefix]
// B/I(m,s,v) <- B/I(m,s,v+1) [pipeline], B/I(m,s+1,v) [dK/dV of the prefix], F(m,s,v)
// W(m,s,v) <- I(m,s,v)
std::vector<Task> dependencies(const Task& task, const ScenarioConfig& cfg);

// Batch-level kinds hand tensors across stages once per micro-batch: the
// cross-stage edge binds to the unit's last task (reference sim.cpp:54-88).
std::vector<Task> timing_dependencies(const Task& task, const ScenarioConfig& cfg, bool batch_atomic);

struct TaskTiming {
  Task task;
  Rational start{0};
  Rational end{0};
};

struct DeviceReport {
  int device = 1;
  Rational first_start{0};
  Rational last_end{0};
  Rational busy{0};
  Rational idle{0};
  Rational bubble_ratio{0};
  Rational idle_in_makespan{0};
  Rational bubble_ratio_in_makespan{0};
  Rational peak_memory{0};
  std::int64_t peak_allocations = 0;
  int warmup_forward_tasks = 0;
  std::vector<std::pair<Rational, Rational>> memory_series;
};

struct SimReport {
  ScheduleKind kind = ScheduleKind::kOneFOneB;
  ScenarioConfig config;
  std::vector<std::int64_t> partition_lengths;
  std::vector<std::vector<TaskTiming>> task_times;
  Rational makespan{0};
  std::vector<DeviceReport> devices;
  Rational aggregate_bubble_ratio{0};
  Rational aggregate_bubble_ratio_in_makespan{0};
  Rational max_peak_memory{0};
  Rational modeled_throughput{0};
};

struct DeadlockError : std::runtime_error {
  explicit DeadlockError(const std::string& what) : std::runtime_error(what) {}
};
struct MissingDependencyError : std::runtime_error {
  explicit MissingDependencyError(const std::string& what) : std::runtime_error(what) {}
};

SimReport simulate(const Schedule& schedule, const SequencePartition& partition);

// Side-by-side comparison of >= 2 reports (reference sim.hpp:82-99,
// sim.cpp:319-367). Reports must share seq_len and micro_batches unless
// allow_mixed; throws std::invalid_argument otherwise or for < 2 reports.
struct ComparisonRow {
  std::string kind;
  ScenarioConfig config;
  Rational makespan{0};
  Rational bubble_ratio{0};
  Rational max_peak_memory{0};
  Rational throughput{0};
};

struct ComparisonTable {
  std::vector<ComparisonRow> rows;
  // CSV: config columns, the four metrics (6 decimals) and their ratios to the
  // first row (empty where the first row's value is zero).
  std::string to_csv() const;
};

ComparisonTable compare(const std::vector<SimReport>& reports, bool allow_mixed = false);

// Position-level replay order: a topological interleaving of all device
// orders (device-round-robin, each device advancing while its front task is
// ready). The single-GPU engine executes ops in exactly this order.
// Throws DeadlockError if the orders cannot all complete.
std::vector<std::pair<int, int>> replay_order(const Schedule& schedule);

}  // namespace seqpipe
