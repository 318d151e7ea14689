// seqpipe partitions: split one micro-batch's sequence into k contiguous segments.
// API of /root/reference/proj/core/include/seqpipe/partition.hpp:21-59.
//   even  — floor(n/k), remainder to the earliest segments (partition.cpp:78-93)
//   cwp   — computation-wise partition: bisection on a common per-segment cost,
//           positive quadratic root per segment, largest-remainder rounding,
//           n_i >= 1 repair (partition.cpp:100-207). Bit-exact with the reference.
//   oracle— exhaustive (test oracle; seq_len <= 512, k <= 4).
#pragma once

#include <cstdint>
#include <string_view>
#include <vector>

#include "seqpipe/rational.hpp"
#include "seqpipe/scenario.hpp"

namespace seqpipe {

struct SequencePartition {
  std::vector<std::int64_t> lengths;
  std::int64_t total = 0;
  Rational imbalance{0};  // (max - min) * k / sum of Eq. 8 segment FLOPs, exact
  int segment_count() const { return static_cast<int>(lengths.size()); }
};

enum class PartitionMode { kEven, kCwp, kOracle };
const char* partition_mode_name(PartitionMode mode);
PartitionMode parse_partition_mode(std::string_view name);

SequencePartition make_partition(std::vector<std::int64_t> lengths, const ScenarioConfig& cfg);
SequencePartition even_partition(std::int64_t n, int k, const ScenarioConfig& cfg);
SequencePartition even_partition(const ScenarioConfig& cfg);
SequencePartition cwp_partition(const ScenarioConfig& cfg);
SequencePartition oracle_partition(const ScenarioConfig& cfg);
SequencePartition partition_for(const ScenarioConfig& cfg, PartitionMode mode);

struct BalanceReport {
  std::vector<Rational> segment_costs;
  Rational imbalance{0};
};
BalanceReport balance_report(const SequencePartition& partition, const ScenarioConfig& cfg);

// Continuous cwp lengths for a common per-segment cost (exposed for the device
// kernel cross-check); same double operation order as the host solver.
std::vector<double> cwp_continuous_lengths(const ScenarioConfig& cfg, double target);

}  // namespace seqpipe
