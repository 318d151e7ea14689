// Eq. 8 cost model (reference: /root/reference/proj/core/include/seqpipe/cost.hpp:18-33,
// core/src/cost.cpp:10-55).
//   segment_flops(prefix_before, n) = 2*n*params + 2*L*n*(prefix_before+n)*d   (exact __int128)
//   forward_cost  = segment_flops / total_stages * time_per_flop     (kFlops)
//                 = uniform_forward / (segments * stages_per_device) (kUniform)
//   task_cost     = forward_cost * {1, backward_ratio, bw_input_ratio, bw_weight_ratio}
#pragma once

#include <cstdint>

#include "seqpipe/partition.hpp"
#include "seqpipe/rational.hpp"
#include "seqpipe/scenario.hpp"
#include "seqpipe/task.hpp"

namespace seqpipe {

std::int64_t segment_prefix(const SequencePartition& partition, int i);
detail::Int128 segment_flops(const ScenarioConfig& cfg, std::int64_t prefix_before, std::int64_t length);
Rational forward_cost(const ScenarioConfig& cfg, const SequencePartition& partition, int i);
Rational task_cost(const ScenarioConfig& cfg, const SequencePartition& partition, const Task& task);

}  // namespace seqpipe
