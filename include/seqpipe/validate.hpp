// Schedule legality checker (reference: core/include/seqpipe/validate.hpp:17-59,
// core/src/validate.cpp:36-325). Violation codes are the reference's:
// device_count, task_out_of_range, wrong_device_field, misplaced_task,
// completeness, accumulation_count, forward_segment_order,
// backward_segment_order, order_deadlock, warmup_count.
// The engine runs check_schedule on the op log it actually executed.
#pragma once

#include <cstddef>
#include <string>
#include <vector>

#include "seqpipe/schedule.hpp"

namespace seqpipe {

struct Violation {
  std::string code;
  int device = 0;
  std::string detail;
};

std::string violations_to_string(const std::vector<Violation>& violations);
std::vector<Violation> check_schedule(const Schedule& schedule);
std::vector<Violation> check_warmup_formulas(const Schedule& schedule);

// Mutation-based fault injection (reference validate.hpp:50-59, validate.cpp:510-535):
// every same-device (prerequisite, dependent) position pair of a schedule; swapping
// one inverts a dependency, which check_schedule must flag. The engine's executed
// op logs go through the same checker, so the same mutations test it.
struct DependencyPair {
  int device = 1;  // 1-based
  std::size_t prerequisite_index = 0;
  std::size_t dependent_index = 0;
};

std::vector<DependencyPair> dependency_order_pairs(const Schedule& schedule);
Schedule swap_order_pair(const Schedule& schedule, const DependencyPair& pair);

}  // namespace seqpipe
