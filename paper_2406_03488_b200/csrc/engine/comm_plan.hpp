#pragma once

#include <vector>

#include "seqpipe/schedule.hpp"
#include "seqpipe_b200.h"

namespace spe {

// P2P transfers of device `device` (1-based) in issue order; see comm_plan.cpp.
std::vector<sp_comm_op> comm_plan(const seqpipe::Schedule& sch, const std::vector<int64_t>& lengths, int device,
                                  int64_t hidden);

}  // namespace spe
