#pragma once

#include <vector>

#include "seqpipe/schedule.hpp"
#include "seqpipe_b200.h"

namespace spe {

// P2P transfers of device `device` (1-based) in issue order; see comm_plan.cpp.
std::vector<sp_comm_op> comm_plan(const seqpipe::Schedule& sch, const std::vector<int64_t>& lengths, int device,
                                  int64_t hidden);
// Number of channels (pipeline edges x 2 directions).
int comm_channels(const seqpipe::ScenarioConfig& cfg);
// Tag (transport.hpp comm_tag) of the message a plan entry sends or receives.
uint64_t comm_entry_tag(const sp_comm_op& c);
// Throws std::logic_error unless, on every channel, the receiver posts exactly the
// sender's messages in the sender's order (FIFO pairing by construction).
void comm_plan_check(const seqpipe::Schedule& sch, const std::vector<int64_t>& lengths, int64_t hidden);

}  // namespace spe
