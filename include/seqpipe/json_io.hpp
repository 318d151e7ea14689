// seqpipe JSON wire formats: the schedule document "seqpipe.schedule.v1" and
// the simulation / measured-execution report "seqpipe.simreport.v1". Same
// signatures and canonical bytes as the reference
// (core/include/seqpipe/json_io.hpp:19-26, core/src/json_io.cpp:59-159):
// objects with sorted keys, exact rational strings, indent-formatted, trailing
// newline, so dump(parse(text)) == text and a schedule emitted here can be fed
// to the reference `seqpipe validate`.
#pragma once

#include <cstddef>
#include <string>

#include "seqpipe/schedule.hpp"
#include "seqpipe/sim.hpp"

namespace seqpipe {

std::string schedule_to_json(const Schedule& schedule, int indent = 2);
Schedule schedule_from_json(const std::string& text);

/// memory_downsample > 0 keeps at most that many points per device (uniform
/// stride, first and last always retained).
std::string report_to_json(const SimReport& report, int indent = 2, std::size_t memory_downsample = 0);

}  // namespace seqpipe
