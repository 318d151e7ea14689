// Shared helpers of the extern "C" layer: exception -> status mapping.
#pragma once

#include <stdexcept>
#include <string>
#include <vector>

#include "seqpipe/partition.hpp"
#include "seqpipe/scenario.hpp"
#include "seqpipe/schedule.hpp"
#include "seqpipe_b200.h"

namespace spc {

// Carries an explicit SP_ERR_* code (CUDA / NCCL failures).
struct SpStatusError : std::runtime_error {
  int code;
  SpStatusError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

void set_error(const std::string& msg);
int map_exception();  // call inside catch(...)

seqpipe::ScenarioConfig from_c(const sp_scenario* c);
void to_c(const seqpipe::ScenarioConfig& s, sp_scenario* c);
seqpipe::Task from_c(const sp_task& t);
sp_task to_c(const seqpipe::Task& t);
seqpipe::ScheduleKind kind_from_c(int32_t k);
seqpipe::SequencePartition partition_from_c(const seqpipe::ScenarioConfig& cfg, const int64_t* lengths, int k);
seqpipe::Schedule schedule_from_c(const seqpipe::ScenarioConfig& cfg, int32_t kind, const sp_task* ops,
                                  const int64_t* counts);
void schedule_to_c(const seqpipe::Schedule& s, sp_task* ops, int64_t* counts);

}  // namespace spc

#define SP_GUARD(...)              \
  try {                            \
    __VA_ARGS__;                   \
    return SP_OK;                  \
  } catch (...) {                  \
    return ::spc::map_exception(); \
  }
