// Point-to-point plan of one device: which tensor crosses which pipeline edge
// before / after each op of the device order. The only exchange steps are the
// pipeline edges of the dependency model (/root/reference/proj/core/src/sim.cpp:
// 20-23 forward activations v -> v+1, :31-33 input gradients v+1 -> v); causal
// and reverse-causal edges (KV prefix, dK/dV) never leave the device.
//
// Channels: one per pipeline edge (v, v+1) and direction --
//   2(v-1)      activations of F(., ., v) sent v -> v+1
//   2(v-1) + 1  input gradients of B/I(., ., v+1) sent v+1 -> v
// so every channel has one sender, one receiver and one stream (and NCCL
// communicator) on each side, and the sender's message order is the receiver's
// (both are the stage's F order m-up s-up, or B order m-up s-down), which
// comm_plan_check() verifies for every channel before anything is launched.
// Interleaved schedules (several stages per device) thus never share a FIFO
// between two stage edges of the same device pair.
#include "engine/comm_plan.hpp"

#include <map>
#include <stdexcept>
#include <string>

#include "engine/transport.hpp"

namespace spe {

int comm_channels(const seqpipe::ScenarioConfig& cfg) { return 2 * (cfg.total_stages() - 1); }

std::vector<sp_comm_op> comm_plan(const seqpipe::Schedule& sch, const std::vector<int64_t>& lengths, int device,
                                  int64_t hidden) {
  const seqpipe::ScenarioConfig& cfg = sch.config;
  const int P = cfg.pipeline_size, V = cfg.total_stages();
  std::vector<sp_comm_op> out;
  const auto& order = sch.device_orders.at(static_cast<size_t>(device - 1));
  auto dev_of = [&](int stage) { return (stage - 1) % P + 1; };
  for (size_t i = 0; i < order.size(); ++i) {
    const seqpipe::Task& t = order[i];
    const int64_t elems = lengths.at(static_cast<size_t>(t.segment - 1)) * hidden;
    auto add = [&](int when, int dir, int peer_stage, int channel) {
      sp_comm_op o{};
      o.op_index = static_cast<int32_t>(i);
      o.when = when;
      o.dir = dir;
      o.peer = dev_of(peer_stage) - 1;
      o.channel = channel;
      o.kind = static_cast<int32_t>(t.kind);
      o.micro_batch = t.micro_batch;
      o.segment = t.segment;
      o.stage = t.stage;
      o.elems = elems;
      out.push_back(o);
    };
    if (t.kind == seqpipe::TaskKind::kForward) {
      if (t.stage > 1 && dev_of(t.stage - 1) != device) add(0, SP_COMM_RECV, t.stage - 1, 2 * (t.stage - 2));
      if (t.stage < V && dev_of(t.stage + 1) != device) add(1, SP_COMM_SEND, t.stage + 1, 2 * (t.stage - 1));
    } else if (t.kind == seqpipe::TaskKind::kFusedBackward || t.kind == seqpipe::TaskKind::kInputGrad) {
      if (t.stage < V && dev_of(t.stage + 1) != device) add(0, SP_COMM_RECV, t.stage + 1, 2 * (t.stage - 1) + 1);
      if (t.stage > 1 && dev_of(t.stage - 1) != device) add(1, SP_COMM_SEND, t.stage - 1, 2 * (t.stage - 2) + 1);
    }
  }
  return out;
}

// Message tag of a plan entry: the op that PRODUCES the message (the sender's op).
uint64_t comm_entry_tag(const sp_comm_op& c) {
  const int producer_stage = c.dir == SP_COMM_SEND ? c.stage : (c.kind == 0 ? c.stage - 1 : c.stage + 1);
  const int kind = c.kind == 0 ? 0 : 1;  // F activations; B and I both send input gradients
  return comm_tag(kind, c.micro_batch, c.segment, producer_stage);
}

void comm_plan_check(const seqpipe::Schedule& sch, const std::vector<int64_t>& lengths, int64_t hidden) {
  const int P = sch.config.pipeline_size;
  std::map<int, std::vector<std::pair<uint64_t, int64_t>>> sent, recvd;  // channel -> (tag, elems) in issue order
  for (int d = 1; d <= P; ++d)
    for (const sp_comm_op& c : comm_plan(sch, lengths, d, hidden))
      (c.dir == SP_COMM_SEND ? sent : recvd)[c.channel].push_back({comm_entry_tag(c), c.elems});
  for (const auto& [ch, seq] : sent) {
    auto it = recvd.find(ch);
    if (it == recvd.end() || it->second != seq)
      throw std::logic_error("P2P plan: channel " + std::to_string(ch) +
                             " is not issued in the same order by its sender and its receiver");
  }
  if (sent.size() != recvd.size()) throw std::logic_error("P2P plan: a channel has receives but no sends");
}

}  // namespace spe
