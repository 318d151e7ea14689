// Point-to-point plan of one device: which tensor crosses which pipeline edge
// before / after each op of the device order. The only exchange steps are the
// pipeline edges of the dependency model (/root/reference/proj/core/src/sim.cpp:
// 20-23 forward activations v -> v+1, :31-33 input gradients v+1 -> v); causal
// and reverse-causal edges (KV prefix, dK/dV) never leave the device.
//
// Channels (one NCCL communicator + stream pairing each):
//   0/1  activations on edges whose lower stage is even/odd
//   2/3  gradients   on edges whose lower stage is even/odd
// A device touches edges (v-1, v) and (v, v+1), which have different parity,
// so it uses each communicator in exactly one direction.
#include "engine/comm_plan.hpp"

namespace spe {

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
      if (t.stage > 1 && dev_of(t.stage - 1) != device) add(0, SP_COMM_RECV, t.stage - 1, (t.stage - 1) % 2);
      if (t.stage < V && dev_of(t.stage + 1) != device) add(1, SP_COMM_SEND, t.stage + 1, t.stage % 2);
    } else if (t.kind == seqpipe::TaskKind::kFusedBackward || t.kind == seqpipe::TaskKind::kInputGrad) {
      if (t.stage < V && dev_of(t.stage + 1) != device) add(0, SP_COMM_RECV, t.stage + 1, 2 + t.stage % 2);
      if (t.stage > 1 && dev_of(t.stage - 1) != device) add(1, SP_COMM_SEND, t.stage - 1, 2 + (t.stage - 1) % 2);
    }
  }
  return out;
}

}  // namespace spe
