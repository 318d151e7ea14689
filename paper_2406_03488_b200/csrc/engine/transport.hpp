// Point-to-point data plane of the multi-rank engine.
//
// The only exchange steps of a Seq1F1B step are the pipeline edges of the
// dependency model (/root/reference/proj/core/src/sim.cpp:20-23 activations
// v -> v+1 after F, :31-33 input gradients v+1 -> v after B). Each edge and
// direction is its own channel (comm_plan.cpp), so every channel has exactly one
// sending rank, one receiving rank and one stream on each side, and the messages
// of a channel are FIFO-ordered identically on both sides (checked when the
// engine is built, comm_plan_check()).
//
// Three transports implement the same stream-ordered send / recv:
//   * NcclTransport  -- production: one NCCL communicator per channel, ncclSend /
//     ncclRecv over NVLink between processes (one process per GPU).
//   * IpcTransport   -- one process per GPU, copies straight into the receiver's memory
//     over CUDA-IPC-mapped rings with flag words (transport_ipc.cu);
//   * LocalTransport -- several engines in one process (one host thread each, on
//     one or more GPUs): the sender copies the message into a hub-owned staging
//     buffer on its stream and records an event; the receiver's stream waits on
//     that event and copies the message out. The receive blocks the HOST thread
//     until the matching send has been enqueued -- a watchdog turns a receive that
//     never matches into seqpipe::DeadlockError (the reference's failure mode for
//     an order that cannot complete, sim.cpp:217-231). The tag of every message
//     (kind, micro-batch, segment, stage of the op that produced it) is checked,
//     so an order mismatch is an error, not silent corruption.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <string>
#include <vector>

namespace spe {

// (kind, micro_batch, segment, stage) of the producing op, packed.
inline uint64_t comm_tag(int kind, int m, int s, int stage) {
  return (static_cast<uint64_t>(kind & 0xff) << 56) | (static_cast<uint64_t>(m & 0xffffff) << 32) |
         (static_cast<uint64_t>(s & 0xffff) << 16) | static_cast<uint64_t>(stage & 0xffff);
}

class Transport {
 public:
  virtual ~Transport() = default;
  virtual const char* name() const = 0;
  // Stream-ordered transfers of `bytes` on `channel` to / from rank `peer`.
  virtual void send(const void* buf, size_t bytes, int peer, int channel, uint64_t tag, cudaStream_t s) = 0;
  virtual void recv(void* buf, size_t bytes, int peer, int channel, uint64_t tag, cudaStream_t s) = 0;
  // Non-blocking receive post: returns false (and posts nothing) when the transport would have to
  // block the host to post it now. NCCL posts are always asynchronous.
  virtual bool try_recv(void* buf, size_t bytes, int peer, int channel, uint64_t tag, cudaStream_t s) = 0;
  // Tear down after a watchdog timeout (NCCL: ncclCommAbort).
  virtual void abort() {}
};

std::unique_ptr<Transport> make_nccl_transport(int world, int rank, const std::vector<std::string>& ids);

// Peer-memory transport (transport_ipc.cu): one process per GPU, the receive rings and flag
// words of every rank exported with CUDA IPC and mapped by its neighbours. Two-phase set-up:
// every rank exports a blob, the blobs travel over any side channel (rank order), then every
// rank connects with all of them.
class IpcExporter : public Transport {
 public:
  virtual std::string export_blob() const = 0;
  // send_peer[c] / recv_peer[c]: peer rank of this rank's send / receive channel c, or -1
  virtual void connect(const std::vector<std::string>& blobs, const std::vector<int>& send_peer,
                       const std::vector<int>& recv_peer) = 0;
};
std::unique_ptr<IpcExporter> make_ipc_transport(int rank, int channels, const std::vector<int>& recv_channels,
                                                size_t slot_bytes, double timeout_s);

struct LocalHub;
std::shared_ptr<LocalHub> make_local_hub(int world, double watchdog_seconds);
// sends_per_step / max_bytes: the rank's sends of one step (its comm plan); that many staging
// slots are reserved for it up front and used in rotation (see transport.cpp).
std::unique_ptr<Transport> make_local_transport(std::shared_ptr<LocalHub> hub, int rank, size_t sends_per_step = 0,
                                                size_t max_bytes = 0);

}  // namespace spe
