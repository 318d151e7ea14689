// Peer-memory transport of the pipeline P2P data plane (transport.hpp): one process per GPU,
// each rank's receive rings and flag words exported with CUDA IPC and mapped by its
// neighbours, so a message is one device-to-device copy straight into the receiver's
// memory (NVLink between GPUs of a node; the same device when two ranks share a GPU) plus
// two flag words -- no NCCL kernels, no host round trip.
//
// Channel c (one pipeline edge and direction, comm_plan.cpp) with message counter seq:
//   sender:   wait consumed[c] >= seq - R + 1     (its own flag word, written by the receiver)
//             copy buf -> receiver ring slot seq % R
//             ready[c] := seq + 1                 (the receiver's flag word, st.release.sys)
//   receiver: wait ready[c] >= seq + 1            (ld.acquire.sys)
//             copy ring slot -> buf
//             consumed[c] := seq + 1              (the sender's flag word)
// All of it is enqueued on the caller's stream (the waits are one-thread spin kernels with a
// global-timer timeout that traps, so a transfer that never pairs up fails the context instead
// of hanging it). Counters grow monotonically across steps.
#include <cuda_runtime.h>

#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "cuda/common.cuh"
#include "engine/transport.hpp"

namespace spe {
namespace {

constexpr int kIpcSlots = 2;

__global__ void ipc_wait_k(const unsigned long long* flag, unsigned long long target, unsigned long long timeout_ns) {
  unsigned long long t0, t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
  for (;;) {
    unsigned long long v;
    asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(flag) : "memory");
    if (v >= target) return;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    if (t - t0 > timeout_ns) __trap();  // the peer never sent / consumed: fail the context
    __nanosleep(2000);
  }
}

__global__ void ipc_signal_k(unsigned long long* flag, unsigned long long value) {
  __threadfence_system();
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(flag), "l"(value) : "memory");
}

struct BlobHeader {
  int32_t rank, channels, recv_channels, reserved;
  uint64_t slot_bytes;
  cudaIpcMemHandle_t flags;
};
struct BlobChannel {
  int32_t channel, reserved;
  cudaIpcMemHandle_t ring;
};

class IpcTransport final : public IpcExporter {
 public:
  IpcTransport(int rank, int channels, const std::vector<int>& recv_channels, size_t slot_bytes, double timeout_s)
      : rank_(rank), C_(channels), slot_bytes_(slot_bytes), timeout_ns_(static_cast<unsigned long long>(timeout_s * 1e9)) {
    SPK_CUDA(cudaMalloc(&flags_, sizeof(unsigned long long) * 2 * C_));
    SPK_CUDA(cudaMemset(flags_, 0, sizeof(unsigned long long) * 2 * C_));
    for (int c : recv_channels) {
      void* ring = nullptr;
      SPK_CUDA(cudaMalloc(&ring, slot_bytes_ * kIpcSlots));
      rings_[c] = static_cast<uint8_t*>(ring);
    }
    SPK_CUDA(cudaDeviceSynchronize());
    send_seq_.assign(static_cast<size_t>(C_), 0);
    recv_seq_.assign(static_cast<size_t>(C_), 0);
    peer_ring_.assign(static_cast<size_t>(C_), nullptr);
  }
  ~IpcTransport() override {
    for (void* p : opened_) cudaIpcCloseMemHandle(p);
    for (auto& [c, r] : rings_) cudaFree(r);
    if (flags_) cudaFree(flags_);
  }
  const char* name() const override { return "ipc"; }

  std::string export_blob() const override {
    BlobHeader h{};
    h.rank = rank_;
    h.channels = C_;
    h.recv_channels = static_cast<int32_t>(rings_.size());
    h.slot_bytes = slot_bytes_;
    SPK_CUDA(cudaIpcGetMemHandle(&h.flags, flags_));
    std::string out(reinterpret_cast<const char*>(&h), sizeof(h));
    for (const auto& [c, r] : rings_) {
      BlobChannel b{};
      b.channel = c;
      SPK_CUDA(cudaIpcGetMemHandle(&b.ring, r));
      out.append(reinterpret_cast<const char*>(&b), sizeof(b));
    }
    return out;
  }

  // blobs[r] = rank r's export_blob(); send_peer[c] / recv_peer[c]: the peer rank of this
  // rank's send / receive channel c (-1 when it has none).
  void connect(const std::vector<std::string>& blobs, const std::vector<int>& send_peer,
               const std::vector<int>& recv_peer) override {
    std::map<int, const BlobHeader*> head;
    for (const std::string& b : blobs) {
      if (b.size() < sizeof(BlobHeader)) throw std::invalid_argument("ipc: blob too short");
      const auto* h = reinterpret_cast<const BlobHeader*>(b.data());
      if (b.size() != sizeof(BlobHeader) + sizeof(BlobChannel) * static_cast<size_t>(h->recv_channels))
        throw std::invalid_argument("ipc: malformed blob of rank " + std::to_string(h->rank));
      if (h->channels != C_ || h->slot_bytes != slot_bytes_)
        throw std::invalid_argument("ipc: rank " + std::to_string(h->rank) + " has another channel layout");
      head[h->rank] = h;
    }
    auto peer_flags = [&](int p) {
      auto it = peer_flags_.find(p);
      if (it != peer_flags_.end()) return it->second;
      auto hit = head.find(p);
      if (hit == head.end()) throw std::invalid_argument("ipc: no blob from rank " + std::to_string(p));
      void* ptr = nullptr;
      SPK_CUDA(cudaIpcOpenMemHandle(&ptr, hit->second->flags, cudaIpcMemLazyEnablePeerAccess));
      opened_.push_back(ptr);
      return peer_flags_[p] = static_cast<unsigned long long*>(ptr);
    };
    for (int c = 0; c < C_; ++c) {
      const int p = send_peer[static_cast<size_t>(c)];
      if (p >= 0) {
        peer_flags(p);
        const BlobHeader* h = head.at(p);
        const auto* ch = reinterpret_cast<const BlobChannel*>(h + 1);
        void* ptr = nullptr;
        for (int i = 0; i < h->recv_channels; ++i)
          if (ch[i].channel == c) {
            SPK_CUDA(cudaIpcOpenMemHandle(&ptr, ch[i].ring, cudaIpcMemLazyEnablePeerAccess));
            opened_.push_back(ptr);
          }
        if (!ptr) throw std::invalid_argument("ipc: rank " + std::to_string(p) + " exports no ring for channel " +
                                              std::to_string(c));
        peer_ring_[static_cast<size_t>(c)] = static_cast<uint8_t*>(ptr);
        send_peer_[c] = p;
      }
      const int q = recv_peer[static_cast<size_t>(c)];
      if (q >= 0) {
        peer_flags(q);
        recv_peer_[c] = q;
      }
    }
  }

  void send(const void* buf, size_t bytes, int peer, int channel, uint64_t, cudaStream_t s) override {
    check(channel, bytes);
    uint8_t* ring = peer_ring_[static_cast<size_t>(channel)];
    if (!ring || send_peer_.at(channel) != peer) throw std::logic_error("ipc: send on an unconnected channel");
    const unsigned long long seq = send_seq_[static_cast<size_t>(channel)]++;
    if (seq >= kIpcSlots) {
      ipc_wait_k<<<1, 1, 0, s>>>(flags_ + C_ + channel, seq - kIpcSlots + 1, timeout_ns_);
      SPK_LAUNCH_CHECK();
    }
    SPK_CUDA(cudaMemcpyAsync(ring + (seq % kIpcSlots) * slot_bytes_, buf, bytes, cudaMemcpyDeviceToDevice, s));
    ipc_signal_k<<<1, 1, 0, s>>>(peer_flags_.at(peer) + channel, seq + 1);
    SPK_LAUNCH_CHECK();
  }
  void recv(void* buf, size_t bytes, int peer, int channel, uint64_t, cudaStream_t s) override {
    check(channel, bytes);
    auto it = rings_.find(channel);
    if (it == rings_.end() || recv_peer_.at(channel) != peer) throw std::logic_error("ipc: recv on an unconnected channel");
    const unsigned long long seq = recv_seq_[static_cast<size_t>(channel)]++;
    ipc_wait_k<<<1, 1, 0, s>>>(flags_ + channel, seq + 1, timeout_ns_);
    SPK_LAUNCH_CHECK();
    SPK_CUDA(cudaMemcpyAsync(buf, it->second + (seq % kIpcSlots) * slot_bytes_, bytes, cudaMemcpyDeviceToDevice, s));
    ipc_signal_k<<<1, 1, 0, s>>>(peer_flags_.at(peer) + C_ + channel, seq + 1);
    SPK_LAUNCH_CHECK();
  }
  bool try_recv(void* buf, size_t bytes, int peer, int channel, uint64_t tag, cudaStream_t s) override {
    recv(buf, bytes, peer, channel, tag, s);  // posting is asynchronous, like NCCL
    return true;
  }

 private:
  void check(int channel, size_t bytes) const {
    if (channel < 0 || channel >= C_) throw std::logic_error("ipc: channel out of range");
    if (bytes > slot_bytes_) throw std::logic_error("ipc: message larger than a ring slot");
  }
  int rank_, C_;
  size_t slot_bytes_;
  unsigned long long timeout_ns_;
  unsigned long long* flags_ = nullptr;  // [ready x C | consumed x C], written by the peers
  std::map<int, uint8_t*> rings_;        // receive channel -> R slots (exported)
  std::vector<uint8_t*> peer_ring_;      // send channel -> the receiver's ring (mapped)
  std::map<int, unsigned long long*> peer_flags_;
  std::map<int, int> send_peer_, recv_peer_;
  std::vector<unsigned long long> send_seq_, recv_seq_;
  std::vector<void*> opened_;
};

}  // namespace

std::unique_ptr<IpcExporter> make_ipc_transport(int rank, int channels, const std::vector<int>& recv_channels,
                                                size_t slot_bytes, double timeout_s) {
  return std::make_unique<IpcTransport>(rank, channels, recv_channels, slot_bytes, timeout_s);
}

}  // namespace spe
