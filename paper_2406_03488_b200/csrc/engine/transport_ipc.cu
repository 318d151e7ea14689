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
// All of it is enqueued on the caller's stream as stream memory operations (cuStreamWaitValue64 /
// cuStreamWriteValue64: the stream front end waits, no SM spins); a transfer that never pairs up
// is caught by the engine's step watchdog, which releases the waits (abort) and raises
// DeadlockError. Counters grow monotonically across steps.
#include <cuda.h>
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

// Stream memory operations (driver API, resolved once): the stream itself waits on / writes the
// flag word -- no kernel occupies an SM while waiting, so ranks that time-share one GPU (separate
// contexts) and ranks on different GPUs behave the same. The write is ordered after the
// stream's prior work (the ring copy) by the default memory barrier.
using WaitValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
using WriteValue64 = CUresult (*)(CUstream, CUdeviceptr, cuuint64_t, unsigned int);
struct StreamMemOps {
  WaitValue64 wait = nullptr;
  WriteValue64 write = nullptr;
};
const StreamMemOps& mem_ops() {
  static const StreamMemOps ops = [] {
    StreamMemOps o;
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWaitValue64", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      o.wait = reinterpret_cast<WaitValue64>(f);
    f = nullptr;
    if (cudaGetDriverEntryPoint("cuStreamWriteValue64", &f, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      o.write = reinterpret_cast<WriteValue64>(f);
    if (!o.wait || !o.write) throw std::runtime_error("ipc transport: stream memory operations unavailable");
    return o;
  }();
  return ops;
}
void wait_geq(cudaStream_t s, const unsigned long long* flag, unsigned long long v) {
  const CUresult r = mem_ops().wait(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), v,
                                    CU_STREAM_WAIT_VALUE_GEQ);
  if (r != CUDA_SUCCESS) throw ::spk::CudaError("cuStreamWaitValue64 failed: " + std::to_string(static_cast<int>(r)));
}
void write_value(cudaStream_t s, unsigned long long* flag, unsigned long long v) {
  const CUresult r = mem_ops().write(reinterpret_cast<CUstream>(s), reinterpret_cast<CUdeviceptr>(flag), v,
                                     CU_STREAM_WRITE_VALUE_DEFAULT);
  if (r != CUDA_SUCCESS) throw ::spk::CudaError("cuStreamWriteValue64 failed: " + std::to_string(static_cast<int>(r)));
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
      : rank_(rank), C_(channels), slot_bytes_(slot_bytes) {
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
    if (seq >= kIpcSlots) wait_geq(s, flags_ + C_ + channel, seq - kIpcSlots + 1);  // ring slot consumed
    SPK_CUDA(cudaMemcpyAsync(ring + (seq % kIpcSlots) * slot_bytes_, buf, bytes, cudaMemcpyDeviceToDevice, s));
    write_value(s, peer_flags_.at(peer) + channel, seq + 1);  // ready
  }
  void recv(void* buf, size_t bytes, int peer, int channel, uint64_t, cudaStream_t s) override {
    check(channel, bytes);
    auto it = rings_.find(channel);
    if (it == rings_.end() || recv_peer_.at(channel) != peer) throw std::logic_error("ipc: recv on an unconnected channel");
    const unsigned long long seq = recv_seq_[static_cast<size_t>(channel)]++;
    wait_geq(s, flags_ + channel, seq + 1);  // message seq landed
    SPK_CUDA(cudaMemcpyAsync(buf, it->second + (seq % kIpcSlots) * slot_bytes_, bytes, cudaMemcpyDeviceToDevice, s));
    write_value(s, peer_flags_.at(peer) + C_ + channel, seq + 1);  // consumed
  }
  bool try_recv(void* buf, size_t bytes, int peer, int channel, uint64_t tag, cudaStream_t s) override {
    recv(buf, bytes, peer, channel, tag, s);  // posting is asynchronous, like NCCL
    return true;
  }
  // Watchdog (the engine's step timed out): release every stream still waiting on this rank's
  // flag words so the process can tear down and report DeadlockError.
  void abort() override {
    cudaStream_t t = nullptr;
    if (cudaStreamCreateWithFlags(&t, cudaStreamNonBlocking) == cudaSuccess) {
      cudaMemsetAsync(flags_, 0xff, sizeof(unsigned long long) * 2 * C_, t);
      cudaStreamDestroy(t);
    }
  }

 private:
  void check(int channel, size_t bytes) const {
    if (channel < 0 || channel >= C_) throw std::logic_error("ipc: channel out of range");
    if (bytes > slot_bytes_) throw std::logic_error("ipc: message larger than a ring slot");
  }
  int rank_, C_;
  size_t slot_bytes_;
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
