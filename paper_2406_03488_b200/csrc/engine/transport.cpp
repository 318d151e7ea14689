// NCCL and in-process transports of the pipeline P2P data plane (transport.hpp).
#include "engine/transport.hpp"

#include <nccl.h>

#include <chrono>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <mutex>
#include <stdexcept>
#include <tuple>

#include "cuda/common.cuh"
#include "seqpipe/sim.hpp"

namespace spe {

#define SPE_NCCL(call)                                                                               \
  do {                                                                                               \
    ncclResult_t _r = (call);                                                                        \
    if (_r != ncclSuccess) throw std::runtime_error(std::string("NCCL: ") + ncclGetErrorString(_r)); \
  } while (0)

// ------------------------------------------------------------------ NCCL

namespace {

class NcclTransport final : public Transport {
 public:
  NcclTransport(int world, int rank, const std::vector<std::string>& ids) {
    comms_.assign(ids.size(), nullptr);
    SPE_NCCL(ncclGroupStart());
    for (size_t i = 0; i < ids.size(); ++i) {
      ncclUniqueId id;
      if (ids[i].size() < sizeof(id)) throw std::invalid_argument("NCCL unique id too short");
      std::memcpy(&id, ids[i].data(), sizeof(id));
      SPE_NCCL(ncclCommInitRank(&comms_[i], world, id, rank));
    }
    SPE_NCCL(ncclGroupEnd());
  }
  ~NcclTransport() override {
    for (ncclComm_t c : comms_)
      if (c) ncclCommDestroy(c);
  }
  const char* name() const override { return "nccl"; }
  void send(const void* buf, size_t bytes, int peer, int channel, uint64_t, cudaStream_t s) override {
    SPE_NCCL(ncclSend(buf, bytes, ncclUint8, peer, comm(channel), s));
  }
  void recv(void* buf, size_t bytes, int peer, int channel, uint64_t, cudaStream_t s) override {
    SPE_NCCL(ncclRecv(buf, bytes, ncclUint8, peer, comm(channel), s));
  }
  bool try_recv(void* buf, size_t bytes, int peer, int channel, uint64_t tag, cudaStream_t s) override {
    recv(buf, bytes, peer, channel, tag, s);
    return true;
  }
  void abort() override {
    for (ncclComm_t& c : comms_)
      if (c) {
        ncclCommAbort(c);
        c = nullptr;
      }
  }

 private:
  ncclComm_t comm(int channel) const {
    if (channel < 0 || channel >= static_cast<int>(comms_.size()) || !comms_[static_cast<size_t>(channel)])
      throw std::logic_error("NCCL transport: no communicator for channel " + std::to_string(channel));
    return comms_[static_cast<size_t>(channel)];
  }
  std::vector<ncclComm_t> comms_;
};

}  // namespace

std::unique_ptr<Transport> make_nccl_transport(int world, int rank, const std::vector<std::string>& ids) {
  return std::make_unique<NcclTransport>(world, rank, ids);
}

// ------------------------------------------------------------------ in-process hub

struct LocalHub {
  struct Slot {
    void* ptr = nullptr;
    size_t cap = 0;
    int device = 0;
    cudaEvent_t ready = nullptr;  // recorded on the sender stream after the copy in
    cudaEvent_t freed = nullptr;  // recorded on the receiver stream after the copy out
    bool busy = false, used = false;
    int owner = -1;  // rank that reserved it (its sends only, in a fixed rotation), -1 = shared pool
  };
  struct Msg {
    size_t slot;
    size_t bytes;
    uint64_t tag;
  };
  int world;
  double watchdog_s;
  std::mutex mu;
  std::condition_variable cv;
  std::vector<Slot> slots;
  std::map<std::tuple<int, int, int>, std::deque<Msg>> queues;  // (src, dst, channel) FIFO
  bool aborted = false;

  LocalHub(int w, double wd) : world(w), watchdog_s(wd) {}
  ~LocalHub() {
    for (Slot& s : slots) {
      cudaSetDevice(s.device);
      if (s.ptr) cudaFree(s.ptr);
      if (s.ready) cudaEventDestroy(s.ready);
      if (s.freed) cudaEventDestroy(s.freed);
    }
  }
  // Staging slots owned by one rank, allocated before any step, one per send of its step: the
  // i-th send of a step always uses slot i. A slot shared by all ranks and reused as soon as
  // its receiver had *enqueued* the copy-out made the next sender's stream wait (on the GPU)
  // for that copy-out, which waits for the receiver's compute, which can wait for the next
  // sender -- a cross-rank cycle that hung a 4-stage GPT-2.7B step on one GPU. With owned
  // slots a slot is reused only by the same send of the next step, whose copy-out depends on
  // the previous step alone. (It also keeps cudaMalloc out of the step.)
  std::vector<size_t> reserve(int rank, int dev, size_t n, size_t bytes) {
    std::lock_guard<std::mutex> lk(mu);
    std::vector<size_t> idx;
    for (size_t i = 0; i < n; ++i) {
      Slot s;
      s.cap = bytes;
      s.device = dev;
      s.owner = rank;
      s.busy = true;  // never handed out by acquire()
      idx.push_back(slots.size());
      SPK_CUDA(cudaMalloc(&s.ptr, bytes));
      SPK_CUDA(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
      SPK_CUDA(cudaEventCreateWithFlags(&s.freed, cudaEventDisableTiming));
      slots.push_back(s);
    }
    return idx;
  }
  // A staging buffer of >= bytes on the calling thread's device (caller holds mu).
  size_t acquire(size_t bytes) {
    int dev = 0;
    SPK_CUDA(cudaGetDevice(&dev));
    for (size_t i = 0; i < slots.size(); ++i)
      if (!slots[i].busy && slots[i].cap >= bytes && slots[i].device == dev) {
        slots[i].busy = true;
        return i;
      }
    Slot s;
    s.cap = bytes;
    s.device = dev;
    SPK_CUDA(cudaMalloc(&s.ptr, bytes));
    SPK_CUDA(cudaEventCreateWithFlags(&s.ready, cudaEventDisableTiming));
    SPK_CUDA(cudaEventCreateWithFlags(&s.freed, cudaEventDisableTiming));
    s.busy = true;
    slots.push_back(s);
    return slots.size() - 1;
  }
};

std::shared_ptr<LocalHub> make_local_hub(int world, double watchdog_seconds) {
  if (world < 1) throw std::invalid_argument("local hub: world must be >= 1");
  return std::make_shared<LocalHub>(world, watchdog_seconds);
}

namespace {

std::string tag_str(uint64_t t) {
  static const char* k = "FBIW";
  const int kind = static_cast<int>(t >> 56);
  return std::string(1, kind >= 0 && kind < 4 ? k[kind] : '?') + "(" + std::to_string((t >> 32) & 0xffffff) + "," +
         std::to_string((t >> 16) & 0xffff) + ",stage " + std::to_string(t & 0xffff) + ")";
}

class LocalTransport final : public Transport {
 public:
  LocalTransport(std::shared_ptr<LocalHub> hub, int rank) : hub_(std::move(hub)), rank_(rank) {
    if (rank < 0 || rank >= hub_->world) throw std::invalid_argument("local transport: rank out of range");
  }
  const char* name() const override { return "local"; }

  void send(const void* buf, size_t bytes, int peer, int channel, uint64_t tag, cudaStream_t s) override {
    std::unique_lock<std::mutex> lk(hub_->mu);
    size_t i;
    if (!own_.empty() && hub_->slots[own_[next_ % own_.size()]].cap >= bytes)
      i = own_[next_++ % own_.size()];
    else
      i = hub_->acquire(bytes);
    LocalHub::Slot& sl = hub_->slots[i];
    if (sl.used) SPK_CUDA(cudaStreamWaitEvent(s, sl.freed, 0));  // the previous receiver has copied it out
    SPK_CUDA(cudaMemcpyAsync(sl.ptr, buf, bytes, cudaMemcpyDefault, s));
    SPK_CUDA(cudaEventRecord(sl.ready, s));
    sl.used = true;
    hub_->queues[{rank_, peer, channel}].push_back({i, bytes, tag});
    lk.unlock();
    hub_->cv.notify_all();
  }

  void recv(void* buf, size_t bytes, int peer, int channel, uint64_t tag, cudaStream_t s) override {
    std::unique_lock<std::mutex> lk(hub_->mu);
    auto& q = hub_->queues[{peer, rank_, channel}];
    const auto limit = std::chrono::duration<double>(hub_->watchdog_s);
    if (!hub_->cv.wait_for(lk, limit, [&] { return !q.empty() || hub_->aborted; })) {
      hub_->aborted = true;
      hub_->cv.notify_all();
      throw seqpipe::DeadlockError("P2P watchdog: rank " + std::to_string(rank_) + " waited " +
                                   std::to_string(hub_->watchdog_s) + " s for " + tag_str(tag) + " from rank " +
                                   std::to_string(peer) + " on channel " + std::to_string(channel));
    }
    if (hub_->aborted && q.empty()) throw seqpipe::DeadlockError("P2P aborted: another rank hit the watchdog");
    take(q, buf, bytes, peer, channel, tag, s);
  }

  bool try_recv(void* buf, size_t bytes, int peer, int channel, uint64_t tag, cudaStream_t s) override {
    std::unique_lock<std::mutex> lk(hub_->mu);
    auto& q = hub_->queues[{peer, rank_, channel}];
    if (q.empty()) return false;
    take(q, buf, bytes, peer, channel, tag, s);
    return true;
  }

  void abort() override {
    std::lock_guard<std::mutex> lk(hub_->mu);
    hub_->aborted = true;
    hub_->cv.notify_all();
  }

 private:
  void take(std::deque<LocalHub::Msg>& q, void* buf, size_t bytes, int peer, int channel, uint64_t tag,
            cudaStream_t s) {
    const LocalHub::Msg m = q.front();
    q.pop_front();
    if (m.tag != tag || m.bytes != bytes)
      throw std::logic_error("P2P order mismatch on channel " + std::to_string(channel) + ": rank " +
                             std::to_string(rank_) + " expected " + tag_str(tag) + " (" + std::to_string(bytes) +
                             " B) from rank " + std::to_string(peer) + ", got " + tag_str(m.tag) + " (" +
                             std::to_string(m.bytes) + " B)");
    LocalHub::Slot& sl = hub_->slots[m.slot];
    SPK_CUDA(cudaStreamWaitEvent(s, sl.ready, 0));
    SPK_CUDA(cudaMemcpyAsync(buf, sl.ptr, bytes, cudaMemcpyDefault, s));
    SPK_CUDA(cudaEventRecord(sl.freed, s));
    if (sl.owner < 0) sl.busy = false;
  }

 public:
  std::vector<size_t> own_;  // this rank's reserved slots, used in rotation
  size_t next_ = 0;

 private:
  std::shared_ptr<LocalHub> hub_;
  int rank_;
};

}  // namespace

std::unique_ptr<Transport> make_local_transport(std::shared_ptr<LocalHub> hub, int rank, size_t sends_per_step,
                                                size_t max_bytes) {
  int dev = 0;
  SPK_CUDA(cudaGetDevice(&dev));
  auto t = std::make_unique<LocalTransport>(hub, rank);
  if (sends_per_step) t->own_ = hub->reserve(rank, dev, sends_per_step, max_bytes);
  return t;
}

}  // namespace spe
