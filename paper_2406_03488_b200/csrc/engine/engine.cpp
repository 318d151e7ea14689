// Engine: executes the op table of one device (or of every device, when a
// single process drives all stages on one GPU) and measures it.
//
// Multi-rank (world == pipeline_size): rank r drives device r+1. The only
// exchange steps are the pipeline edges of the dependency model
// (/root/reference/proj/core/src/sim.cpp:20-23, :31-33): after F(m,s,v) the
// stage output goes to v+1, after B(m,s,v) the input gradient goes to v-1.
// They run through a Transport (transport.hpp: NCCL between processes, or an
// in-process hub between engines driven by separate host threads), one channel
// per edge and direction, each with its own stream on each side. Receives are
// posted ahead into per-channel staging slots and copied into the op's input
// on the compute stream right before the op, so a receive never waits for
// unrelated compute; sends are enqueued on the channel's stream after the
// producing op and never block compute.
//
// Single rank: the step body (every op + the optimizer) can be captured once
// into a CUDA graph and replayed (enable_graph). For gpipe / 1f1b / seq1f1b the
// op table the engine executes is the one the GPU-resident launcher kernel
// generates (launcher.cu, the closed form of schedule.cpp:68-126), checked
// bit-for-bit against the host generate() before it is used.
#include "engine/engine.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <thread>

#include "engine/comm_plan.hpp"
#include "seqpipe/sim.hpp"
#include "seqpipe/validate.hpp"

namespace spk {
std::vector<sp_task> device_op_table(const seqpipe::ScenarioConfig& cfg, seqpipe::ScheduleKind kind, int dev);
}

namespace spe {

namespace {

bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  SPK_CUDA(cudaStreamIsCapturing(s, &st));
  return st == cudaStreamCaptureStatusActive;
}

// Timeline events must survive graph capture as event-record nodes (not capture-internal
// dependency markers), so they are recorded as external events while capturing.
void record_timing(cudaEvent_t e, cudaStream_t s) {
  SPK_CUDA(cudaEventRecordWithFlags(e, s, capturing(s) ? cudaEventRecordExternal : cudaEventRecordDefault));
}

seqpipe::Schedule schedule_from_device(const seqpipe::ScenarioConfig& cfg, seqpipe::ScheduleKind kind, int dev) {
  const std::vector<sp_task> flat = spk::device_op_table(cfg, kind, dev);
  seqpipe::Schedule s;
  s.config = cfg;
  s.kind = kind;
  const size_t per = flat.size() / static_cast<size_t>(cfg.pipeline_size);
  s.device_orders.assign(static_cast<size_t>(cfg.pipeline_size), {});
  for (size_t i = 0; i < flat.size(); ++i) {
    const sp_task& t = flat[i];
    s.device_orders[i / per].push_back(seqpipe::Task{static_cast<seqpipe::TaskKind>(t.kind), t.micro_batch, t.segment,
                                                     t.stage, t.device});
  }
  return s;
}

}  // namespace

Engine::Engine(const seqpipe::ScenarioConfig& cfg, seqpipe::ScheduleKind kind, const std::vector<int64_t>& lengths,
               const ModelCfg& m, int rank, int world, int cuda_device)
    : cfg_(cfg), kind_(kind), len_(lengths), mc_(m), rank_(rank), world_(world), dev_(cuda_device) {
  cfg_.validate();
  if (world != 1 && world != cfg.pipeline_size)
    throw std::invalid_argument("world_size must be 1 (all stages in-process) or pipeline_size");
  if (rank < 0 || rank >= world) throw std::invalid_argument("rank out of range");
  if (mc_.h != mc_.H * mc_.hd) throw std::invalid_argument("hidden must equal heads * head_dim");
  if ((mc_.flags & SP_FLAG_RECOMPUTE_MLP) && seqpipe::is_zero_bubble(kind))
    throw std::invalid_argument("SP_FLAG_RECOMPUTE_MLP: the zero-bubble kinds keep the MLP operands for W");
  if (mc_.family == SP_MODEL_GPT && mc_.max_seq < cfg.seq_len) throw std::invalid_argument("max_seq < seq_len");
  if (mc_.dt == DType::kBF16) {  // production mode runs tensor-core kernels only: refuse shapes they cannot take
    if (!(mc_.flags & SP_FLAG_NO_TC_ATTN) && mc_.hd != 64 && mc_.hd != 80 && mc_.hd != 128)
      throw std::invalid_argument("bf16 mode: tensor-core attention supports head_dim 64, 80 or 128");
    if (!(mc_.flags & SP_FLAG_NO_TCGEN05) && (mc_.h % 8 || mc_.F % 8))
      throw std::invalid_argument("bf16 mode: hidden and ffn must be multiples of 8 (TMA row strides)");
  }
  if (const char* w = std::getenv("SP_P2P_WATCHDOG_S")) watchdog_s_ = std::atof(w);
  SPK_CUDA(cudaSetDevice(dev_));
  const seqpipe::SequencePartition part = seqpipe::make_partition(len_, cfg_);
  sched_ = seqpipe::generate(cfg_, kind_, part);
  if (!seqpipe::is_interleaved(kind_) && !seqpipe::is_zero_bubble(kind_)) {
    // GPU-resident launcher: the op table comes from the closed-form device kernel; the host
    // generate() (POQ, schedule.cpp:68-126) is the cross-check, bit for bit.
    seqpipe::Schedule dev_sched = schedule_from_device(cfg_, kind_, dev_);
    if (!(dev_sched == sched_)) throw std::logic_error("device op table differs from generate()");
    sched_ = std::move(dev_sched);
    table_from_device_ = true;
  }
  const auto viol = seqpipe::check_schedule(sched_);
  if (!viol.empty()) throw std::logic_error("generated schedule failed validation:\n" + seqpipe::violations_to_string(viol));

  SPK_CUDA(cudaStreamCreateWithFlags(&s_, cudaStreamNonBlocking));
  const int V = cfg_.total_stages();
  std::vector<int> my_devices;
  if (world_ == 1) {
    for (int d = 1; d <= cfg_.pipeline_size; ++d) my_devices.push_back(d);
  } else {
    my_devices.push_back(rank_ + 1);
  }
  for (int v = 1; v <= V; ++v) {
    const int d = (v - 1) % cfg_.pipeline_size + 1;
    if (std::find(my_devices.begin(), my_devices.end(), d) == my_devices.end()) continue;
    stages_[v] = std::make_unique<Stage>(mc_, cfg_, len_, v, V, s_);
  }
  for (auto& [v, st] : stages_) {
    const int d = (v - 1) % cfg_.pipeline_size + 1;
    st->plan_arena(sched_.device_orders[static_cast<size_t>(d - 1)]);
    st->probe = &probe_;
  }
  // Execution order of this process: dependency-respecting interleaving of its device orders.
  if (world_ == 1) {
    replay_ = seqpipe::replay_order(sched_);
  } else {
    comm_plan_check(sched_, len_, mc_.h);  // FIFO pairing of every channel, by construction
    const auto& order = sched_.device_orders[static_cast<size_t>(rank_)];
    for (size_t j = 0; j < order.size(); ++j) replay_.emplace_back(rank_, static_cast<int>(j));
    plan_ = comm_plan(sched_, len_, rank_ + 1, mc_.h);
    plan_pre_.assign(order.size(), {});
    plan_post_.assign(order.size(), {});
    for (const sp_comm_op& c : plan_)
      (c.when == 0 ? plan_pre_ : plan_post_)[static_cast<size_t>(c.op_index)].push_back(c);
  }
  // In-process stage hand-off: F(m,s,v) copies stage v-1's output into its own layer-0
  // input slot (exec_op). Aliasing the two is unsafe for the zero-bubble kinds: W(m,s,v)
  // still reads x_in[0] after W(m,s,v-1) may have freed stage v-1's record (only I, not W,
  // is ordered by the dependency rules, sim.cpp:29-41).
  const size_t tok_bytes = sizeof(int32_t) * cfg_.micro_batches * (cfg_.seq_len + 1);
  SPK_CUDA(cudaMalloc(&tokens_owned_, tok_bytes));
  SPK_CUDA(cudaMalloc(&loss_dev_, sizeof(double)));
  SPK_CUDA(cudaMalloc(&adam_bc_dev_, 2 * sizeof(float)));
  SPK_CUDA(cudaMallocHost(&adam_bc_host_, 2 * sizeof(float)));
  SPK_CUDA(cudaMallocHost(&loss_host_, sizeof(double)));
  const size_t nops = replay_.size();
  ev_start_.resize(nops);
  ev_end_.resize(nops);
  for (size_t i = 0; i < nops; ++i) {
    SPK_CUDA(cudaEventCreate(&ev_start_[i]));
    SPK_CUDA(cudaEventCreate(&ev_end_[i]));
  }
  SPK_CUDA(cudaEventCreate(&ev_step0_));
  SPK_CUDA(cudaEventCreate(&ev_step1_));
  SPK_CUDA(cudaEventCreateWithFlags(&ev_tmp_, cudaEventDisableTiming));
  SPK_CUDA(cudaStreamSynchronize(s_));
}

Engine::~Engine() {
  cudaSetDevice(dev_);
  if (poisoned_) {
    // After a P2P watchdog: streams may stay parked on a peer that will never answer. Leak the
    // device state instead of blocking in a synchronize or an implicitly synchronizing free;
    // the process is expected to exit (the reference raises DeadlockError and stops too).
    for (auto& [v, st] : stages_) (void)st.release();
    (void)transport_.release();
    (void)cudaGetLastError();
    return;
  }
  if (s_) cudaStreamSynchronize(s_);
  for (auto& [c, st] : send_s_) cudaStreamSynchronize(st);
  for (auto& [c, rc] : recv_ch_) cudaStreamSynchronize(rc.s);
  transport_.reset();
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (graph_) cudaGraphDestroy(graph_);
  stages_.clear();
  for (auto e : ev_start_) cudaEventDestroy(e);
  for (auto e : ev_end_) cudaEventDestroy(e);
  for (auto e : send_ring_ev_) cudaEventDestroy(e);
  for (auto e : act_sent_)
    if (e) cudaEventDestroy(e);  // only the F-send slots hold events
  for (auto p : send_ring_) cudaFree(p);
  for (auto& [c, rc] : recv_ch_) {
    for (void* p : rc.slot) cudaFree(p);
    for (auto e : rc.done) cudaEventDestroy(e);
    for (auto e : rc.freed) cudaEventDestroy(e);
    cudaStreamDestroy(rc.s);
  }
  for (auto& [c, st] : send_s_) cudaStreamDestroy(st);
  if (ev_step0_) cudaEventDestroy(ev_step0_);
  if (ev_step1_) cudaEventDestroy(ev_step1_);
  if (ev_tmp_) cudaEventDestroy(ev_tmp_);
  if (tokens_owned_) cudaFree(tokens_owned_);
  if (loss_dev_) cudaFree(loss_dev_);
  if (adam_bc_dev_) cudaFree(adam_bc_dev_);
  if (adam_bc_host_) cudaFreeHost(adam_bc_host_);
  if (loss_host_) cudaFreeHost(loss_host_);
  if (s_) cudaStreamDestroy(s_);
  (void)cudaGetLastError();  // teardown errors must not surface in the next API call of this thread
}

int Engine::comm_channels() const { return spe::comm_channels(cfg_); }

void Engine::comm_init(const std::vector<std::string>& ids) {
  if (world_ == 1) return;
  if (static_cast<int>(ids.size()) != comm_channels())
    throw std::invalid_argument("comm_init expects one NCCL unique id per channel (" + std::to_string(comm_channels()) +
                                ")");
  SPK_CUDA(cudaSetDevice(dev_));
  transport_ = make_nccl_transport(world_, rank_, ids);
  comm_ready_setup();
}

std::string Engine::ipc_export() {
  if (world_ == 1) throw std::logic_error("ipc_export: world size 1 has no transfers");
  if (ipc_) return ipc_blob_;  // exported already (a size query, then the copy)
  SPK_CUDA(cudaSetDevice(dev_));
  std::vector<int> recv_channels;
  size_t max_bytes = 0;
  for (const sp_comm_op& c : plan_) {
    max_bytes = std::max(max_bytes, spk::dtype_size(mc_.dt) * static_cast<size_t>(c.elems));
    if (c.dir == SP_COMM_RECV && std::find(recv_channels.begin(), recv_channels.end(), c.channel) == recv_channels.end())
      recv_channels.push_back(c.channel);
  }
  // every rank must size its rings alike: the largest message of any rank is a segment's [n, h]
  int64_t nmax = 0;
  for (int64_t n : len_) nmax = std::max(nmax, n);
  max_bytes = std::max(max_bytes, spk::dtype_size(mc_.dt) * static_cast<size_t>(nmax) * static_cast<size_t>(mc_.h));
  auto t = make_ipc_transport(rank_, comm_channels(), recv_channels, max_bytes, watchdog_s_);
  ipc_blob_ = t->export_blob();
  ipc_ = t.get();
  transport_ = std::move(t);
  return ipc_blob_;
}

void Engine::ipc_connect(const std::vector<std::string>& blobs) {
  if (!ipc_) throw std::logic_error("ipc_connect: call ipc_export first");
  if (static_cast<int>(blobs.size()) != world_) throw std::invalid_argument("ipc_connect expects one blob per rank");
  SPK_CUDA(cudaSetDevice(dev_));
  std::vector<int> send_peer(static_cast<size_t>(comm_channels()), -1), recv_peer(send_peer);
  for (const sp_comm_op& c : plan_)
    (c.dir == SP_COMM_SEND ? send_peer : recv_peer)[static_cast<size_t>(c.channel)] = c.peer;
  ipc_->connect(blobs, send_peer, recv_peer);
  ipc_ = nullptr;
  comm_ready_setup();
}

void Engine::attach_local(std::shared_ptr<LocalHub> hub) {
  if (world_ == 1) return;
  SPK_CUDA(cudaSetDevice(dev_));
  size_t sends = 0, max_bytes = 0;
  for (const sp_comm_op& c : plan_)
    if (c.dir == SP_COMM_SEND) {
      ++sends;
      max_bytes = std::max(max_bytes, spk::dtype_size(mc_.dt) * static_cast<size_t>(c.elems));
    }
  transport_ = make_local_transport(std::move(hub), rank_, sends, max_bytes);
  local_transport_ = true;
  comm_ready_setup();
}

// Streams, staging slots and events of this rank's channels.
void Engine::comm_ready_setup() {
  spk::preload_kernels();  // no lazy kernel load may stall a launch behind a parked receive (ops.h)
  const int64_t nmax = *std::max_element(len_.begin(), len_.end());
  const size_t max_bytes = spk::dtype_size(mc_.dt) * nmax * mc_.h;
  for (const sp_comm_op& c : plan_) {
    if (c.dir == SP_COMM_SEND) {
      if (!send_s_.count(c.channel)) {
        cudaStream_t st;
        SPK_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
        send_s_[c.channel] = st;
      }
      continue;
    }
    if (recv_ch_.count(c.channel)) continue;
    RecvChannel& rc = recv_ch_[c.channel];
    rc.peer = c.peer;
    SPK_CUDA(cudaStreamCreateWithFlags(&rc.s, cudaStreamNonBlocking));
    for (int i = 0; i < kRecvSlots; ++i) {
      void* p = nullptr;
      SPK_CUDA(cudaMalloc(&p, max_bytes));
      rc.slot.push_back(p);
      cudaEvent_t a, b;
      SPK_CUDA(cudaEventCreateWithFlags(&a, cudaEventDisableTiming));
      SPK_CUDA(cudaEventCreateWithFlags(&b, cudaEventDisableTiming));
      SPK_CUDA(cudaEventRecord(b, s_));  // slots start free
      rc.done.push_back(a);
      rc.freed.push_back(b);
    }
  }
  for (const sp_comm_op& c : plan_)
    if (c.dir == SP_COMM_RECV) recv_ch_[c.channel].msgs.push_back(&c);
  // Gradient send ring: a slot is reused only after its previous send completed.
  for (int i = 0; i < 4; ++i) {
    void* p = nullptr;
    SPK_CUDA(cudaMalloc(&p, max_bytes));
    send_ring_.push_back(p);
    cudaEvent_t e;
    SPK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SPK_CUDA(cudaEventRecord(e, s_));
    send_ring_ev_.push_back(e);
  }
  act_sent_.assign(static_cast<size_t>(cfg_.total_stages() + 1) * cfg_.micro_batches * cfg_.segments, nullptr);
  for (const sp_comm_op& c : plan_)
    if (c.dir == SP_COMM_SEND && c.kind == SP_TASK_F) {
      cudaEvent_t& e = act_sent_[(static_cast<size_t>(c.stage) * cfg_.micro_batches + (c.micro_batch - 1)) *
                                     cfg_.segments + (c.segment - 1)];
      SPK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
  SPK_CUDA(cudaStreamSynchronize(s_));
}

// Posts this step's receives of one channel into its staging slots, up to kRecvSlots ahead of
// the consumer. block_for_next: the next unconsumed message is needed now (a blocking post).
void Engine::post_recvs(RecvChannel& rc, int ch, bool block_for_next) {
  while (rc.posted < rc.msgs.size() && rc.posted < rc.consumed + kRecvSlots) {
    const size_t i = rc.posted, slot = i % kRecvSlots;
    const sp_comm_op& c = *rc.msgs[i];
    const size_t bytes = spk::dtype_size(mc_.dt) * static_cast<size_t>(c.elems);
    SPK_CUDA(cudaStreamWaitEvent(rc.s, rc.freed[slot], 0));  // message i - kRecvSlots copied out
    const uint64_t tag = comm_entry_tag(c);
    if (block_for_next && i == rc.consumed) {
      transport_->recv(rc.slot[slot], bytes, rc.peer, ch, tag, rc.s);
    } else if (!transport_->try_recv(rc.slot[slot], bytes, rc.peer, ch, tag, rc.s)) {
      break;
    }
    SPK_CUDA(cudaEventRecord(rc.done[slot], rc.s));
    ++rc.posted;
  }
}

// Executes op `t` (position `pos` of its device order, `i`-th op of this step).
void Engine::exec_op(const seqpipe::Task& t, int i, int pos) {
  Stage* st = stage_obj(t.stage);
  Stage::Seg& sg = st->seg(t.micro_batch, t.segment);
  const bool fwd = t.kind == seqpipe::TaskKind::kForward;
  const size_t esz = spk::dtype_size(mc_.dt);
  if (t.kind == seqpipe::TaskKind::kWeightGrad) {  // zero-bubble W: local weight-gradient GEMMs, no transfers
    record_timing(ev_start_[i], s_);
    st->backward_weight(t.micro_batch, t.segment);
    record_timing(ev_end_[i], s_);
    return;
  }
  const bool input_only = t.kind == seqpipe::TaskKind::kInputGrad;  // zero-bubble I: B without the W GEMMs
  const std::vector<sp_comm_op>* post = nullptr;
  if (world_ > 1) {
    for (const sp_comm_op& c : plan_pre_[static_cast<size_t>(pos)]) {  // the op's input from the peer
      RecvChannel& rc = recv_ch_.at(c.channel);
      // plan_pre_ holds copies of the plan entries: compare the message, not its address.
      if (rc.consumed >= rc.msgs.size() || rc.msgs[rc.consumed]->op_index != c.op_index ||
          comm_entry_tag(*rc.msgs[rc.consumed]) != comm_entry_tag(c))
        throw std::logic_error("P2P: receive consumed out of plan order");
      post_recvs(rc, c.channel, /*block_for_next=*/true);
      const size_t slot = rc.consumed % kRecvSlots;
      SPK_CUDA(cudaStreamWaitEvent(s_, rc.done[slot], 0));
      SPK_CUDA(cudaMemcpyAsync(fwd ? sg.x_in[0] : sg.dy_in, rc.slot[slot], esz * static_cast<size_t>(c.elems),
                               cudaMemcpyDeviceToDevice, s_));
      SPK_CUDA(cudaEventRecord(rc.freed[slot], s_));
      ++rc.consumed;
      post_recvs(rc, c.channel, false);  // prefetch the channel's next messages
    }
    post = &plan_post_[static_cast<size_t>(pos)];
    if (!fwd && !act_sent_.empty()) {  // the record's stage output must have left before the record is reused
      cudaEvent_t e = act_sent_[(static_cast<size_t>(t.stage) * cfg_.micro_batches + (t.micro_batch - 1)) *
                                    cfg_.segments + (t.segment - 1)];
      if (e) SPK_CUDA(cudaStreamWaitEvent(s_, e, 0));
    }
  }
  if (fwd) {
    record_timing(ev_start_[i], s_);
    if (world_ == 1 && t.stage > 1) {
      const Stage::Seg& up = stage_obj(t.stage - 1)->seg(t.micro_batch, t.segment);
      SPK_CUDA(cudaMemcpyAsync(sg.x_in[0], up.x_out, esz * sg.n * mc_.h, cudaMemcpyDeviceToDevice, s_));
    }
    st->forward(t.micro_batch, t.segment, tokens_dev_, loss_dev_, 1.0f / (float)(cfg_.micro_batches * cfg_.seq_len));
    record_timing(ev_end_[i], s_);
    if (post)
      for (const sp_comm_op& c : *post) {
        cudaStream_t ss = send_s_.at(c.channel);
        SPK_CUDA(cudaStreamWaitEvent(ss, ev_end_[i], 0));
        transport_->send(sg.x_out, esz * static_cast<size_t>(c.elems), c.peer, c.channel, comm_entry_tag(c), ss);
        SPK_CUDA(cudaEventRecord(act_sent_[(static_cast<size_t>(t.stage) * cfg_.micro_batches + (t.micro_batch - 1)) *
                                               cfg_.segments + (t.segment - 1)],
                                 ss));
      }
    return;
  }
  void* dx_target = nullptr;
  int slot = -1;
  if (post && !post->empty()) {
    slot = send_ring_next_;
    send_ring_next_ = (send_ring_next_ + 1) % static_cast<int>(send_ring_.size());
    SPK_CUDA(cudaStreamWaitEvent(s_, send_ring_ev_[static_cast<size_t>(slot)], 0));
    dx_target = send_ring_[static_cast<size_t>(slot)];
  } else if (t.stage > 1) {
    dx_target = stage_obj(t.stage - 1)->seg(t.micro_batch, t.segment).dy_in;  // in-process hand-off
  }
  record_timing(ev_start_[i], s_);
  if (input_only)
    st->backward_input(t.micro_batch, t.segment, dx_target, tokens_dev_);
  else
    st->backward(t.micro_batch, t.segment, dx_target, tokens_dev_);
  record_timing(ev_end_[i], s_);
  if (slot >= 0) {
    for (const sp_comm_op& c : *post) {
      cudaStream_t ss = send_s_.at(c.channel);
      SPK_CUDA(cudaStreamWaitEvent(ss, ev_end_[i], 0));
      transport_->send(dx_target, esz * static_cast<size_t>(c.elems), c.peer, c.channel, comm_entry_tag(c), ss);
      SPK_CUDA(cudaEventRecord(send_ring_ev_[static_cast<size_t>(slot)], ss));
    }
  }
}

// The step body: loss / gradient reset, every op of this process in order, the P2P drain and
// the optimizer -- all on the engine streams (and capturable as one CUDA graph at world 1).
void Engine::enqueue_ops() {
  SPK_CUDA(cudaMemsetAsync(loss_dev_, 0, sizeof(double), s_));
  for (auto& [v, st] : stages_) st->zero_grads();
  for (auto& [c, rc] : recv_ch_) {
    rc.posted = rc.consumed = 0;
    post_recvs(rc, c, false);  // receives in flight before the first op needs them
  }
  op_log_.clear();
  for (size_t i = 0; i < replay_.size(); ++i) {
    const auto [d, j] = replay_[i];
    const seqpipe::Task& t = sched_.device_orders[static_cast<size_t>(d)][static_cast<size_t>(j)];
    exec_op(t, static_cast<int>(i), j);
    op_log_.push_back(t);
  }
  for (auto& [c, rc] : recv_ch_)
    if (rc.consumed != rc.msgs.size()) throw std::logic_error("P2P: a planned receive was never consumed");
  for (auto& [c, ss] : send_s_) {  // the step ends when this device's sends have drained
    SPK_CUDA(cudaEventRecord(ev_tmp_, ss));
    SPK_CUDA(cudaStreamWaitEvent(s_, ev_tmp_, 0));
  }
  for (auto& [v, st] : stages_) st->optimizer_step(adam_bc_dev_);
}

void Engine::drop_graph() {
  if (graph_exec_) SPK_CUDA(cudaGraphExecDestroy(graph_exec_));
  if (graph_) SPK_CUDA(cudaGraphDestroy(graph_));
  graph_exec_ = nullptr;
  graph_ = nullptr;
}

void Engine::enable_graph(bool on) {
  graph_wanted_ = on && world_ == 1;
  if (!graph_wanted_) drop_graph();
}

void Engine::step(const int32_t* tokens, bool on_device, sp_step_report* rep) {
  if (poisoned_)
    throw seqpipe::DeadlockError("engine unusable after a P2P watchdog timeout: destroy it and restart the job");
  SPK_CUDA(cudaSetDevice(dev_));
  if (world_ > 1 && !transport_)
    throw std::logic_error("multi-rank engine: call sp_engine_comm_init / sp_engine_attach_local first");
  // Several engines on one GPU (in-process transport, one host thread each): their 2-CTA
  // GEMMs run concurrently, and a cta_group::2 cluster then intermittently stopped in its
  // first cluster barrier with one CTA's TMEM allocation never completing (cuda-gdb: the
  // only kernel left on the GPU; 3 of 4 runs of a 3-stage GPT-2.7B step without side
  // streams, 0 of 8 with the 1-CTA GEMM). These engines use the 1-CTA GEMM; one engine per
  // GPU (P = 1, or one process per GPU over NCCL) keeps the 2-CTA kernel.
  spk::set_gemm_single_cta(local_transport_);
  ++step_no_;
  adam_bc_host_[0] = 1.f - std::pow(mc_.b1, static_cast<float>(step_no_));
  adam_bc_host_[1] = 1.f - std::pow(mc_.b2, static_cast<float>(step_no_));
  probe_.enabled = (mc_.flags & SP_FLAG_KPROBE) != 0;
  probe_.reset();
  const bool use_graph = graph_wanted_ && !probe_.enabled;  // probes time kernels eagerly
  if (use_graph && graph_exec_ && graph_flags_ != mc_.flags) drop_graph();  // recapture for the new flags
  SPK_CUDA(cudaEventRecord(ev_step0_, s_));
  const size_t tok_bytes = sizeof(int32_t) * cfg_.micro_batches * (cfg_.seq_len + 1);
  if (on_device && !use_graph) {
    tokens_dev_ = const_cast<int32_t*>(tokens);
  } else {  // the graph reads the engine's own token buffer
    SPK_CUDA(cudaMemcpyAsync(tokens_owned_, tokens, tok_bytes,
                             on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, s_));
    tokens_dev_ = tokens_owned_;
  }
  SPK_CUDA(cudaMemcpyAsync(adam_bc_dev_, adam_bc_host_, 2 * sizeof(float), cudaMemcpyHostToDevice, s_));
  int64_t launches0 = 0;
  for (auto& [v, st] : stages_) {
    st->flops = 0;
    launches0 += st->launches;
  }
  if (use_graph) {
    if (!graph_exec_) {
      SPK_CUDA(cudaStreamBeginCapture(s_, cudaStreamCaptureModeRelaxed));
      try {
        enqueue_ops();
      } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(s_, &g);
        if (g) cudaGraphDestroy(g);
        throw;
      }
      SPK_CUDA(cudaStreamEndCapture(s_, &graph_));
      SPK_CUDA(cudaGraphInstantiate(&graph_exec_, graph_, 0));
      graph_flags_ = mc_.flags;
      graph_launches_ = 0;
      graph_flops_ = 0;
      for (auto& [v, st] : stages_) {
        graph_launches_ += st->launches;
        graph_flops_ += st->flops;
      }
      graph_launches_ -= launches0;
    }
    SPK_CUDA(cudaGraphLaunch(graph_exec_, s_));
  } else {
    enqueue_ops();
  }
  // pinned: a pageable read-back would block this thread until the step ends, before the watchdog
  SPK_CUDA(cudaMemcpyAsync(loss_host_, loss_dev_, sizeof(double), cudaMemcpyDeviceToHost, s_));
  SPK_CUDA(cudaEventRecord(ev_step1_, s_));
  if (world_ > 1 && watchdog_s_ > 0) {  // a transfer that never pairs up must not hang the process
    const auto t0 = std::chrono::steady_clock::now();
    while (true) {
      const cudaError_t q = cudaEventQuery(ev_step1_);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) SPK_CUDA(q);
      if (std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count() > watchdog_s_) {
        transport_->abort();
        poisoned_ = true;
        throw seqpipe::DeadlockError("P2P watchdog: step of rank " + std::to_string(rank_) + " did not complete in " +
                                     std::to_string(watchdog_s_) + " s");
      }
      std::this_thread::sleep_for(std::chrono::microseconds(200));
    }
  }
  SPK_CUDA(cudaEventSynchronize(ev_step1_));

  // Measured timeline (SimReport definitions, sim.cpp:234-274).
  t_start_.assign(replay_.size(), 0);
  t_end_.assign(replay_.size(), 0);
  double busy = 0, first = 1e300, last = 0;
  for (size_t i = 0; i < replay_.size(); ++i) {
    float a = 0, b = 0;
    SPK_CUDA(cudaEventElapsedTime(&a, ev_step0_, ev_start_[i]));
    SPK_CUDA(cudaEventElapsedTime(&b, ev_step0_, ev_end_[i]));
    t_start_[i] = a;
    t_end_[i] = b;
    busy += b - a;
    first = std::min(first, (double)a);
    last = std::max(last, (double)b);
  }
  float total = 0;
  SPK_CUDA(cudaEventElapsedTime(&total, ev_step0_, ev_step1_));
  if (rep) {
    std::memset(rep, 0, sizeof(*rep));
    rep->step_ms = total;
    rep->busy_ms = busy;
    rep->first_start_ms = first;
    rep->last_end_ms = last;
    const double window = last - first;
    rep->bubble_ratio = window > 0 ? std::max(0.0, (window - busy) / window) : 0.0;
    rep->loss = *loss_host_ / (static_cast<double>(cfg_.micro_batches) * cfg_.seq_len);
    double peak = 0, arena = 0, wbytes = 0, flops = 0;
    int64_t launches = 0;
    for (auto& [v, st] : stages_) {
      peak = std::max(peak, st->live_peak_bytes());
      arena = std::max(arena, st->arena_bytes());
      wbytes += st->weight_bytes();
      flops += st->flops;
      launches += st->launches;
    }
    rep->peak_activation_bytes = peak;
    rep->arena_bytes = arena;
    rep->weight_bytes = wbytes;
    rep->ops_executed = static_cast<int64_t>(replay_.size());
    rep->kernel_launches = use_graph ? graph_launches_ : launches - launches0;
    rep->dominant_kernel_flops = use_graph ? graph_flops_ : flops;
    if (probe_.enabled) {
      double ms[KernelProbe::kNumClasses], fl[KernelProbe::kNumClasses];
      int64_t cnt[KernelProbe::kNumClasses];
      probe_.totals(ms, fl, cnt);
      int dom = 0;
      for (int c = 0; c < KernelProbe::kNumClasses; ++c) {
        rep->class_ms[c] = ms[c];
        rep->class_flops[c] = fl[c];
        rep->class_launches[c] = cnt[c];
        if (ms[c] > ms[dom]) dom = c;
      }
      rep->dominant_kernel_class = dom;
      rep->dominant_kernel_ms = ms[dom];
      rep->dominant_kernel_flops = fl[dom];
      rep->dominant_kernel_launches = cnt[dom];
    }
  }
}

std::vector<std::vector<seqpipe::Task>> Engine::op_log_by_device() const {
  std::vector<std::vector<seqpipe::Task>> out(static_cast<size_t>(cfg_.pipeline_size));
  for (const auto& t : op_log_) out[static_cast<size_t>(t.device - 1)].push_back(t);
  return out;
}

Stage* Engine::stage_for_param(const std::string& name, Param* out) {
  for (auto& [v, st] : stages_)
    for (const Param& p : st->params())
      if (p.name == name) {
        *out = p;
        return st.get();
      }
  return nullptr;
}

std::vector<std::pair<Stage*, Param>> Engine::all_params() {
  std::vector<std::pair<Stage*, Param>> out;
  for (auto& [v, st] : stages_)
    for (const Param& p : st->params()) out.emplace_back(st.get(), p);
  return out;
}

seqpipe::SimReport Engine::measured_report() const {
  using seqpipe::Rational;
  using seqpipe::TaskKind;
  seqpipe::SimReport r;
  r.kind = sched_.kind;
  r.config = cfg_;
  r.partition_lengths = len_;
  const int P = cfg_.pipeline_size;
  r.task_times.assign(static_cast<size_t>(P), {});
  auto ns = [](double ms) { return static_cast<std::int64_t>(std::llround(ms * 1e6)); };
  for (size_t i = 0; i < op_log_.size() && i < t_start_.size(); ++i) {
    const seqpipe::Task& t = op_log_[i];
    seqpipe::TaskTiming tt_i;
    tt_i.task = t;
    tt_i.start = Rational(ns(t_start_[i]));
    tt_i.end = Rational(ns(t_end_[i]));
    r.task_times[static_cast<size_t>(t.device - 1)].push_back(tt_i);
  }
  Rational makespan(0), sum_idle(0), sum_window(0), max_peak(0);
  for (const auto& tt : r.task_times)
    for (const auto& x : tt) makespan = std::max(makespan, x.end);
  for (int d = 1; d <= P; ++d) {
    auto& tt = r.task_times[static_cast<size_t>(d - 1)];
    std::sort(tt.begin(), tt.end(), [](const auto& a, const auto& b) { return a.start < b.start; });
    seqpipe::DeviceReport dev;
    dev.device = d;
    if (!tt.empty()) {
      dev.first_start = tt.front().start;
      dev.last_end = tt.front().end;
      for (const auto& x : tt) {
        dev.busy = dev.busy + (x.end - x.start);
        dev.last_end = std::max(dev.last_end, x.end);
      }
      const Rational window = dev.last_end - dev.first_start;
      dev.idle = window > Rational(0) ? window - dev.busy : Rational(0);
      if (dev.idle < Rational(0)) dev.idle = Rational(0);  // overlapping events on one stream
      dev.bubble_ratio = window > Rational(0) ? dev.idle / window : Rational(0);
      dev.idle_in_makespan = makespan > dev.busy ? makespan - dev.busy : Rational(0);
      dev.bubble_ratio_in_makespan = makespan > Rational(0) ? dev.idle_in_makespan / makespan : Rational(0);
      sum_idle = sum_idle + dev.idle;
      sum_window = sum_window + window;
      // warm-up forwards: F tasks before the first backward (sim.cpp:240-250)
      for (const auto& x : tt) {
        if (x.task.kind != TaskKind::kForward) break;
        ++dev.warmup_forward_tasks;
      }
      // memory series: + record (and the KV slab at segment 1) at F end, - at B end
      // (time, bytes delta, record-count delta); the W record I leaves is counted in bytes
      // (it is real arena memory) but not as an allocation (sim.cpp counts (m,s) records).
      struct MemEv {
        Rational t;
        std::int64_t bytes;
        int recs;
      };
      std::vector<MemEv> ev;
      for (const auto& x : tt) {
        auto it = stages_.find(x.task.stage);
        if (it == stages_.end()) continue;
        const Stage& st = *it->second;
        const std::int64_t b = st.record_bytes(x.task.segment) + (x.task.segment == 1 ? st.kv_slab_bytes() : 0);
        const std::int64_t wb = st.w_record_bytes(x.task.segment);
        if (x.task.kind == TaskKind::kForward) ev.push_back({x.end, b, 1});
        else if (x.task.kind == TaskKind::kFusedBackward) ev.push_back({x.end, -b, -1});
        else if (x.task.kind == TaskKind::kInputGrad) ev.push_back({x.end, wb, 0});  // W operands held until W
        else if (x.task.kind == TaskKind::kWeightGrad)
          ev.push_back({x.end, -(b + wb), -1});  // zero-bubble kinds free at W end (sim.cpp:279-293)
      }
      std::stable_sort(ev.begin(), ev.end(), [](const MemEv& a, const MemEv& b) { return a.t < b.t; });
      std::int64_t live = 0, live_recs = 0, peak_recs = 0;
      dev.memory_series.push_back({Rational(0), Rational(0)});
      for (const MemEv& e : ev) {
        live += e.bytes;
        live_recs += e.recs;
        peak_recs = std::max(peak_recs, live_recs);
        dev.memory_series.push_back({e.t, Rational(live)});
        dev.peak_memory = std::max(dev.peak_memory, Rational(live));
      }
      dev.peak_allocations = peak_recs;
    }
    max_peak = std::max(max_peak, dev.peak_memory);
    r.devices.push_back(std::move(dev));
  }
  r.makespan = makespan;
  r.aggregate_bubble_ratio = sum_window > Rational(0) ? sum_idle / sum_window : Rational(0);
  Rational in_mk(0);
  for (const auto& dv : r.devices) in_mk = in_mk + dv.idle_in_makespan;
  r.aggregate_bubble_ratio_in_makespan =
      makespan > Rational(0) ? in_mk / (makespan * Rational(P)) : Rational(0);
  r.max_peak_memory = max_peak;
  r.modeled_throughput = makespan > Rational(0)
                             ? Rational(static_cast<std::int64_t>(cfg_.micro_batches) * cfg_.seq_len) / makespan
                             : Rational(0);
  return r;
}

}  // namespace spe
