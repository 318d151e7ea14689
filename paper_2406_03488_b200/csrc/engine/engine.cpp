// Engine: executes the op table of one device (or of every device, when a
// single process drives all stages on one GPU) and measures it.
//
// Multi-process (world == pipeline_size): rank r drives device r+1. The only
// exchange steps are the pipeline edges of the dependency model
// (/root/reference/proj/core/src/sim.cpp:20-23, :31-33): after F(m,s,v) the
// stage output goes to v+1, after B(m,s,v) the input gradient goes to v-1.
// They run as ncclSend/ncclRecv on four communicators (activation / gradient x
// even / odd edge) each bound to its own stream, so no communicator is ever
// used from two streams and the compute stream only waits on receives. Both
// sides of every edge issue the transfers in their own device order, which
// agree (forwards m-up s-up, backwards m-up s-down), so the FIFOs match.
#include "engine/engine.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>

#include "engine/comm_plan.hpp"
#include "seqpipe/sim.hpp"
#include "seqpipe/validate.hpp"

namespace spe {

#define SPE_NCCL(call)                                                                               \
  do {                                                                                               \
    ncclResult_t _r = (call);                                                                        \
    if (_r != ncclSuccess) throw std::runtime_error(std::string("NCCL: ") + ncclGetErrorString(_r)); \
  } while (0)

Engine::Engine(const seqpipe::ScenarioConfig& cfg, seqpipe::ScheduleKind kind, const std::vector<int64_t>& lengths,
               const ModelCfg& m, int rank, int world, int cuda_device)
    : cfg_(cfg), kind_(kind), len_(lengths), mc_(m), rank_(rank), world_(world), dev_(cuda_device) {
  cfg_.validate();
  if (world != 1 && world != cfg.pipeline_size)
    throw std::invalid_argument("world_size must be 1 (all stages in-process) or pipeline_size");
  if (world > 1 && cfg.stages_per_device > 1 && cfg.pipeline_size % 2)
    throw std::invalid_argument("multi-process interleaved schedules need an even pipeline_size");
  if (rank < 0 || rank >= world) throw std::invalid_argument("rank out of range");
  if (mc_.h != mc_.H * mc_.hd) throw std::invalid_argument("hidden must equal heads * head_dim");
  if (mc_.family == SP_MODEL_GPT && mc_.max_seq < cfg.seq_len) throw std::invalid_argument("max_seq < seq_len");
  SPK_CUDA(cudaSetDevice(dev_));
  sched_ = seqpipe::generate(cfg_, kind_, seqpipe::make_partition(len_, cfg_));
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
    const auto& order = sched_.device_orders[static_cast<size_t>(rank_)];
    for (size_t j = 0; j < order.size(); ++j) replay_.emplace_back(rank_, static_cast<int>(j));
    plan_pre_.assign(order.size(), {});
    plan_post_.assign(order.size(), {});
    for (const sp_comm_op& c : comm_plan(sched_, len_, rank_ + 1, mc_.h))
      (c.when == 0 ? plan_pre_ : plan_post_)[static_cast<size_t>(c.op_index)].push_back(c);
  }
  // In-process stage hand-off: stage v's layer-0 input aliases stage v-1's output.
  for (auto& [v, st] : stages_) {
    if (v == 1 || !stages_.count(v - 1)) continue;
    for (int mb = 1; mb <= cfg_.micro_batches; ++mb)
      for (int s = 1; s <= cfg_.segments; ++s) st->seg(mb, s).x_in[0] = stages_[v - 1]->seg(mb, s).x_out;
  }
  const size_t tok_bytes = sizeof(int32_t) * cfg_.micro_batches * (cfg_.seq_len + 1);
  SPK_CUDA(cudaMalloc(&tokens_owned_, tok_bytes));
  SPK_CUDA(cudaMalloc(&loss_dev_, sizeof(double)));
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
  if (s_) cudaStreamSynchronize(s_);
  for (auto& c : comms_)
    if (c) ncclCommDestroy(c);
  stages_.clear();
  for (auto e : ev_start_) cudaEventDestroy(e);
  for (auto e : ev_end_) cudaEventDestroy(e);
  for (auto e : send_ring_ev_) cudaEventDestroy(e);
  for (auto p : send_ring_) cudaFree(p);
  if (ev_step0_) cudaEventDestroy(ev_step0_);
  if (ev_step1_) cudaEventDestroy(ev_step1_);
  if (ev_tmp_) cudaEventDestroy(ev_tmp_);
  if (tokens_owned_) cudaFree(tokens_owned_);
  if (loss_dev_) cudaFree(loss_dev_);
  if (s_send_) cudaStreamDestroy(s_send_);
  if (s_recv_) cudaStreamDestroy(s_recv_);
  if (s_) cudaStreamDestroy(s_);
}

void Engine::comm_init(const std::vector<std::string>& ids) {
  if (world_ == 1) return;
  if (ids.size() != 4) throw std::invalid_argument("comm_init expects 4 NCCL unique ids");
  SPK_CUDA(cudaSetDevice(dev_));
  SPE_NCCL(ncclGroupStart());
  for (int i = 0; i < 4; ++i) {
    ncclUniqueId id;
    std::memcpy(&id, ids[static_cast<size_t>(i)].data(), sizeof(id));
    SPE_NCCL(ncclCommInitRank(&comms_[i], world_, id, rank_));
  }
  SPE_NCCL(ncclGroupEnd());
  SPK_CUDA(cudaStreamCreateWithFlags(&s_send_, cudaStreamNonBlocking));
  SPK_CUDA(cudaStreamCreateWithFlags(&s_recv_, cudaStreamNonBlocking));
  // Gradient send ring: a slot is reused only after its previous send completed.
  int64_t nmax = *std::max_element(len_.begin(), len_.end());
  for (int i = 0; i < 4; ++i) {
    void* p = nullptr;
    SPK_CUDA(cudaMalloc(&p, spk::dtype_size(mc_.dt) * nmax * mc_.h));
    send_ring_.push_back(p);
    cudaEvent_t e;
    SPK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    SPK_CUDA(cudaEventRecord(e, s_));
    send_ring_ev_.push_back(e);
  }
  comm_ready_ = true;
}

static ncclDataType_t nccl_type(DType t) { return t == DType::kF32 ? ncclFloat32 : ncclBfloat16; }

// Executes op `t` (position `pos` of its device order, `i`-th op of this step).
// Multi-process: the transfers are exactly sp_comm_plan's entries for this op —
// receives on s_recv_ before the op (the compute stream waits on them), sends
// on s_send_ after it (the compute stream never waits on a send).
void Engine::exec_op(const seqpipe::Task& t, int i, int pos) {
  Stage* st = stage_obj(t.stage);
  Stage::Seg& sg = st->seg(t.micro_batch, t.segment);
  const bool fwd = t.kind == seqpipe::TaskKind::kForward;
  if (t.kind == seqpipe::TaskKind::kWeightGrad) {  // zero-bubble W: local weight-gradient GEMMs, no transfers
    SPK_CUDA(cudaEventRecord(ev_start_[i], s_));
    st->backward_weight(t.micro_batch, t.segment);
    SPK_CUDA(cudaEventRecord(ev_end_[i], s_));
    return;
  }
  const bool input_only = t.kind == seqpipe::TaskKind::kInputGrad;  // zero-bubble I: B without the W GEMMs
  const std::vector<sp_comm_op>* pre = nullptr;
  const std::vector<sp_comm_op>* post = nullptr;
  if (world_ > 1) {
    pre = &plan_pre_[static_cast<size_t>(pos)];
    post = &plan_post_[static_cast<size_t>(pos)];
  }
  if (pre) {
    for (const sp_comm_op& c : *pre) {  // receive into this op's input buffer
      SPK_CUDA(cudaEventRecord(ev_tmp_, s_));  // buffer region free once earlier ops retired
      SPK_CUDA(cudaStreamWaitEvent(s_recv_, ev_tmp_));
      SPE_NCCL(ncclRecv(fwd ? sg.x_in[0] : sg.dy_in, static_cast<size_t>(c.elems), nccl_type(mc_.dt), c.peer,
                        comms_[c.channel], s_recv_));
      SPK_CUDA(cudaEventRecord(ev_tmp_, s_recv_));
      SPK_CUDA(cudaStreamWaitEvent(s_, ev_tmp_));
    }
  }
  if (fwd) {
    SPK_CUDA(cudaEventRecord(ev_start_[i], s_));
    st->forward(t.micro_batch, t.segment, tokens_dev_, loss_dev_, 1.0f / (float)(cfg_.micro_batches * cfg_.seq_len));
    SPK_CUDA(cudaEventRecord(ev_end_[i], s_));
    if (post)
      for (const sp_comm_op& c : *post) {
        SPK_CUDA(cudaStreamWaitEvent(s_send_, ev_end_[i]));
        SPE_NCCL(ncclSend(sg.x_out, static_cast<size_t>(c.elems), nccl_type(mc_.dt), c.peer, comms_[c.channel],
                          s_send_));
      }
    return;
  }
  void* dx_target = nullptr;
  int slot = -1;
  if (post && !post->empty()) {
    slot = send_ring_next_;
    send_ring_next_ = (send_ring_next_ + 1) % static_cast<int>(send_ring_.size());
    SPK_CUDA(cudaStreamWaitEvent(s_, send_ring_ev_[static_cast<size_t>(slot)]));
    dx_target = send_ring_[static_cast<size_t>(slot)];
  } else if (t.stage > 1) {
    dx_target = stage_obj(t.stage - 1)->seg(t.micro_batch, t.segment).dy_in;  // in-process hand-off
  }
  SPK_CUDA(cudaEventRecord(ev_start_[i], s_));
  if (input_only)
    st->backward_input(t.micro_batch, t.segment, dx_target, tokens_dev_);
  else
    st->backward(t.micro_batch, t.segment, dx_target, tokens_dev_);
  SPK_CUDA(cudaEventRecord(ev_end_[i], s_));
  if (slot >= 0) {
    for (const sp_comm_op& c : *post) {
      SPK_CUDA(cudaStreamWaitEvent(s_send_, ev_end_[i]));
      SPE_NCCL(ncclSend(dx_target, static_cast<size_t>(c.elems), nccl_type(mc_.dt), c.peer, comms_[c.channel], s_send_));
    }
    SPK_CUDA(cudaEventRecord(send_ring_ev_[static_cast<size_t>(slot)], s_send_));
  }
}

void Engine::step(const int32_t* tokens, bool on_device, sp_step_report* rep) {
  SPK_CUDA(cudaSetDevice(dev_));
  if (world_ > 1 && !comm_ready_) throw std::logic_error("multi-process engine: call sp_engine_comm_init first");
  ++step_no_;
  SPK_CUDA(cudaEventRecord(ev_step0_, s_));
  const size_t tok_bytes = sizeof(int32_t) * cfg_.micro_batches * (cfg_.seq_len + 1);
  if (on_device) {
    tokens_dev_ = const_cast<int32_t*>(tokens);
  } else {
    SPK_CUDA(cudaMemcpyAsync(tokens_owned_, tokens, tok_bytes, cudaMemcpyHostToDevice, s_));
    tokens_dev_ = tokens_owned_;
  }
  SPK_CUDA(cudaMemsetAsync(loss_dev_, 0, sizeof(double), s_));
  probe_.enabled = (mc_.flags & SP_FLAG_KPROBE) != 0;
  probe_.reset();
  int64_t launches0 = 0;
  for (auto& [v, st] : stages_) {
    st->zero_grads();
    st->flops = 0;
    launches0 += st->launches;
  }
  op_log_.clear();
  for (size_t i = 0; i < replay_.size(); ++i) {
    const auto [d, j] = replay_[i];
    const seqpipe::Task& t = sched_.device_orders[static_cast<size_t>(d)][static_cast<size_t>(j)];
    exec_op(t, static_cast<int>(i), j);
    op_log_.push_back(t);
  }
  if (s_send_) {  // the step ends when this device's sends have drained
    SPK_CUDA(cudaEventRecord(ev_tmp_, s_send_));
    SPK_CUDA(cudaStreamWaitEvent(s_, ev_tmp_));
  }
  for (auto& [v, st] : stages_) st->optimizer_step(step_no_);
  double loss_h = 0;
  SPK_CUDA(cudaMemcpyAsync(&loss_h, loss_dev_, sizeof(double), cudaMemcpyDeviceToHost, s_));
  SPK_CUDA(cudaEventRecord(ev_step1_, s_));
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
    rep->loss = loss_h / (static_cast<double>(cfg_.micro_batches) * cfg_.seq_len);
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
    rep->kernel_launches = launches - launches0;
    rep->dominant_kernel_flops = flops;
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
      std::vector<std::pair<Rational, std::int64_t>> ev;
      for (const auto& x : tt) {
        auto it = stages_.find(x.task.stage);
        if (it == stages_.end()) continue;
        const Stage& st = *it->second;
        const std::int64_t b = st.record_bytes(x.task.segment) + (x.task.segment == 1 ? st.kv_slab_bytes() : 0);
        if (x.task.kind == TaskKind::kForward) ev.push_back({x.end, b});
        else if (x.task.kind == TaskKind::kFusedBackward || x.task.kind == TaskKind::kWeightGrad)
          ev.push_back({x.end, -b});  // zero-bubble kinds free at W end (sim.cpp:279-293)
      }
      std::stable_sort(ev.begin(), ev.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      std::int64_t live = 0, live_recs = 0, peak_recs = 0;
      dev.memory_series.push_back({Rational(0), Rational(0)});
      for (const auto& [t, b] : ev) {
        live += b;
        live_recs += b > 0 ? 1 : -1;
        peak_recs = std::max(peak_recs, live_recs);
        dev.memory_series.push_back({t, Rational(live)});
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
