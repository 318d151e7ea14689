// Seq1F1B execution engine: one object per device (GPU). It owns every
// pipeline stage mapped to that device (stage -> device round-robin as
// seqpipe::StageMap), executes the device's op order from seqpipe::generate()
// with real sm_100a kernels, and reports SimReport-shaped measurements.
#pragma once

#include <cuda_runtime.h>

#include <map>
#include <memory>
#include <string>
#include <vector>

#include "cuda/common.cuh"
#include "cuda/ops.h"
#include "engine/transport.hpp"
#include "seqpipe/partition.hpp"
#include "seqpipe/scenario.hpp"
#include "seqpipe/schedule.hpp"
#include "seqpipe/sim.hpp"
#include "seqpipe_b200.h"

namespace spe {

using spk::DType;

struct ModelCfg {
  int family = SP_MODEL_GPT;
  DType dt = DType::kBF16;
  int V = 0, Vpad = 0, h = 0, L = 0, H = 0, hd = 0, F = 0, Fup = 0;
  int64_t max_seq = 0;
  uint64_t seed = 0;
  float init_std = 0.02f, eps = 1e-5f, theta = 10000.f;
  float lr = 0.f, b1 = 0.9f, b2 = 0.95f, adam_eps = 1e-8f, wd = 0.f;
  int flags = 0;
  bool rms() const { return family == SP_MODEL_LLAMA; }
};

struct Param {
  std::string name;
  int64_t off = 0, numel = 0;
  int rows = 0, cols = 0;
};

// CUDA-event probes around every GEMM / attention launch (SP_FLAG_KPROBE):
// per-class device time and algorithmic FLOPs for the live roofline.
struct KernelProbe {
  enum Class { kGemm = 0, kAttnFwd = 1, kAttnBwd = 2, kNumClasses = 3 };
  struct Rec {
    int cls;
    cudaEvent_t a, b;
    double flops;
  };
  std::vector<cudaEvent_t> pool;
  std::vector<Rec> recs;
  size_t next = 0;
  bool enabled = false;
  cudaEvent_t get();
  void begin(int cls, cudaStream_t s, double flops);
  void end(cudaStream_t s);
  void reset() {
    recs.clear();
    next = 0;
  }
  // Sums per class after the stream has been synchronised.
  void totals(double (&ms)[kNumClasses], double (&fl)[kNumClasses], int64_t (&n)[kNumClasses]);
  ~KernelProbe();
};

// First-fit arena plan over a fixed alloc/free sequence.
struct ArenaPlan {
  int64_t size = 0;       // high-water mark of the address range
  int64_t live_peak = 0;  // high-water mark of live bytes
  std::map<int64_t, int64_t> free_;  // offset -> bytes
  std::map<int64_t, int64_t> used_;
  int64_t live = 0;
  int64_t alloc(int64_t bytes);
  void release(int64_t off);
};

// Two pools: fixed-size per-micro-batch KV-prefix slabs, and variable-size
// per-(m,s) activation records. Separating them keeps the record pool from
// fragmenting around the large slabs. Offsets of pool 1 are relative to the
// end of pool 0 once finalised.
struct DualArena {
  ArenaPlan pool[2];
  int64_t live = 0, live_peak = 0;
  int64_t alloc(int p, int64_t bytes) {
    const int64_t before = pool[p].live;
    const int64_t off = pool[p].alloc(bytes);
    live += pool[p].live - before;
    live_peak = std::max(live_peak, live);
    return off;
  }
  void release(int p, int64_t off) {
    const int64_t before = pool[p].live;
    pool[p].release(off);
    live += pool[p].live - before;
  }
  int64_t size() const { return pool[0].size + pool[1].size; }
};

DualArena plan_stage_memory(const ModelCfg& mc, const seqpipe::ScenarioConfig& cfg, const std::vector<int64_t>& len,
                            const std::vector<seqpipe::Task>& order, int stage);

class Stage {
 public:
  Stage(const ModelCfg& m, const seqpipe::ScenarioConfig& cfg, const std::vector<int64_t>& lengths, int stage,
        int total_stages, cudaStream_t s);
  ~Stage();

  // Per-(micro-batch, segment) activation record inside the arena.
  struct Seg {
    int64_t n = 0, pos0 = 0;
    std::vector<void*> x_in;  // L_s layer inputs [n,h]
    void* x_out = nullptr;    // stage output [n,h]
    void* dy_in = nullptr;    // gradient w.r.t. the stage output [n,h]
    std::vector<void*> q, o, x_mid, u;
    std::vector<float*> mean1, rstd1, mean2, rstd2, lse;
    // Zero-bubble split (I / W tasks): weight-gradient operands the I task leaves
    // for the W task, per layer: layer-output grad [n,h], activation grad
    // [n,Fup], attention-output grad [n,h], dQKV [n,3h].
    std::vector<void*> w_dy, w_du, w_dxm, w_dqkv;
  };

  void plan_arena(const std::vector<seqpipe::Task>& order);
  void bind_step();  // (re)bind Seg views to the arena for every (m,s) of this stage

  void forward(int m, int s, const int32_t* tokens_dev, double* loss_acc, float loss_scale);
  // dx_target: where the gradient w.r.t. this stage's input goes (another stage's dy_in or a send buffer).
  void backward(int m, int s, void* dx_target, const int32_t* tokens_dev);
  // Zero-bubble split (reference TaskKind I / W, schedule.cpp:217-309): I = the
  // backward without the weight-gradient GEMMs (their operands saved in the W
  // record), W = those GEMMs (norm-output / activation operands recomputed).
  void backward_input(int m, int s, void* dx_target, const int32_t* tokens_dev);
  void backward_weight(int m, int s);

  Seg& seg(int m, int s) { return segs_[(m - 1) * k_ + (s - 1)]; }
  void* kv(int m, int layer) const;  // [T, 2h] slab of layer (local index)
  float* dkv(int layer) const { return dkv_ + static_cast<size_t>(layer) * T_ * 2 * mc_.h; }

  void set_flags(int f) {  // the record layout flag stays what the stage was built with
    mc_.flags = (f & ~SP_FLAG_RECOMPUTE_MLP) | (mc_.flags & SP_FLAG_RECOMPUTE_MLP);
  }
  bool recompute_mlp() const { return (mc_.flags & SP_FLAG_RECOMPUTE_MLP) != 0; }
  void zero_grads();
  void sync_compute();  // recast the compute-dtype weight copy after a master write
  // AdamW over this stage's parameters; bias corrections {1-b1^t, 1-b2^t} read from device memory
  // (written per step outside any captured graph).
  void optimizer_step(const float* bc_dev);
  void init_weights();
  const std::vector<Param>& params() const { return params_; }
  float* master() const { return master_; }
  float* grads() const { return grad_; }
  int64_t param_numel() const { return nparams_; }
  double weight_bytes() const;
  double arena_bytes() const { return static_cast<double>(arena_.size()); }
  double live_peak_bytes() const { return static_cast<double>(arena_.live_peak); }
  // Planned bytes of one (m, s) activation record (segment s, 1-based) and of a
  // micro-batch's KV-prefix slab: the units of the measured memory series.
  int64_t record_bytes(int s) const;
  int64_t kv_slab_bytes() const;
  // Planned bytes of one zero-bubble W record (operands I leaves for W) of segment s.
  int64_t w_record_bytes(int s) const;
  double dkv_bytes() const { return static_cast<double>(L_s_) * T_ * 2 * mc_.h * 4; }
  int stage() const { return stage_; }
  bool first() const { return stage_ == 1; }
  bool last() const { return stage_ == total_stages_; }

  // Count of GEMM FLOPs + attention FLOPs (algorithmic) issued by this stage since the last reset.
  double flops = 0;
  int64_t launches = 0;
  KernelProbe* probe = nullptr;

 private:
  struct LayerW {
    int64_t norm1, wqkv, wo, norm2, w1, w2;
  };
  void* wc(int64_t off) const;  // compute-dtype weight pointer
  float* wm(int64_t off) const { return master_ + off; }
  float* wg(int64_t off) const { return grad_ + off; }
  void gemm(const spk::GemmArgs& a, double flop);
  // Weight-gradient GEMM on the side stream, concurrent with the dgrad GEMM that
  // follows it (the two read the same operands and write disjoint outputs); the
  // persistent kernels then fill each other's last-wave tails. join() makes the
  // compute stream wait before anything overwrites the wgrad operands.
  void wgrad(const spk::GemmArgs& a, double flop);
  void join();
  cudaStream_t s2_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
  bool pending_join_ = false;
  void head_forward_backward(Seg& sg, int m, const int32_t* tokens_dev, double* loss_acc, float loss_scale);
  int64_t add_param(const std::string& name, int rows, int cols);

  ModelCfg mc_;
  seqpipe::ScenarioConfig cfg_;
  std::vector<int64_t> len_, prefix_;
  int stage_, total_stages_, l0_, L_s_, k_, M_;
  int64_t T_, nmax_;
  cudaStream_t s_;
  size_t esz_;

  std::vector<Param> params_;
  std::vector<LayerW> lw_;
  int64_t embed_ = -1, pos_ = -1, fnorm_ = -1, lm_ = -1;
  int64_t nparams_ = 0;
  float *master_ = nullptr, *grad_ = nullptr, *adam_m_ = nullptr, *adam_v_ = nullptr;
  void* compute_ = nullptr;  // == master_ in fp32 mode

  DualArena arena_;
  uint8_t* arena_ptr_ = nullptr;
  std::vector<int64_t> seg_off_, kv_off_, w_off_;
  void backward_impl(int m, int s, void* dx_target, const int32_t* tokens_dev, bool defer_w);
  std::vector<Seg> segs_;
  float* dkv_ = nullptr;

  // workspace
  void *w_a_ = nullptr, *w_big1_ = nullptr, *w_big2_ = nullptr, *w_t1_ = nullptr, *w_t2_ = nullptr, *w_t3_ = nullptr,
       *w_dqkv_ = nullptr, *w_logits_ = nullptr, *w_u_ = nullptr;  // w_u_: recomputed u (SP_FLAG_RECOMPUTE_MLP)
  float *w_delta_ = nullptr, *w_dq_ = nullptr, *w_fmean_ = nullptr, *w_frstd_ = nullptr;
  int64_t logits_rows_ = 0;
};

class Engine {
 public:
  Engine(const seqpipe::ScenarioConfig& cfg, seqpipe::ScheduleKind kind, const std::vector<int64_t>& lengths,
         const ModelCfg& m, int rank, int world, int cuda_device);
  ~Engine();
  // Multi-rank data plane: NCCL communicators from `ids` (one per channel), or an in-process hub.
  void comm_init(const std::vector<std::string>& ids);
  void attach_local(std::shared_ptr<LocalHub> hub);
  // Peer-memory (CUDA IPC) data plane: export this rank's rings / flags, then connect with
  // every rank's blob (rank order).
  std::string ipc_export();
  void ipc_connect(const std::vector<std::string>& blobs);
  int comm_channels() const;
  void step(const int32_t* tokens, bool on_device, sp_step_report* rep);
  // Capture the step (ops + optimizer) once into a CUDA graph and replay it (single-rank engines).
  void enable_graph(bool on);
  bool graph_active() const { return graph_exec_ != nullptr; }
  const std::vector<seqpipe::Task>& op_log() const { return op_log_; }
  std::vector<std::vector<seqpipe::Task>> op_log_by_device() const;
  const std::vector<double>& t_start() const { return t_start_; }
  const std::vector<double>& t_end() const { return t_end_; }
  // The last step as a SimReport (sim.hpp) with MEASURED values: integer
  // nanoseconds from the step start, per-device busy / idle / bubble ratios with
  // the definitions of sim.cpp:234-274, memory in bytes (activation records +
  // KV-prefix slabs: +at F end, -at B end, sim.cpp:276-311).
  seqpipe::SimReport measured_report() const;
  Stage* stage_for_param(const std::string& name, Param* out);
  std::vector<std::pair<Stage*, Param>> all_params();
  int device() const { return dev_; }
  bool table_from_device() const { return table_from_device_; }
  void set_flags(int f) {
    mc_.flags = (f & ~SP_FLAG_RECOMPUTE_MLP) | (mc_.flags & SP_FLAG_RECOMPUTE_MLP);
    for (auto& kv : stages_) kv.second->set_flags(f);
  }

 private:
  bool local_transport_ = false;  // attached to the in-process hub: shares its GPU with other engines' threads
  IpcExporter* ipc_ = nullptr;    // transport_ when it is the IPC transport (between export and connect)
  std::string ipc_blob_;
  void enqueue_ops();  // every op of this process's order (+ transfers), on the engine streams
  void exec_op(const seqpipe::Task& t, int order_index, int device_pos);
  // Receive side of one channel: R staging slots so receives are posted ahead of the op that
  // consumes them (the op copies the message out of its slot on the compute stream).
  struct RecvChannel {
    int peer = -1;
    cudaStream_t s = nullptr;
    std::vector<void*> slot;
    std::vector<cudaEvent_t> done, freed;  // recv completed / slot consumed
    std::vector<const sp_comm_op*> msgs;   // this step's messages in order
    size_t posted = 0, consumed = 0;
  };
  static constexpr int kRecvSlots = 2;
  void post_recvs(RecvChannel& rc, int ch, bool block_for_next);
  std::map<int, RecvChannel> recv_ch_;
  std::map<int, cudaStream_t> send_s_;  // per send channel
  std::vector<std::vector<sp_comm_op>> plan_pre_, plan_post_;  // per device-order position
  std::vector<sp_comm_op> plan_;
  Stage* stage_obj(int stage) { return stages_.at(stage).get(); }
  void comm_ready_setup();
  void drop_graph();

  seqpipe::ScenarioConfig cfg_;
  seqpipe::ScheduleKind kind_;
  std::vector<int64_t> len_;
  ModelCfg mc_;
  int rank_, world_, dev_;
  seqpipe::Schedule sched_;
  bool table_from_device_ = false;
  std::vector<std::pair<int, int>> replay_;  // (device, position) execution order for this process
  std::map<int, std::unique_ptr<Stage>> stages_;
  cudaStream_t s_ = nullptr;
  int32_t* tokens_dev_ = nullptr;
  int32_t* tokens_owned_ = nullptr;
  double* loss_dev_ = nullptr;
  float* adam_bc_dev_ = nullptr;   // {1 - b1^t, 1 - b2^t} of the current step (device)
  float* adam_bc_host_ = nullptr;  // pinned staging for it
  double* loss_host_ = nullptr;    // pinned loss read-back
  int step_no_ = 0;
  std::vector<seqpipe::Task> op_log_;
  std::vector<cudaEvent_t> ev_start_, ev_end_;
  cudaEvent_t ev_step0_ = nullptr, ev_step1_ = nullptr;
  std::vector<double> t_start_, t_end_;
  std::unique_ptr<Transport> transport_;
  // Set when the P2P watchdog fired and the transport could not release every parked stream
  // wait: device work may never retire, so teardown must neither synchronize nor free memory
  // that work can still touch (cudaFree synchronizes the device).
  bool poisoned_ = false;
  std::vector<void*> send_ring_;
  std::vector<cudaEvent_t> send_ring_ev_;
  int send_ring_next_ = 0;
  std::vector<cudaEvent_t> act_sent_;  // per (m,s) of a sending stage: activation send retired
  cudaEvent_t ev_tmp_ = nullptr;
  double watchdog_s_ = 600.0;
  KernelProbe probe_;
  // CUDA graph of the step body (world == 1)
  bool graph_wanted_ = false;
  int graph_flags_ = 0;
  cudaGraph_t graph_ = nullptr;
  cudaGraphExec_t graph_exec_ = nullptr;
  int64_t graph_launches_ = 0;  // kernels in the captured step body
  double graph_flops_ = 0;
};

}  // namespace spe
