// One pipeline stage: weights, activation arena, and the forward / backward op
// bodies of a sub-sequence (Seq1F1B unit) over this stage's layers.
//
// Data flow per (micro-batch m, segment s) — the reference dependency rules
// (/root/reference/proj/core/src/sim.cpp:14-44) made concrete:
//   F(m,s): K/V of this segment are written into the micro-batch's KV slab at
//           rows [prefix_{s-1}, prefix_s); attention reads rows [0, prefix_s)
//           (the causal edge F(m,s-1) -> F(m,s)).
//   B(m,s): attention backward adds dK/dV for rows [0, prefix_s) into the
//           stage's fp32 dKV accumulator; rows of segment s are then complete
//           (reverse edge B(m,s+1) -> B(m,s)), feed the QKV weight/input grads.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "engine/engine.hpp"

namespace spe {

using spk::Epi;
using spk::GemmArgs;

// ------------------------------------------------------------------ arena

int64_t ArenaPlan::alloc(int64_t bytes) {
  bytes = (bytes + 255) / 256 * 256;
  if (bytes == 0) bytes = 256;
  int64_t off = -1;
  for (auto it = free_.begin(); it != free_.end(); ++it) {
    if (it->second >= bytes) {
      off = it->first;
      const int64_t rest = it->second - bytes;
      free_.erase(it);
      if (rest) free_[off + bytes] = rest;
      break;
    }
  }
  if (off < 0) {
    // extend the top; merge with a free block that ends at the top
    off = size;
    if (!free_.empty()) {
      auto last = std::prev(free_.end());
      if (last->first + last->second == size) {
        off = last->first;
        free_.erase(last);
      }
    }
    size = off + bytes;
  }
  used_[off] = bytes;
  live += bytes;
  live_peak = std::max(live_peak, live);
  return off;
}

void ArenaPlan::release(int64_t off) {
  auto it = used_.find(off);
  if (it == used_.end()) throw std::logic_error("arena: double free");
  int64_t bytes = it->second;
  used_.erase(it);
  live -= bytes;
  auto nx = free_.lower_bound(off);
  if (nx != free_.end() && off + bytes == nx->first) {
    bytes += nx->second;
    free_.erase(nx);
  }
  auto pv = free_.lower_bound(off);
  if (pv != free_.begin()) {
    --pv;
    if (pv->first + pv->second == off) {
      off = pv->first;
      bytes += pv->second;
      free_.erase(pv);
    }
  }
  free_[off] = bytes;
}

// ------------------------------------------------------------------ stage

namespace {
uint64_t fnv1a(const std::string& s, uint64_t seed) {
  uint64_t h = 1469598103934665603ULL ^ seed;
  for (unsigned char c : s) {
    h ^= c;
    h *= 1099511628211ULL;
  }
  return h;
}
int64_t align64(int64_t x) { return (x + 63) / 64 * 64; }
}  // namespace

int64_t Stage::add_param(const std::string& name, int rows, int cols) {
  Param p;
  p.name = name;
  p.off = nparams_;
  p.rows = rows;
  p.cols = cols;
  p.numel = static_cast<int64_t>(rows) * cols;
  nparams_ += align64(p.numel);
  params_.push_back(p);
  return p.off;
}

Stage::Stage(const ModelCfg& m, const seqpipe::ScenarioConfig& cfg, const std::vector<int64_t>& lengths, int stage,
             int total_stages, cudaStream_t s)
    : mc_(m), cfg_(cfg), len_(lengths), stage_(stage), total_stages_(total_stages), s_(s) {
  if (mc_.L % total_stages) throw std::invalid_argument("model layers must divide evenly over the pipeline stages");
  L_s_ = mc_.L / total_stages;
  l0_ = (stage - 1) * L_s_;
  k_ = cfg.segments;
  M_ = cfg.micro_batches;
  T_ = cfg.seq_len;
  prefix_.assign(len_.size() + 1, 0);
  for (size_t i = 0; i < len_.size(); ++i) prefix_[i + 1] = prefix_[i] + len_[i];
  nmax_ = *std::max_element(len_.begin(), len_.end());
  esz_ = spk::dtype_size(mc_.dt);

  const int h = mc_.h;
  if (first()) {
    embed_ = add_param("embed", mc_.V, h);
    if (mc_.family == SP_MODEL_GPT) pos_ = add_param("pos", static_cast<int>(mc_.max_seq), h);
  }
  for (int l = 0; l < L_s_; ++l) {
    const std::string p = "layer" + std::to_string(l0_ + l) + ".";
    LayerW w;
    w.norm1 = add_param(p + "norm1", 1, h);
    w.wqkv = add_param(p + "wqkv", 3 * h, h);
    w.wo = add_param(p + "wo", h, h);
    w.norm2 = add_param(p + "norm2", 1, h);
    w.w1 = add_param(p + "w1", mc_.Fup, h);
    w.w2 = add_param(p + "w2", h, mc_.F);
    lw_.push_back(w);
  }
  if (last()) {
    fnorm_ = add_param("final_norm", 1, h);
    lm_ = add_param("lm_head", mc_.Vpad, h);
  }
  const size_t pbytes = sizeof(float) * nparams_;
  SPK_CUDA(cudaMalloc(&master_, pbytes));
  SPK_CUDA(cudaMalloc(&grad_, pbytes));
  SPK_CUDA(cudaMalloc(&adam_m_, pbytes));
  SPK_CUDA(cudaMalloc(&adam_v_, pbytes));
  SPK_CUDA(cudaMemsetAsync(adam_m_, 0, pbytes, s_));
  SPK_CUDA(cudaMemsetAsync(adam_v_, 0, pbytes, s_));
  if (mc_.dt == DType::kF32) {
    compute_ = master_;
  } else {
    SPK_CUDA(cudaMalloc(&compute_, esz_ * nparams_));
  }
  init_weights();

  // workspace
  const int64_t n = nmax_;
  SPK_CUDA(cudaMalloc(&w_a_, esz_ * n * h));
  SPK_CUDA(cudaMalloc(&w_big1_, esz_ * n * mc_.Fup));
  SPK_CUDA(cudaMalloc(&w_big2_, esz_ * n * mc_.Fup));
  if (recompute_mlp()) SPK_CUDA(cudaMalloc(&w_u_, esz_ * n * mc_.Fup));
  SPK_CUDA(cudaMalloc(&w_t1_, esz_ * n * h));
  SPK_CUDA(cudaMalloc(&w_t2_, esz_ * n * h));
  SPK_CUDA(cudaMalloc(&w_t3_, esz_ * n * h));
  SPK_CUDA(cudaMalloc(&w_dqkv_, esz_ * n * 3 * h));
  SPK_CUDA(cudaMalloc(&w_delta_, sizeof(float) * spk::attn_bwd_ws_delta_floats(n, mc_.H)));
  SPK_CUDA(cudaMalloc(&w_dq_, sizeof(float) * n * h));
  if (last()) {
    SPK_CUDA(cudaMalloc(&w_fmean_, sizeof(float) * n));
    SPK_CUDA(cudaMalloc(&w_frstd_, sizeof(float) * n));
    // logits chunk: bounded to ~512 MB
    logits_rows_ = std::max<int64_t>(128, std::min<int64_t>(n, (512LL << 20) / (esz_ * mc_.Vpad)));
    logits_rows_ = std::min<int64_t>(n, (logits_rows_ + 127) / 128 * 128);
    SPK_CUDA(cudaMalloc(&w_logits_, esz_ * logits_rows_ * mc_.Vpad));
  }
  SPK_CUDA(cudaMalloc(&dkv_, sizeof(float) * L_s_ * T_ * 2 * h));
  segs_.resize(static_cast<size_t>(M_) * k_);
  seg_off_.assign(segs_.size(), -1);
  kv_off_.assign(static_cast<size_t>(M_), -1);
}

Stage::~Stage() {
  if (s2_) cudaStreamDestroy(s2_);
  if (ev_fork_) cudaEventDestroy(ev_fork_);
  if (ev_join_) cudaEventDestroy(ev_join_);
  for (void* p : {(void*)master_, (void*)grad_, (void*)adam_m_, (void*)adam_v_, w_a_, w_big1_, w_big2_, w_u_, w_t1_, w_t2_,
                  w_t3_, w_dqkv_, (void*)w_delta_, (void*)w_dq_, (void*)w_fmean_, (void*)w_frstd_, w_logits_,
                  (void*)dkv_, (void*)arena_ptr_})
    if (p) cudaFree(p);
  if (compute_ && compute_ != master_) cudaFree(compute_);
}

double Stage::weight_bytes() const {
  return static_cast<double>(nparams_) * (4.0 * 4 + (mc_.dt == DType::kF32 ? 0 : esz_));
}

void* Stage::wc(int64_t off) const { return static_cast<uint8_t*>(compute_) + off * esz_; }

void Stage::init_weights() {
  const float out_std = mc_.init_std / std::sqrt(2.0f * mc_.L);
  for (const Param& p : params_) {
    const bool gain = p.name.find("norm") != std::string::npos;
    const bool outp = p.name.size() > 3 && (p.name.compare(p.name.size() - 3, 3, ".wo") == 0 ||
                                            p.name.compare(p.name.size() - 3, 3, ".w2") == 0);
    if (gain) {
      spk::fill_const(master_ + p.off, p.numel, 1.f, s_);
    } else if (p.name == "lm_head") {
      spk::fill_normal(master_ + p.off, static_cast<int64_t>(mc_.V) * mc_.h, fnv1a(p.name, mc_.seed), mc_.init_std, s_);
      SPK_CUDA(cudaMemsetAsync(master_ + p.off + static_cast<int64_t>(mc_.V) * mc_.h, 0,
                               sizeof(float) * (p.numel - static_cast<int64_t>(mc_.V) * mc_.h), s_));
    } else {
      spk::fill_normal(master_ + p.off, p.numel, fnv1a(p.name, mc_.seed), outp ? out_std : mc_.init_std, s_);
    }
  }
  if (compute_ != master_) spk::cast_from_f32(mc_.dt, master_, compute_, nparams_, s_);
}

void Stage::sync_compute() {
  if (compute_ != master_) spk::cast_from_f32(mc_.dt, master_, compute_, nparams_, s_);
  SPK_CUDA(cudaStreamSynchronize(s_));
}

void Stage::zero_grads() { SPK_CUDA(cudaMemsetAsync(grad_, 0, sizeof(float) * nparams_, s_)); }

void Stage::optimizer_step(const float* bc_dev) {
  if (mc_.lr <= 0.f) return;
  spk::adamw(master_, grad_, adam_m_, adam_v_, compute_ == master_ ? nullptr : compute_, mc_.dt, nparams_, mc_.lr,
             mc_.b1, mc_.b2, mc_.adam_eps, mc_.wd, bc_dev, s_);
  ++launches;
}

// Activation bytes of one (m, s) record with n tokens.
static int64_t seg_bytes(const ModelCfg& mc, int L_s, int64_t n, size_t esz) {
  const int64_t h = mc.h;
  int64_t b = 0;
  b += (L_s + 2) * n * h * esz;            // x_in[L_s], x_out, dy_in
  b += 3LL * L_s * n * h * esz;            // q, o, x_mid
  if (!(mc.flags & SP_FLAG_RECOMPUTE_MLP)) b += static_cast<int64_t>(L_s) * n * mc.Fup * esz;  // u
  b += static_cast<int64_t>(L_s) * n * (4 + mc.H) * 4;  // norm stats + lse
  return b + 256LL * (8 * L_s + 4);        // per-field alignment slack
}

// Bytes of one (m, s) zero-bubble W record (operands of the deferred
// weight-gradient GEMMs): per layer dy [n,h], du [n,Fup], dxm [n,h], dqkv [n,3h].
static int64_t w_bytes(const ModelCfg& mc, int L_s, int64_t n, size_t esz) {
  return static_cast<int64_t>(L_s) * n * (5LL * mc.h + mc.Fup) * static_cast<int64_t>(esz) + 256LL * 4 * L_s;
}

// Offline placement of buffers whose lifetimes (op indices [a, f], inclusive) are all
// known up front -- the stage's whole op order is fixed before the step runs. Greedy by
// size: largest buffer first, each at the best-fitting gap among the already placed
// buffers that overlap it in time (else on top). Near the live high-water on the
// Seq1F1B orders, where the online first-fit over records of 16 different segment
// lengths left ~15 % of the pool as holes (cfg-4 stage 1: 156.5 -> 133 GB).
struct PlacedBuf {
  int64_t bytes, a, f, off;
};
static int64_t place_offline(std::vector<PlacedBuf>& b) {
  std::vector<size_t> ord(b.size());
  for (size_t i = 0; i < ord.size(); ++i) ord[i] = i;
  std::stable_sort(ord.begin(), ord.end(), [&](size_t x, size_t y) { return b[x].bytes > b[y].bytes; });
  std::vector<size_t> placed;
  int64_t extent = 0;
  std::vector<std::pair<int64_t, int64_t>> busy;
  for (size_t i : ord) {
    busy.clear();
    for (size_t j : placed)
      if (b[j].a <= b[i].f && b[i].a <= b[j].f) busy.emplace_back(b[j].off, b[j].off + b[j].bytes);
    std::sort(busy.begin(), busy.end());
    int64_t cur = 0, best = -1, best_gap = INT64_MAX;
    for (const auto& [o, e] : busy) {
      if (o - cur >= b[i].bytes && o - cur < best_gap) {
        best = cur;
        best_gap = o - cur;
      }
      cur = std::max(cur, e);
    }
    b[i].off = best >= 0 ? best : cur;
    extent = std::max(extent, b[i].off + b[i].bytes);
    placed.push_back(i);
  }
  // invariant: buffers live at the same time never share bytes
  for (size_t i = 0; i < b.size(); ++i)
    for (size_t j = i + 1; j < b.size(); ++j)
      if (b[i].a <= b[j].f && b[j].a <= b[i].f && b[i].off < b[j].off + b[j].bytes && b[j].off < b[i].off + b[i].bytes)
        throw std::logic_error("arena: offline placement overlaps two live buffers");
  return extent;
}

// Host-only replay of the arena plan of one stage (no device memory): the
// analytical activation footprint used to report OOM configurations. F
// allocates the (m,s) record (and at s = 1 the micro-batch's KV slab); B frees
// them; with the zero-bubble split I allocates the W record and W frees all
// three, as the reference frees memory at W end (sim.cpp:279-293). The online
// replay gives the live high-water; offsets come from the offline placement when
// it is tighter than the replay's first-fit (it always is on the measured orders).
static DualArena replay_plan(const ModelCfg& mc, const seqpipe::ScenarioConfig& cfg, const std::vector<int64_t>& len,
                             const std::vector<seqpipe::Task>& order, int stage, std::vector<int64_t>& seg,
                             std::vector<int64_t>& kvo, std::vector<int64_t>& wo) {
  const int L_s = mc.L / cfg.total_stages();
  const size_t esz = spk::dtype_size(mc.dt);
  const int64_t kv_bytes = static_cast<int64_t>(L_s) * cfg.seq_len * 2 * mc.h * esz;
  DualArena a;
  seg.assign(static_cast<size_t>(cfg.micro_batches) * cfg.segments, -1);
  wo.assign(static_cast<size_t>(cfg.micro_batches) * cfg.segments, -1);
  kvo.assign(static_cast<size_t>(cfg.micro_batches), -1);
  // offline view: one buffer per allocation, tagged with the vector slot it fills
  struct Tag {
    int pool;
    std::vector<int64_t>* vec;
    size_t idx;
  };
  std::vector<PlacedBuf> bufs;
  std::vector<Tag> tags;
  std::map<std::pair<std::vector<int64_t>*, size_t>, size_t> open;
  auto on_alloc = [&](int pool, std::vector<int64_t>& v, size_t idx, int64_t bytes, int64_t t) {
    v[idx] = a.alloc(pool, bytes);
    open[{&v, idx}] = bufs.size();
    bufs.push_back({(std::max<int64_t>(bytes, 1) + 255) / 256 * 256, t, INT64_MAX, 0});
    tags.push_back({pool, &v, idx});
  };
  auto on_free = [&](int pool, std::vector<int64_t>& v, size_t idx, int64_t t) {
    a.release(pool, v[idx]);
    auto it = open.find({&v, idx});
    bufs[it->second].f = t;
    open.erase(it);
  };
  int64_t t = 0;
  for (const seqpipe::Task& tk : order) {
    if (tk.stage != stage) continue;
    ++t;
    const size_t idx = static_cast<size_t>(tk.micro_batch - 1) * cfg.segments + (tk.segment - 1);
    const size_t mb = static_cast<size_t>(tk.micro_batch - 1);
    switch (tk.kind) {
      case seqpipe::TaskKind::kForward:
        if (tk.segment == 1) on_alloc(0, kvo, mb, kv_bytes, t);
        on_alloc(1, seg, idx, seg_bytes(mc, L_s, len[tk.segment - 1], esz), t);
        break;
      case seqpipe::TaskKind::kFusedBackward:
        on_free(1, seg, idx, t);
        if (tk.segment == 1) on_free(0, kvo, mb, t);
        break;
      case seqpipe::TaskKind::kInputGrad:
        on_alloc(1, wo, idx, w_bytes(mc, L_s, len[tk.segment - 1], esz), t);
        break;
      case seqpipe::TaskKind::kWeightGrad:
        on_free(1, wo, idx, t);
        on_free(1, seg, idx, t);
        if (tk.segment == 1) on_free(0, kvo, mb, t);
        break;
    }
  }
  for (int p = 0; p < 2; ++p) {
    std::vector<PlacedBuf> pb;
    std::vector<size_t> who;
    for (size_t i = 0; i < bufs.size(); ++i)
      if (tags[i].pool == p) {
        pb.push_back(bufs[i]);
        who.push_back(i);
      }
    const int64_t extent = place_offline(pb);
    if (extent < a.pool[p].size) {
      a.pool[p].size = extent;
      for (size_t q = 0; q < pb.size(); ++q) (*tags[who[q]].vec)[tags[who[q]].idx] = pb[q].off;
    }
  }
  for (int64_t& o : seg)
    if (o >= 0) o += a.pool[0].size;  // record pool sits after the slab pool
  for (int64_t& o : wo)
    if (o >= 0) o += a.pool[0].size;
  return a;
}

DualArena plan_stage_memory(const ModelCfg& mc, const seqpipe::ScenarioConfig& cfg, const std::vector<int64_t>& len,
                            const std::vector<seqpipe::Task>& order, int stage) {
  std::vector<int64_t> seg, kvo, wo;
  return replay_plan(mc, cfg, len, order, stage, seg, kvo, wo);
}

int64_t Stage::record_bytes(int s) const { return seg_bytes(mc_, L_s_, len_[static_cast<size_t>(s - 1)], esz_); }
int64_t Stage::w_record_bytes(int s) const { return w_bytes(mc_, L_s_, len_[static_cast<size_t>(s - 1)], esz_); }
int64_t Stage::kv_slab_bytes() const { return static_cast<int64_t>(L_s_) * T_ * 2 * mc_.h * static_cast<int64_t>(esz_); }

void Stage::plan_arena(const std::vector<seqpipe::Task>& order) {
  arena_ = replay_plan(mc_, cfg_, len_, order, stage_, seg_off_, kv_off_, w_off_);
  if (arena_ptr_) cudaFree(arena_ptr_);
  SPK_CUDA(cudaMalloc(&arena_ptr_, std::max<int64_t>(arena_.size(), 256)));
  bind_step();
}

void Stage::bind_step() {
  const int64_t h = mc_.h;
  for (int m = 1; m <= M_; ++m) {
    for (int s = 1; s <= k_; ++s) {
      const size_t idx = static_cast<size_t>(m - 1) * k_ + (s - 1);
      Seg& g = segs_[idx];
      g.n = len_[s - 1];
      g.pos0 = prefix_[s - 1];
      if (seg_off_[idx] < 0) continue;
      uint8_t* p = arena_ptr_ + seg_off_[idx];
      auto take = [&](int64_t bytes) {
        void* r = p;
        p += (bytes + 255) / 256 * 256;
        return r;
      };
      const int64_t n = g.n;
      g.x_in.resize(L_s_);
      g.q.resize(L_s_);
      g.o.resize(L_s_);
      g.x_mid.resize(L_s_);
      g.u.resize(L_s_);
      g.mean1.resize(L_s_);
      g.rstd1.resize(L_s_);
      g.mean2.resize(L_s_);
      g.rstd2.resize(L_s_);
      g.lse.resize(L_s_);
      for (int l = 0; l < L_s_; ++l) g.x_in[l] = take(n * h * esz_);
      g.x_out = take(n * h * esz_);
      g.dy_in = take(n * h * esz_);
      for (int l = 0; l < L_s_; ++l) {
        g.q[l] = take(n * h * esz_);
        g.o[l] = take(n * h * esz_);
        g.x_mid[l] = take(n * h * esz_);
        g.u[l] = recompute_mlp() ? nullptr : take(n * mc_.Fup * esz_);
        g.mean1[l] = static_cast<float*>(take(n * 4));
        g.rstd1[l] = static_cast<float*>(take(n * 4));
        g.mean2[l] = static_cast<float*>(take(n * 4));
        g.rstd2[l] = static_cast<float*>(take(n * 4));
        g.lse[l] = static_cast<float*>(take(n * mc_.H * 4));
      }
      g.w_dy.assign(static_cast<size_t>(L_s_), nullptr);
      g.w_du.assign(static_cast<size_t>(L_s_), nullptr);
      g.w_dxm.assign(static_cast<size_t>(L_s_), nullptr);
      g.w_dqkv.assign(static_cast<size_t>(L_s_), nullptr);
      if (w_off_.size() > idx && w_off_[idx] >= 0) {
        p = arena_ptr_ + w_off_[idx];
        for (int l = 0; l < L_s_; ++l) {
          g.w_dy[l] = take(n * h * esz_);
          g.w_du[l] = take(n * mc_.Fup * esz_);
          g.w_dxm[l] = take(n * h * esz_);
          g.w_dqkv[l] = take(n * 3 * h * esz_);
        }
      }
    }
  }
}

void* Stage::kv(int m, int layer) const {
  const int64_t off = kv_off_[m - 1];
  if (off < 0) throw std::logic_error("KV slab not planned");
  return arena_ptr_ + off + static_cast<int64_t>(layer) * T_ * 2 * mc_.h * esz_;
}

void Stage::wgrad(const GemmArgs& a, double flop) {
  static const bool side = [] {
    const char* e = std::getenv("SP_WGRAD_STREAM");  // tuning: 0 = weight gradients in stream order
    return e ? std::atoi(e) != 0 : true;
  }();
  if (!side || (mc_.flags & SP_FLAG_NO_TCGEN05) || mc_.dt == DType::kF32) {
    gemm(a, flop);
    return;
  }
  if (!s2_) {
    SPK_CUDA(cudaStreamCreateWithFlags(&s2_, cudaStreamNonBlocking));
    SPK_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
    SPK_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
  }
  SPK_CUDA(cudaEventRecord(ev_fork_, s_));
  SPK_CUDA(cudaStreamWaitEvent(s2_, ev_fork_, 0));
  if (probe && probe->enabled) probe->begin(KernelProbe::kGemm, s2_, flop);  // timed on its own stream
  spk::gemm(a, s2_, spk::kGemmAuto);
  if (probe && probe->enabled) probe->end(s2_);
  SPK_CUDA(cudaEventRecord(ev_join_, s2_));
  pending_join_ = true;
  flops += flop;
  ++launches;
}

void Stage::join() {
  if (!pending_join_) return;
  SPK_CUDA(cudaStreamWaitEvent(s_, ev_join_, 0));
  pending_join_ = false;
}

void Stage::gemm(const GemmArgs& a, double flop) {
  int impl = spk::kGemmAuto;
  if (mc_.flags & SP_FLAG_NO_TCGEN05) impl = spk::kGemmSimt;
  if (probe && probe->enabled) probe->begin(KernelProbe::kGemm, s_, flop);
  spk::gemm(a, s_, impl);
  if (probe && probe->enabled) probe->end(s_);
  flops += flop;
  ++launches;
}

// ------------------------------------------------------------------ probes

cudaEvent_t KernelProbe::get() {
  if (next == pool.size()) {
    cudaEvent_t e;
    SPK_CUDA(cudaEventCreate(&e));
    pool.push_back(e);
  }
  return pool[next++];
}

void KernelProbe::begin(int cls, cudaStream_t s, double flops) {
  Rec r{cls, get(), get(), flops};
  SPK_CUDA(cudaEventRecord(r.a, s));
  recs.push_back(r);
}

void KernelProbe::end(cudaStream_t s) { SPK_CUDA(cudaEventRecord(recs.back().b, s)); }

void KernelProbe::totals(double (&ms)[kNumClasses], double (&fl)[kNumClasses], int64_t (&n)[kNumClasses]) {
  for (int c = 0; c < kNumClasses; ++c) {
    ms[c] = fl[c] = 0;
    n[c] = 0;
  }
  for (const Rec& r : recs) {
    float t = 0;
    SPK_CUDA(cudaEventElapsedTime(&t, r.a, r.b));
    ms[r.cls] += t;
    fl[r.cls] += r.flops;
    n[r.cls] += 1;
  }
}

KernelProbe::~KernelProbe() {
  for (cudaEvent_t e : pool) cudaEventDestroy(e);
}

namespace {
GemmArgs G(DType dt, int64_t M, int64_t N, int64_t K, const void* A, int64_t lda, bool ak, const void* B, int64_t ldb,
           bool bk, void* C, int64_t ldc, DType ct) {
  GemmArgs g;
  g.M = M;
  g.N = N;
  g.K = K;
  g.ab = dt;
  g.A = A;
  g.lda = lda;
  g.a_kmajor = ak;
  g.B = B;
  g.ldb = ldb;
  g.b_kmajor = bk;
  g.C = C;
  g.ldc = ldc;
  g.c = ct;
  return g;
}
}  // namespace

void Stage::forward(int m, int s, const int32_t* tokens, double* loss_acc, float loss_scale) {
  Seg& sg = seg(m, s);
  const int64_t n = sg.n, pos0 = sg.pos0, h = mc_.h;
  const DType dt = mc_.dt;
  const int attn_impl = (mc_.flags & SP_FLAG_NO_TC_ATTN) ? spk::kAttnSimt : spk::kAttnAuto;
  if (first()) {
    spk::embed_fwd(dt, tokens + (int64_t)(m - 1) * (T_ + 1) + pos0, wm(embed_), pos_ >= 0 ? wm(pos_) : nullptr, pos0,
                   sg.x_in[0], n, mc_.h, s_);
    ++launches;
  }
  for (int l = 0; l < L_s_; ++l) {
    const LayerW& w = lw_[l];
    void* x = sg.x_in[l];
    spk::norm_fwd(dt, mc_.rms(), x, wm(w.norm1), w_a_, mc_.rms() ? nullptr : sg.mean1[l], sg.rstd1[l], n, mc_.h,
                  mc_.eps, s_);
    // QKV projection; K/V columns land directly in the KV-prefix slab rows of this segment.
    void* kv_rows = static_cast<uint8_t*>(kv(m, l)) + pos0 * 2 * h * esz_;
    GemmArgs g = G(dt, n, 3 * h, h, w_a_, h, true, wc(w.wqkv), h, true, sg.q[l], h, dt);
    g.C2 = kv_rows;
    g.ldc2 = 2 * h;
    g.split_n = h;
    gemm(g, 2.0 * n * 3 * h * h);
    if (mc_.family == SP_MODEL_LLAMA) {
      spk::rope(dt, sg.q[l], h, n, mc_.H, mc_.hd, pos0, mc_.theta, false, s_);
      spk::rope(dt, kv_rows, 2 * h, n, mc_.H, mc_.hd, pos0, mc_.theta, false, s_);
      launches += 2;
    }
    const double attn_flops = 4.0 * h * (static_cast<double>(n) * pos0 + 0.5 * static_cast<double>(n) * n);
    if (probe && probe->enabled) probe->begin(KernelProbe::kAttnFwd, s_, attn_flops);
    spk::attn_fwd(dt, attn_impl, sg.q[l], kv(m, l), sg.o[l], sg.lse[l], n, pos0, pos0 + n, mc_.H, mc_.hd, s_);
    if (probe && probe->enabled) probe->end(s_);
    flops += attn_flops;
    ++launches;
    g = G(dt, n, h, h, sg.o[l], h, true, wc(w.wo), h, true, sg.x_mid[l], h, dt);
    g.epi = Epi::kAddResid;
    g.R = x;
    g.ldr = h;
    gemm(g, 2.0 * n * h * h);
    spk::norm_fwd(dt, mc_.rms(), sg.x_mid[l], wm(w.norm2), w_a_, mc_.rms() ? nullptr : sg.mean2[l], sg.rstd2[l], n,
                  mc_.h, mc_.eps, s_);
    void* u = recompute_mlp() ? w_big2_ : sg.u[l];  // w_big2_ is free in the forward
    gemm(G(dt, n, mc_.Fup, h, w_a_, h, true, wc(w.w1), h, true, u, mc_.Fup, dt), 2.0 * n * mc_.Fup * h);
    spk::act_fwd(dt, mc_.family, u, w_big1_, n, mc_.F, s_);
    void* y = (l + 1 < L_s_) ? sg.x_in[l + 1] : sg.x_out;
    g = G(dt, n, h, mc_.F, w_big1_, mc_.F, true, wc(w.w2), mc_.F, true, y, h, dt);
    g.epi = Epi::kAddResid;
    g.R = sg.x_mid[l];
    g.ldr = h;
    gemm(g, 2.0 * n * h * mc_.F);
    launches += 3;
  }
  if (last()) head_forward_backward(sg, m, tokens, loss_acc, loss_scale);
}

// Final norm + LM head + cross-entropy, fused with their backward so the
// [n, V] logits never persist: chunks of rows go logits -> CE/dlogits ->
// dgrad (dx_f) and wgrad (dW_lm) while resident. The stage output gradient is
// stored in dy_in for B(m,s).
void Stage::head_forward_backward(Seg& sg, int m, const int32_t* tokens, double* loss_acc, float loss_scale) {
  const int64_t n = sg.n, pos0 = sg.pos0, h = mc_.h, Vp = mc_.Vpad;
  const DType dt = mc_.dt;
  void* xf = w_t1_;
  void* dxf = w_t2_;
  spk::norm_fwd(dt, mc_.rms(), sg.x_out, wm(fnorm_), xf, mc_.rms() ? nullptr : w_fmean_, w_frstd_, n, mc_.h, mc_.eps, s_);
  const int32_t* labels = tokens + (int64_t)(m - 1) * (T_ + 1) + pos0 + 1;
  for (int64_t c0 = 0; c0 < n; c0 += logits_rows_) {
    const int64_t rows = std::min(logits_rows_, n - c0);
    const void* xf_c = static_cast<uint8_t*>(xf) + c0 * h * esz_;
    gemm(G(dt, rows, Vp, h, xf_c, h, true, wc(lm_), h, true, w_logits_, Vp, dt), 2.0 * rows * Vp * h);
    spk::ce_fwd_bwd(dt, w_logits_, Vp, labels + c0, rows, mc_.V, loss_scale, loss_acc, s_);
    gemm(G(dt, rows, h, Vp, w_logits_, Vp, true, wc(lm_), h, false, static_cast<uint8_t*>(dxf) + c0 * h * esz_, h, dt),
         2.0 * rows * Vp * h);
    GemmArgs g = G(dt, Vp, h, rows, w_logits_, Vp, false, xf_c, h, false, wg(lm_), h, DType::kF32);
    g.epi = Epi::kAccumF32;
    gemm(g, 2.0 * rows * Vp * h);
    ++launches;
  }
  spk::norm_bwd(dt, mc_.rms(), dxf, sg.x_out, wm(fnorm_), mc_.rms() ? nullptr : w_fmean_, w_frstd_, nullptr, sg.dy_in,
                wg(fnorm_), n, mc_.h, s_);
  launches += 2;
}

void Stage::backward(int m, int s, void* dx_target, const int32_t* tokens) {
  backward_impl(m, s, dx_target, tokens, false);
}

void Stage::backward_input(int m, int s, void* dx_target, const int32_t* tokens) {
  backward_impl(m, s, dx_target, tokens, true);
}

// W task: the four weight-gradient GEMMs per layer from the operands the I task
// saved; the norm outputs and the activation output are recomputed (elementwise).
void Stage::backward_weight(int m, int s) {
  Seg& sg = seg(m, s);
  const int64_t n = sg.n, h = mc_.h, F = mc_.F, Fu = mc_.Fup;
  const DType dt = mc_.dt;
  if (sg.w_dy.empty() || !sg.w_dy[0]) throw std::logic_error("W task without a planned W record");
  for (int l = L_s_ - 1; l >= 0; --l) {
    const LayerW& w = lw_[l];
    spk::act_fwd(dt, mc_.family, sg.u[l], w_big1_, n, F, s_);
    GemmArgs g = G(dt, h, F, n, sg.w_dy[l], h, false, w_big1_, F, false, wg(w.w2), F, DType::kF32);
    g.epi = Epi::kAccumF32;
    gemm(g, 2.0 * n * h * F);
    spk::norm_apply(dt, mc_.rms(), sg.x_mid[l], wm(w.norm2), sg.mean2[l], sg.rstd2[l], w_a_, n, mc_.h, s_);
    g = G(dt, Fu, h, n, sg.w_du[l], Fu, false, w_a_, h, false, wg(w.w1), h, DType::kF32);
    g.epi = Epi::kAccumF32;
    gemm(g, 2.0 * n * Fu * h);
    g = G(dt, h, h, n, sg.w_dxm[l], h, false, sg.o[l], h, false, wg(w.wo), h, DType::kF32);
    g.epi = Epi::kAccumF32;
    gemm(g, 2.0 * n * h * h);
    spk::norm_apply(dt, mc_.rms(), sg.x_in[l], wm(w.norm1), sg.mean1[l], sg.rstd1[l], w_a_, n, mc_.h, s_);
    g = G(dt, 3 * h, h, n, sg.w_dqkv[l], 3 * h, false, w_a_, h, false, wg(w.wqkv), h, DType::kF32);
    g.epi = Epi::kAccumF32;
    gemm(g, 2.0 * n * 3 * h * h);
    launches += 2;
  }
}

void Stage::backward_impl(int m, int s, void* dx_target, const int32_t* tokens, bool defer_w) {
  Seg& sg = seg(m, s);
  const int64_t n = sg.n, pos0 = sg.pos0, h = mc_.h, F = mc_.F, Fu = mc_.Fup;
  const DType dt = mc_.dt;
  const int attn_impl = (mc_.flags & SP_FLAG_NO_TC_ATTN) ? spk::kAttnSimt : spk::kAttnAuto;
  // s == k: the first backward op of the micro-batch covers every key row [0, T) and
  // WRITES the dK/dV accumulator (attn_bwd dkv_overwrite) -- no memset, no zero read.
  const void* dy = sg.dy_in;
  for (int l = L_s_ - 1; l >= 0; --l) {
    const LayerW& w = lw_[l];
    // ---- MLP: y = x_mid + act(norm2(x_mid) W1^T) W2^T
    void* u = sg.u[l];
    if (recompute_mlp()) {  // u = norm2(x_mid) W1^T again: the same GEMM on the same operands (bit-identical)
      if (defer_w) throw std::invalid_argument("SP_FLAG_RECOMPUTE_MLP is not supported by the zero-bubble kinds");
      spk::norm_apply(dt, mc_.rms(), sg.x_mid[l], wm(w.norm2), sg.mean2[l], sg.rstd2[l], w_a_, n, mc_.h, s_);
      gemm(G(dt, n, Fu, h, w_a_, h, true, wc(w.w1), h, true, w_u_, Fu, dt), 2.0 * n * Fu * h);
      u = w_u_;
      spk::act_fwd(dt, mc_.family, u, w_big1_, n, F, s_);
      ++launches;
    } else if (!defer_w) {  // recomputed operands of the W2 / W1 weight gradients
      spk::norm_apply(dt, mc_.rms(), sg.x_mid[l], wm(w.norm2), sg.mean2[l], sg.rstd2[l], w_a_, n, mc_.h, s_);
      spk::act_fwd(dt, mc_.family, u, w_big1_, n, F, s_);
    }
    GemmArgs g;
    if (defer_w) {
      SPK_CUDA(cudaMemcpyAsync(sg.w_dy[l], dy, esz_ * n * h, cudaMemcpyDeviceToDevice, s_));
    } else {
      g = G(dt, h, F, n, dy, h, false, w_big1_, F, false, wg(w.w2), F, DType::kF32);
      g.epi = Epi::kAccumF32;
      wgrad(g, 2.0 * n * h * F);
    }
    void* du = w_big1_;
    static const bool fuse_gelu_bwd = [] {
      const char* e = std::getenv("SP_FUSE_GELU_BWD");  // tuning: 0 = dgrad GEMM + elementwise GeLU backward
      return e ? std::atoi(e) != 0 : true;
    }();
    if (mc_.family == SP_MODEL_GPT && fuse_gelu_bwd) {
      // GeLU: du = (dy W2) * gelu'(u) straight from the dgrad GEMM's epilogue into w_big2_ --
      // no dg round trip through HBM, no activation-backward launch, and no wait for the W2
      // weight gradient (still reading g from w_big1_ on the side stream).
      g = G(dt, n, F, h, dy, h, true, wc(w.w2), F, false, w_big2_, F, dt);
      g.epi = Epi::kGeluGrad;
      g.R = u;
      g.ldr = Fu;
      gemm(g, 2.0 * n * h * F);
      du = w_big2_;
    } else {  // SwiGLU (du has two halves per row) or the unfused GeLU: the elementwise backward
      gemm(G(dt, n, F, h, dy, h, true, wc(w.w2), F, false, w_big2_, F, dt), 2.0 * n * h * F);
      join();  // act_bwd overwrites w_big1_
      spk::act_bwd(dt, mc_.family, u, w_big2_, w_big1_, n, F, s_);
      ++launches;
    }
    if (defer_w) {
      SPK_CUDA(cudaMemcpyAsync(sg.w_du[l], du, esz_ * n * Fu, cudaMemcpyDeviceToDevice, s_));
    } else {
      g = G(dt, Fu, h, n, du, Fu, false, w_a_, h, false, wg(w.w1), h, DType::kF32);
      g.epi = Epi::kAccumF32;
      wgrad(g, 2.0 * n * Fu * h);
    }
    gemm(G(dt, n, h, Fu, du, Fu, true, wc(w.w1), h, false, w_t1_, h, dt), 2.0 * n * Fu * h);
    join();
    spk::norm_bwd(dt, mc_.rms(), w_t1_, sg.x_mid[l], wm(w.norm2), sg.mean2[l], sg.rstd2[l], dy, w_t2_, wg(w.norm2), n,
                  mc_.h, s_);
    // ---- attention: x_mid = x + attn(norm1(x)) Wo^T
    if (defer_w) {
      SPK_CUDA(cudaMemcpyAsync(sg.w_dxm[l], w_t2_, esz_ * n * h, cudaMemcpyDeviceToDevice, s_));
    } else {
      g = G(dt, h, h, n, w_t2_, h, false, sg.o[l], h, false, wg(w.wo), h, DType::kF32);
      g.epi = Epi::kAccumF32;
      wgrad(g, 2.0 * n * h * h);
    }
    gemm(G(dt, n, h, h, w_t2_, h, true, wc(w.wo), h, false, w_t3_, h, dt), 2.0 * n * h * h);
    join();
    float* dkv_l = dkv(l);
    // Algorithmic count: backward = 2x forward attention FLOPs (SURVEY §8d convention).
    const double attn_flops = 2.0 * 4.0 * h * (static_cast<double>(n) * pos0 + 0.5 * static_cast<double>(n) * n);
    if (probe && probe->enabled) probe->begin(KernelProbe::kAttnBwd, s_, attn_flops);
    spk::attn_bwd(dt, attn_impl, sg.q[l], kv(m, l), sg.o[l], w_t3_, sg.lse[l], w_delta_, w_dq_, w_t1_, dkv_l, n, pos0,
                  pos0 + n, mc_.H, mc_.hd, s_, /*dkv_overwrite=*/s == k_);
    if (probe && probe->enabled) probe->end(s_);
    flops += attn_flops;
    float* dkv_rows = dkv_l + pos0 * 2 * h;  // complete after this op (reverse causal order)
    if (mc_.family == SP_MODEL_LLAMA) {
      spk::rope(dt, w_t1_, h, n, mc_.H, mc_.hd, pos0, mc_.theta, true, s_);
      spk::rope(DType::kF32, dkv_rows, 2 * h, n, mc_.H, mc_.hd, pos0, mc_.theta, true, s_);
      launches += 2;
    }
    spk::assemble_dqkv(dt, w_t1_, dkv_rows, w_dqkv_, n, mc_.h, s_);
    if (defer_w) {
      SPK_CUDA(cudaMemcpyAsync(sg.w_dqkv[l], w_dqkv_, esz_ * n * 3 * h, cudaMemcpyDeviceToDevice, s_));
    } else {
      spk::norm_apply(dt, mc_.rms(), sg.x_in[l], wm(w.norm1), sg.mean1[l], sg.rstd1[l], w_a_, n, mc_.h, s_);
      g = G(dt, 3 * h, h, n, w_dqkv_, 3 * h, false, w_a_, h, false, wg(w.wqkv), h, DType::kF32);
      g.epi = Epi::kAccumF32;
      wgrad(g, 2.0 * n * 3 * h * h);
    }
    gemm(G(dt, n, h, 3 * h, w_dqkv_, 3 * h, true, wc(w.wqkv), h, false, w_t1_, h, dt), 2.0 * n * 3 * h * h);
    join();
    void* dx = (l > 0) ? w_t2_ : (first() ? w_t3_ : dx_target);
    spk::norm_bwd(dt, mc_.rms(), w_t1_, sg.x_in[l], wm(w.norm1), sg.mean1[l], sg.rstd1[l], w_t2_, dx, wg(w.norm1), n,
                  mc_.h, s_);
    dy = w_t2_;
    launches += 7;  // norm_apply x2, act_fwd, norm_bwd x2, attn_bwd, assemble_dqkv
  }
  if (first()) {
    spk::embed_bwd(dt, tokens + (int64_t)(m - 1) * (T_ + 1) + pos0, w_t3_, wg(embed_), pos_ >= 0 ? wg(pos_) : nullptr,
                   pos0, n, mc_.h, s_);
    ++launches;
  }
}

}  // namespace spe
