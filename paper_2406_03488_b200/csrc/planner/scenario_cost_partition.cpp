// Host planner, part 1: scenario config, Eq. 8 cost model, partitions, POQ.
// Behaviour follows the reference seqpipe core (file:line cited per function);
// the code is written for this engine, not translated.
#include <algorithm>
#include <cmath>
#include <fstream>
#include <numeric>
#include <sstream>
#include <stdexcept>

#include "seqpipe/cost.hpp"
#include "seqpipe/partition.hpp"
#include "seqpipe/poq.hpp"
#include "seqpipe/scenario.hpp"
#include "seqpipe/task.hpp"

namespace seqpipe {

// ---------------------------------------------------------------- task / scenario

TaskKind parse_task_kind(const std::string& name) {  // ref scenario.cpp:14-20
  static const char* kNames[] = {"F", "B", "I", "W"};
  for (int i = 0; i < 4; ++i)
    if (name == kNames[i]) return static_cast<TaskKind>(i);
  throw std::invalid_argument("unknown task kind '" + name + "'");
}

void ScenarioConfig::validate() const {  // ref scenario.cpp:22-41
  struct Bound {
    bool ok;
    const char* msg;
  };
  const Bound bounds[] = {
      {pipeline_size >= 1, "pipeline_size must be >= 1"},
      {stages_per_device >= 1, "stages_per_device must be >= 1"},
      {micro_batches >= 1, "micro_batches must be >= 1"},
      {segments >= 1, "segments must be >= 1"},
      {seq_len >= segments, "seq_len must be >= segments (every segment non-empty)"},
      {layers >= 0, "layers must be >= 0"},
      {hidden_dim >= 0, "hidden_dim must be >= 0"},
      {param_count >= 0, "param_count must be >= 0"},
      {backward_ratio.is_positive(), "backward_ratio must be positive"},
      {bw_input_ratio.is_positive() && bw_weight_ratio.is_positive(), "bw_split_ratio components must be positive"},
      {!comm_latency.is_negative(), "comm_latency must be non-negative"},
      {activation_cost_per_token.is_positive(), "activation_cost_per_token must be positive"},
      {time_per_flop.is_positive(), "time_per_flop must be positive"},
      {uniform_forward.is_positive(), "uniform_forward must be positive"},
  };
  for (const Bound& b : bounds)
    if (!b.ok) throw std::invalid_argument(std::string("invalid scenario: ") + b.msg);
}

const char* cost_model_name(CostModel m) { return m == CostModel::kUniform ? "uniform" : "flops"; }

CostModel parse_cost_model(std::string_view name) {
  if (name == "flops") return CostModel::kFlops;
  if (name == "uniform") return CostModel::kUniform;
  throw std::invalid_argument("unknown cost_model '" + std::string(name) + "'");
}

namespace {

std::string_view strip(std::string_view s) {
  auto ws = [](char c) { return c == ' ' || c == '\t' || c == '\r'; };
  std::size_t b = 0, e = s.size();
  while (b < e && ws(s[b])) ++b;
  while (e > b && ws(s[e - 1])) --e;
  return s.substr(b, e - b);
}

std::int64_t to_int(std::string_view key, std::string_view value) {
  std::string text(value);
  std::size_t used = 0;
  std::int64_t v = 0;
  bool ok = true;
  try {
    v = std::stoll(text, &used);
  } catch (const std::exception&) {
    ok = false;
  }
  if (!ok || used != text.size())
    throw std::invalid_argument("config key '" + std::string(key) + "': expected integer, got '" + text + "'");
  return v;
}

}  // namespace

void apply_scenario_override(ScenarioConfig& cfg, std::string_view key, std::string_view value) {
  // ref scenario.cpp:76-117 (same key set; unknown keys throw)
  key = strip(key);
  value = strip(value);
  auto i32 = [&](int& f) { f = static_cast<int>(to_int(key, value)); };
  auto i64 = [&](std::int64_t& f) { f = to_int(key, value); };
  auto rat = [&](Rational& f) { f = Rational::parse(value); };
  if (key == "pipeline_size") return i32(cfg.pipeline_size);
  if (key == "stages_per_device") return i32(cfg.stages_per_device);
  if (key == "micro_batches") return i32(cfg.micro_batches);
  if (key == "segments") return i32(cfg.segments);
  if (key == "seq_len") return i64(cfg.seq_len);
  if (key == "layers") return i32(cfg.layers);
  if (key == "hidden_dim") return i64(cfg.hidden_dim);
  if (key == "param_count") return i64(cfg.param_count);
  if (key == "backward_ratio") return rat(cfg.backward_ratio);
  if (key == "comm_latency") return rat(cfg.comm_latency);
  if (key == "activation_cost_per_token") return rat(cfg.activation_cost_per_token);
  if (key == "time_per_flop") return rat(cfg.time_per_flop);
  if (key == "uniform_forward") return rat(cfg.uniform_forward);
  if (key == "cost_model") {
    cfg.cost_model = parse_cost_model(value);
    return;
  }
  if (key == "bw_split_ratio") {
    std::size_t comma = value.find(',');
    if (comma == std::string_view::npos) throw std::invalid_argument("bw_split_ratio expects 'input,weight'");
    cfg.bw_input_ratio = Rational::parse(strip(value.substr(0, comma)));
    cfg.bw_weight_ratio = Rational::parse(strip(value.substr(comma + 1)));
    return;
  }
  throw std::invalid_argument("unknown config key '" + std::string(key) + "'");
}

ScenarioConfig parse_scenario_text(std::string_view text) {  // ref scenario.cpp:119-139
  ScenarioConfig cfg;
  std::size_t line_no = 0, pos = 0;
  while (pos <= text.size()) {
    std::size_t nl = text.find('\n', pos);
    std::size_t end = nl == std::string_view::npos ? text.size() : nl;
    std::string_view line = text.substr(pos, end - pos);
    pos = end + 1;
    ++line_no;
    if (std::size_t hash = line.find('#'); hash != std::string_view::npos) line = line.substr(0, hash);
    line = strip(line);
    if (line.empty()) continue;
    std::size_t eq = line.find('=');
    if (eq == std::string_view::npos)
      throw std::invalid_argument("config line " + std::to_string(line_no) + ": expected 'key = value'");
    apply_scenario_override(cfg, line.substr(0, eq), line.substr(eq + 1));
  }
  return cfg;
}

ScenarioConfig load_scenario_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw std::runtime_error("cannot open config file '" + path + "'");
  std::stringstream ss;
  ss << in.rdbuf();
  return parse_scenario_text(ss.str());
}

namespace {
// Table 1 model scales (ref scenario.cpp:163-168): name, P, L, d, seq, M, params. k = 4.
struct PresetRow {
  const char* name;
  int pipeline, layers;
  std::int64_t hidden, seq;
  int micro_batches;
  std::int64_t params;
};
constexpr PresetRow kPresetTable[] = {
    {"gpt-2.7b", 8, 32, 2560, 16384, 32, 2700000000LL},
    {"gpt-7b", 4, 32, 4096, 32768, 16, 7000000000LL},
    {"gpt-13b", 4, 40, 5120, 32768, 16, 13000000000LL},
    {"gpt-30b", 8, 64, 6144, 32768, 32, 30000000000LL},
};
}  // namespace

ScenarioConfig preset_scenario(std::string_view name) {
  for (const PresetRow& r : kPresetTable) {
    if (name != r.name) continue;
    ScenarioConfig cfg;
    cfg.pipeline_size = r.pipeline;
    cfg.micro_batches = r.micro_batches;
    cfg.segments = 4;
    cfg.seq_len = r.seq;
    cfg.layers = r.layers;
    cfg.hidden_dim = r.hidden;
    cfg.param_count = r.params;
    cfg.validate();
    return cfg;
  }
  throw std::invalid_argument("unknown preset '" + std::string(name) + "'");
}

std::vector<std::string> preset_names() {
  std::vector<std::string> out;
  for (const PresetRow& r : kPresetTable) out.emplace_back(r.name);
  return out;
}

bool is_preset_name(std::string_view name) {
  return std::any_of(std::begin(kPresetTable), std::end(kPresetTable),
                     [&](const PresetRow& r) { return name == r.name; });
}

std::string scenario_to_text(const ScenarioConfig& c) {  // same line format as ref scenario.cpp:194-212
  std::ostringstream o;
  o << "pipeline_size = " << c.pipeline_size << "\nstages_per_device = " << c.stages_per_device
    << "\nmicro_batches = " << c.micro_batches << "\nsegments = " << c.segments << "\nseq_len = " << c.seq_len
    << "\nlayers = " << c.layers << "\nhidden_dim = " << c.hidden_dim << "\nparam_count = " << c.param_count
    << "\nbackward_ratio = " << c.backward_ratio.str() << "\nbw_split_ratio = " << c.bw_input_ratio.str() << ','
    << c.bw_weight_ratio.str() << "\ncomm_latency = " << c.comm_latency.str()
    << "\nactivation_cost_per_token = " << c.activation_cost_per_token.str()
    << "\ntime_per_flop = " << c.time_per_flop.str() << "\ncost_model = " << cost_model_name(c.cost_model)
    << "\nuniform_forward = " << c.uniform_forward.str() << '\n';
  return o.str();
}

// ---------------------------------------------------------------- cost (ref cost.cpp)

std::int64_t segment_prefix(const SequencePartition& p, int i) {  // ref cost.cpp:10-18
  if (i < 1 || i > p.segment_count())
    throw std::out_of_range("segment index " + std::to_string(i) + " out of range [1, " +
                            std::to_string(p.segment_count()) + "]");
  return std::accumulate(p.lengths.begin(), p.lengths.begin() + i, std::int64_t{0});
}

detail::Int128 segment_flops(const ScenarioConfig& cfg, std::int64_t prefix_before, std::int64_t n) {
  // ref cost.cpp:20-26: 2*n*params + 2*L*n*(prefix_before+n)*d
  using detail::Int128;
  return Int128(2) * n * cfg.param_count + Int128(2) * cfg.layers * n * (Int128(prefix_before) + n) * cfg.hidden_dim;
}

Rational forward_cost(const ScenarioConfig& cfg, const SequencePartition& p, int i) {  // ref cost.cpp:28-44
  if (i < 1 || i > p.segment_count()) throw std::out_of_range("segment index out of range");
  if (cfg.cost_model == CostModel::kUniform)
    return cfg.uniform_forward / Rational(std::int64_t(cfg.segments) * cfg.stages_per_device);
  const std::int64_t n = p.lengths[static_cast<std::size_t>(i - 1)];
  const std::int64_t before = segment_prefix(p, i) - n;
  Rational cost = Rational::reduce(segment_flops(cfg, before, n), cfg.total_stages()) * cfg.time_per_flop;
  if (!cost.is_positive())
    throw std::domain_error("forward cost is not positive; the cost model is degenerate "
                            "(layers*hidden_dim = 0 and param_count = 0)");
  return cost;
}

Rational task_cost(const ScenarioConfig& cfg, const SequencePartition& p, const Task& t) {  // ref cost.cpp:46-55
  const Rational f = forward_cost(cfg, p, t.segment);
  switch (t.kind) {
    case TaskKind::kForward: return f;
    case TaskKind::kFusedBackward: return f * cfg.backward_ratio;
    case TaskKind::kInputGrad: return f * cfg.bw_input_ratio;
    case TaskKind::kWeightGrad: return f * cfg.bw_weight_ratio;
  }
  throw std::logic_error("unreachable task kind");
}

// ---------------------------------------------------------------- partitions (ref partition.cpp)

const char* partition_mode_name(PartitionMode m) {
  switch (m) {
    case PartitionMode::kEven: return "even";
    case PartitionMode::kCwp: return "cwp";
    case PartitionMode::kOracle: return "oracle";
  }
  return "?";
}

PartitionMode parse_partition_mode(std::string_view name) {
  for (PartitionMode m : {PartitionMode::kEven, PartitionMode::kCwp, PartitionMode::kOracle})
    if (name == partition_mode_name(m)) return m;
  throw std::invalid_argument("unknown partition mode '" + std::string(name) + "'");
}

namespace {

bool all_zero_costs(const ScenarioConfig& cfg) {  // ref partition.cpp:33-35
  return std::int64_t(cfg.layers) * cfg.hidden_dim == 0 && cfg.param_count == 0;
}

// Exact (max - min) * k / sum over segment FLOPs (ref partition.cpp:38-56).
Rational exact_imbalance(const std::vector<std::int64_t>& len, const ScenarioConfig& cfg) {
  using detail::Int128;
  Int128 lo = 0, hi = 0, total = 0;
  std::int64_t before = 0;
  for (std::size_t i = 0; i < len.size(); ++i) {
    Int128 c = segment_flops(cfg, before, len[i]);
    before += len[i];
    total += c;
    lo = i ? std::min(lo, c) : c;
    hi = i ? std::max(hi, c) : c;
  }
  return total == 0 ? Rational(0) : Rational::reduce((hi - lo) * Int128(len.size()), total);
}

}  // namespace

SequencePartition make_partition(std::vector<std::int64_t> lengths, const ScenarioConfig& cfg) {
  if (lengths.empty()) throw std::invalid_argument("partition must have at least one segment");
  std::int64_t sum = 0;
  for (std::int64_t n : lengths) {
    if (n < 1) throw std::invalid_argument("every partition segment must hold at least one token");
    sum += n;
  }
  if (sum != cfg.seq_len)
    throw std::invalid_argument("partition lengths sum to " + std::to_string(sum) + " but seq_len is " +
                                std::to_string(cfg.seq_len));
  SequencePartition out;
  out.imbalance = exact_imbalance(lengths, cfg);
  out.total = sum;
  out.lengths = std::move(lengths);
  return out;
}

SequencePartition even_partition(std::int64_t n, int k, const ScenarioConfig& cfg) {  // ref partition.cpp:78-93
  if (k < 1) throw std::invalid_argument("segment count must be >= 1");
  if (n < k)
    throw std::invalid_argument("cannot split " + std::to_string(n) + " tokens into " + std::to_string(k) +
                                " non-empty segments");
  std::vector<std::int64_t> len(static_cast<std::size_t>(k));
  for (int i = 0; i < k; ++i) len[static_cast<std::size_t>(i)] = n / k + (i < n % k ? 1 : 0);
  ScenarioConfig local = cfg;
  local.seq_len = n;
  local.segments = k;
  return make_partition(std::move(len), local);
}

SequencePartition even_partition(const ScenarioConfig& cfg) { return even_partition(cfg.seq_len, cfg.segments, cfg); }

std::vector<double> cwp_continuous_lengths(const ScenarioConfig& cfg, double target) {
  // ref partition.cpp:100-117. Segment i solves a x^2 + b_i x = target with
  // b_i = 2*params + a*prefix_i; the same double operation order as the
  // reference (the build passes -ffp-contract=off so no FMA is formed).
  const double a = 2.0 * static_cast<double>(cfg.layers) * static_cast<double>(cfg.hidden_dim);
  std::vector<double> x(static_cast<std::size_t>(cfg.segments));
  double prefix = 0.0;
  for (double& xi : x) {
    const double b = 2.0 * static_cast<double>(cfg.param_count) + a * prefix;
    xi = (a == 0.0) ? target / b : (-b + std::sqrt(b * b + 4.0 * a * target)) / (2.0 * a);
    prefix += xi;
  }
  return x;
}

namespace {

// Largest-remainder rounding preserving the integer total (ref partition.cpp:120-153).
std::vector<std::int64_t> largest_remainder(const std::vector<double>& v, std::int64_t total) {
  const std::size_t k = v.size();
  std::vector<std::int64_t> out(k);
  std::vector<std::pair<double, std::size_t>> frac(k);
  std::int64_t assigned = 0;
  for (std::size_t i = 0; i < k; ++i) {
    const double c = std::max(0.0, v[i]);
    out[i] = static_cast<std::int64_t>(std::floor(c));
    frac[i] = {c - static_cast<double>(out[i]), i};
    assigned += out[i];
  }
  std::stable_sort(frac.begin(), frac.end(), [](const auto& x, const auto& y) { return x.first > y.first; });
  std::int64_t left = total - assigned;
  std::size_t turn = 0;
  for (; left > 0; --left, ++turn) out[frac[turn % k].second] += 1;
  while (left < 0) {  // only reachable through floating error: trim smallest remainders first
    std::size_t victim = frac[k - 1 - (turn % k)].second;
    if (out[victim] > 0) {
      out[victim] -= 1;
      ++left;
    }
    ++turn;
  }
  return out;
}

}  // namespace

SequencePartition cwp_partition(const ScenarioConfig& cfg) {  // ref partition.cpp:157-207
  if (cfg.seq_len < cfg.segments) throw std::invalid_argument("seq_len must be >= segments");
  if (all_zero_costs(cfg)) throw std::domain_error("cannot balance segments under an all-zero cost model");
  const std::int64_t n = cfg.seq_len;
  if (cfg.segments == 1) return make_partition({n}, cfg);

  const double nd = static_cast<double>(n);
  double lo = 0.0;
  double hi = 2.0 * nd * static_cast<double>(cfg.param_count) +
              2.0 * static_cast<double>(cfg.layers) * nd * nd * static_cast<double>(cfg.hidden_dim);
  double mid = hi;
  for (int it = 0; it < 200; ++it) {
    mid = 0.5 * (lo + hi);
    std::vector<double> x = cwp_continuous_lengths(cfg, mid);
    const double sum = std::accumulate(x.begin(), x.end(), 0.0);
    if (std::abs(sum - nd) <= 1e-6 * nd) break;
    (sum < nd ? lo : hi) = mid;
  }
  std::vector<std::int64_t> len = largest_remainder(cwp_continuous_lengths(cfg, mid), n);
  for (std::size_t i = 0; i < len.size(); ++i) {  // n_i >= 1 repair from the longest segment
    while (len[i] < 1) {
      std::size_t big = static_cast<std::size_t>(std::max_element(len.begin(), len.end()) - len.begin());
      if (len[big] <= 1) throw std::logic_error("cannot repair degenerate partition");
      --len[big];
      ++len[i];
    }
  }
  return make_partition(std::move(len), cfg);
}

SequencePartition oracle_partition(const ScenarioConfig& cfg) {  // ref partition.cpp:258-272
  if (cfg.seq_len > 512 || cfg.segments > 4)
    throw std::invalid_argument("oracle_partition is guarded to seq_len <= 512 and segments <= 4");
  if (cfg.seq_len < cfg.segments) throw std::invalid_argument("seq_len must be >= segments");
  if (all_zero_costs(cfg)) throw std::domain_error("cannot balance segments under an all-zero cost model");
  using detail::Int128;
  const int k = cfg.segments;
  const std::int64_t n = cfg.seq_len;
  // Iterative odometer over compositions in lexicographic order; strict
  // improvement keeps the lexicographically smallest optimum.
  std::vector<std::int64_t> cur(static_cast<std::size_t>(k), 1), best;
  Int128 best_spread = 0, best_sum = 0;
  cur[static_cast<std::size_t>(k - 1)] = n - (k - 1);
  while (true) {
    Int128 lo = 0, hi = 0, sum = 0;
    std::int64_t before = 0;
    for (int i = 0; i < k; ++i) {
      Int128 c = segment_flops(cfg, before, cur[static_cast<std::size_t>(i)]);
      before += cur[static_cast<std::size_t>(i)];
      sum += c;
      lo = i ? std::min(lo, c) : c;
      hi = i ? std::max(hi, c) : c;
    }
    if (sum != 0 && (best.empty() || (hi - lo) * best_sum < best_spread * sum)) {
      best = cur;
      best_spread = hi - lo;
      best_sum = sum;
    }
    // advance: bump the deepest non-final position that can still grow
    int pos = k - 2;
    while (pos >= 0) {
      std::int64_t head = 0;
      for (int i = 0; i <= pos; ++i) head += cur[static_cast<std::size_t>(i)];
      if (head + 1 <= n - (k - 1 - pos)) break;
      --pos;
    }
    if (pos < 0) break;
    cur[static_cast<std::size_t>(pos)] += 1;
    std::int64_t head = 0;
    for (int i = 0; i <= pos; ++i) head += cur[static_cast<std::size_t>(i)];
    for (int i = pos + 1; i < k - 1; ++i) {
      cur[static_cast<std::size_t>(i)] = 1;
      head += 1;
    }
    cur[static_cast<std::size_t>(k - 1)] = n - head;
  }
  if (best.empty()) throw std::logic_error("oracle found no composition");
  return make_partition(std::move(best), cfg);
}

SequencePartition partition_for(const ScenarioConfig& cfg, PartitionMode mode) {
  switch (mode) {
    case PartitionMode::kEven: return even_partition(cfg);
    case PartitionMode::kCwp: return cwp_partition(cfg);
    case PartitionMode::kOracle: return oracle_partition(cfg);
  }
  throw std::logic_error("unreachable partition mode");
}

BalanceReport balance_report(const SequencePartition& p, const ScenarioConfig& cfg) {  // ref partition.cpp:283-303
  BalanceReport r;
  for (int i = 1; i <= p.segment_count(); ++i) r.segment_costs.push_back(forward_cost(cfg, p, i));
  Rational lo = r.segment_costs.front(), hi = lo, sum{0};
  for (const Rational& c : r.segment_costs) {
    lo = std::min(lo, c);
    hi = std::max(hi, c);
    sum += c;
  }
  r.imbalance = sum.is_zero() ? Rational(0) : (hi - lo) * Rational(p.segment_count()) / sum;
  return r;
}

// ---------------------------------------------------------------- POQ (ref poq.cpp:11-30)

void PartiallyOrderedQueue::push(int micro_batch, int segment) {
  if (!keys_.emplace(micro_batch, -segment).second)
    throw std::invalid_argument("duplicate queue entry (" + std::to_string(micro_batch) + ", " +
                                std::to_string(segment) + ")");
}

std::pair<int, int> PartiallyOrderedQueue::pop() {
  if (keys_.empty()) throw std::out_of_range("pop on empty queue");
  auto front = *keys_.begin();
  keys_.erase(keys_.begin());
  return {front.first, -front.second};
}

}  // namespace seqpipe
