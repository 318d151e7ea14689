// seqpipe_b200: command-line front end of the B200 engine.
//
// The four planning subcommands keep the reference CLI's surface and output
// bytes (tools/src/seqpipe_main.cpp:122-289: simulate, sweep, partition,
// validate; exit codes :29-32 -- 0 ok, 1 runtime error, 2 usage, 3 validation
// failure); `execute` is new: it generates the same op table,
// RUNS it on one B200 through the engine C-ABI and writes the measured step as
// seqpipe.simreport.v1 (+ an optional timeline), so a sweep row can be checked
// against hardware. CLI11 (the reference's parser) is not in this image; the
// option grammar below accepts what the reference's subcommands accept:
// `--opt value`, `--opt=value`, repeated or space-separated `--set k=v`.
#include <cctype>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <ctime>
#include <fstream>
#include <functional>
#include <iostream>
#include <map>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "seqpipe/json_io.hpp"
#include "seqpipe/partition.hpp"
#include "seqpipe/render.hpp"
#include "seqpipe/scenario.hpp"
#include "seqpipe/schedule.hpp"
#include "seqpipe/sim.hpp"
#include "seqpipe/validate.hpp"
#include "capi/capi_common.hpp"
#include "seqpipe_b200.h"

namespace {

using namespace seqpipe;

enum Exit { kOk = 0, kRuntime = 1, kUsage = 2, kValidation = 3 };

struct UsageError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct ValidationFailure : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ---------------------------------------------------------------- options

struct Spec {
  std::string name;   // "--kind"
  std::string alias;  // "-k" or empty
  bool flag = false;  // takes no value
  bool multi = false; // --set: consumes values until the next option
  std::string help;
  std::vector<std::string> choices = {};  // CLI::IsMember of the reference (values normalised to the member)
  bool ignore_case = false;
};

class Options {
 public:
  Options(std::string cmd, std::vector<Spec> specs, std::vector<std::string> positional = {})
      : cmd_(std::move(cmd)), specs_(std::move(specs)), positional_names_(std::move(positional)) {}

  void parse(const std::vector<std::string>& args) {
    for (std::size_t i = 0; i < args.size(); ++i) {
      std::string a = args[i], val;
      bool has_val = false;
      if (a.rfind("--", 0) == 0 && a.find('=') != std::string::npos) {
        val = a.substr(a.find('=') + 1);
        a = a.substr(0, a.find('='));
        has_val = true;
      }
      if (a == "--help" || a == "-h") throw UsageError(usage());
      if (!a.empty() && a[0] == '-' && a.size() > 1) {
        const Spec* s = find(a);
        if (!s) throw UsageError("The following argument was not expected: " + a + "\n" + usage());
        if (s->flag) {
          if (has_val) throw UsageError(s->name + " takes no value");
          flags_[s->name] = true;
          continue;
        }
        auto& dst = values_[s->name];
        if (!s->multi) dst.clear();
        if (has_val) {
          dst.push_back(val);
        } else {
          if (i + 1 >= args.size()) throw UsageError(s->name + " requires an argument");
          dst.push_back(args[++i]);
        }
        while (s->multi && i + 1 < args.size() && !(args[i + 1].size() > 1 && args[i + 1][0] == '-'))
          dst.push_back(args[++i]);
        if (!s->choices.empty()) check_member(*s, dst.back());
        continue;
      }
      if (positional_.size() >= positional_names_.size())
        throw UsageError("The following argument was not expected: " + a + "\n" + usage());
      positional_.push_back(a);
    }
    if (positional_.size() < positional_names_.size())
      throw UsageError(positional_names_[positional_.size()] + " is required\n" + usage());
  }

  bool flag(const std::string& n) const { return flags_.count(n) != 0; }
  bool has(const std::string& n) const { return values_.count(n) != 0; }
  std::string str(const std::string& n, const std::string& dflt = "") const {
    auto it = values_.find(n);
    return it == values_.end() ? dflt : it->second.back();
  }
  std::vector<std::string> all(const std::string& n) const {
    auto it = values_.find(n);
    return it == values_.end() ? std::vector<std::string>{} : it->second;
  }
  long long integer(const std::string& n, long long dflt) const {
    if (!has(n)) return dflt;
    const std::string v = str(n);
    std::size_t used = 0;
    long long x = 0;
    try {
      x = std::stoll(v, &used);
    } catch (const std::exception&) {
      used = 0;
    }
    if (used != v.size() || v.empty()) throw UsageError(n + ": Value " + v + " could not be converted");
    return x;
  }
  const std::string& positional(std::size_t i) const { return positional_.at(i); }

  std::string usage() const {
    std::string u = "Usage: seqpipe_b200 " + cmd_;
    for (const auto& p : positional_names_) u += " " + p;
    u += " [OPTIONS]\n";
    for (const Spec& s : specs_) u += "  " + s.name + (s.alias.empty() ? "" : "," + s.alias) + "  " + s.help + "\n";
    return u;
  }

 private:
  static void check_member(const Spec& s, std::string& v) {
    auto fold = [&](std::string x) {
      if (s.ignore_case)
        for (char& c : x) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
      return x;
    };
    for (const std::string& c : s.choices)
      if (fold(c) == fold(v)) {
        v = c;
        return;
      }
    std::string set;
    for (const std::string& c : s.choices) set += (set.empty() ? "" : ",") + c;
    throw UsageError(s.name + ": " + v + " not in {" + set + "}");
  }
  const Spec* find(const std::string& a) const {
    for (const Spec& s : specs_)
      if (s.name == a || (!s.alias.empty() && s.alias == a)) return &s;
    return nullptr;
  }
  std::string cmd_;
  std::vector<Spec> specs_;
  std::vector<std::string> positional_names_, positional_;
  std::map<std::string, std::vector<std::string>> values_;
  std::map<std::string, bool> flags_;
};

std::vector<Spec> with_config(std::vector<Spec> s) {
  s.push_back({"--config", "", false, false, "scenario config file (key = value lines) or preset name"});
  s.push_back({"--preset", "", false, false, "bundled scenario preset"});
  s.push_back({"--set", "", false, true, "override a config key, e.g. --set segments=4"});
  return s;
}

// Reference resolve_config (seqpipe_main.cpp:53-72): preset | file, then --set overrides, then validate.
ScenarioConfig resolve_config(const Options& o) {
  if (o.has("--config") && o.has("--preset")) throw UsageError("--config excludes --preset");
  ScenarioConfig cfg;
  if (o.has("--preset")) {
    if (!is_preset_name(o.str("--preset"))) throw UsageError("--preset: unknown preset " + o.str("--preset"));
    cfg = preset_scenario(o.str("--preset"));
  } else if (o.has("--config")) {
    const std::string c = o.str("--config");
    cfg = is_preset_name(c) ? preset_scenario(c) : load_scenario_file(c);
  }
  for (const std::string& kv : o.all("--set")) {
    const auto eq = kv.find('=');
    if (eq == std::string::npos) throw std::invalid_argument("--set expects key=value, got '" + kv + "'");
    apply_scenario_override(cfg, kv.substr(0, eq), kv.substr(eq + 1));
  }
  cfg.validate();
  return cfg;
}

void emit(const std::string& path, const std::string& text) {
  if (path.empty() || path == "-") {
    std::cout << text;
    return;
  }
  std::ofstream f(path, std::ios::binary);
  if (!f) throw std::runtime_error("cannot write '" + path + "'");
  f << text;
}

std::string utc_now() {
  const std::time_t t = std::chrono::system_clock::to_time_t(std::chrono::system_clock::now());
  std::tm tm{};
  gmtime_r(&t, &tm);
  char b[32];
  std::strftime(b, sizeof b, "%Y-%m-%dT%H:%M:%SZ", &tm);
  return b;
}

std::string with_stamp(std::string json) {  // generated_at after the schema line (reference :139-144)
  json.insert(json.find('\n') + 1, "  \"generated_at\": \"" + utc_now() + "\",\n");
  return json;
}

std::vector<std::string> csv_items(const std::string& text) {
  std::vector<std::string> out;
  std::string cur;
  std::istringstream in(text);
  while (std::getline(in, cur, ','))
    if (!cur.empty()) out.push_back(cur);
  return out;
}

std::string gantt_of(const SimReport& r, const std::string& mode, int width) {
  return mode == "svg" ? render_svg_gantt(r) : render_ascii_gantt(r, width);
}

// ---------------------------------------------------------------- simulate

int cmd_simulate(const std::vector<std::string>& args) {
  Options o("simulate", with_config({{"--kind", "", false, false, "schedule kind", {"gpipe", "1f1b", "1f1b-i", "seq1f1b", "seq1f1b-i", "zb1p", "seqzb1p"}, true},
                                     {"--partition", "", false, false, "sequence partitioner", {"even", "cwp"}},
                                     {"--out", "", false, false, "report JSON path ('-' = stdout)"},
                                     {"--emit-schedule", "", false, false, "also write the schedule JSON"},
                                     {"--gantt", "", false, false, "render a timeline", {"ascii", "svg"}},
                                     {"--gantt-out", "", false, false, "timeline path ('-' = stdout)"},
                                     {"--gantt-width", "", false, false, "ascii timeline width in columns"},
                                     {"--memory-downsample", "", false, false, "keep every n-th memory point"},
                                     {"--validate", "", true, false, "check the schedule before simulating"},
                                     {"--stamp", "", true, false, "include a generation timestamp"}}));
  o.parse(args);
  if (!o.has("--kind")) throw UsageError("--kind is required\n" + o.usage());
  const ScenarioConfig cfg = resolve_config(o);
  const SequencePartition part = partition_for(cfg, parse_partition_mode(o.str("--partition", "even")));
  const Schedule sch = generate(cfg, parse_schedule_kind(o.str("--kind")), part);
  if (o.flag("--validate")) {
    const auto v = check_schedule(sch);
    if (!v.empty()) throw ValidationFailure(violations_to_string(v));
  }
  if (o.has("--emit-schedule")) emit(o.str("--emit-schedule"), schedule_to_json(sch));
  const SimReport rep = simulate(sch, part);
  const std::string json =
      report_to_json(rep, 2, static_cast<std::size_t>(o.integer("--memory-downsample", 0)));
  emit(o.str("--out"), o.flag("--stamp") ? with_stamp(json) : json);
  if (o.has("--gantt"))
    emit(o.str("--gantt-out"), gantt_of(rep, o.str("--gantt"), static_cast<int>(o.integer("--gantt-width", 120))));
  return kOk;
}

// ---------------------------------------------------------------- sweep

int cmd_sweep(const std::vector<std::string>& args) {
  Options o("sweep", with_config({{"--kinds", "", false, false, "comma-separated schedule kinds"},
                                  {"--pipeline-sizes", "", false, false, "comma-separated P values"},
                                  {"--micro-batches", "", false, false, "comma-separated M values"},
                                  {"--segment-counts", "", false, false, "comma-separated k values"},
                                  {"--stages-per-device", "", false, false, "comma-separated n_v values"},
                                  {"--seq-lens", "", false, false, "comma-separated sequence lengths"},
                                  {"--partition", "", false, false, "sequence partitioner", {"even", "cwp"}},
                                  {"--out", "", false, false, "CSV path ('-' = stdout)"},
                                  {"--stamp", "", true, false, "include a generation timestamp"}}));
  o.parse(args);
  const ScenarioConfig base = resolve_config(o);
  const PartitionMode mode = parse_partition_mode(o.str("--partition", "even"));
  auto ints = [&](const std::string& opt, std::int64_t dflt) {
    std::vector<std::int64_t> v;
    for (const std::string& s : csv_items(o.str(opt))) v.push_back(std::stoll(s));
    if (v.empty()) v.push_back(dflt);
    return v;
  };
  const auto kinds = csv_items(o.str("--kinds", "gpipe,1f1b,1f1b-i,seq1f1b,seq1f1b-i,zb1p,seqzb1p"));
  const auto Ps = ints("--pipeline-sizes", base.pipeline_size), NVs = ints("--stages-per-device", base.stages_per_device),
             Ms = ints("--micro-batches", base.micro_batches), Ks = ints("--segment-counts", base.segments),
             Ts = ints("--seq-lens", base.seq_len);
  auto safe = [](std::string s) {
    for (char& c : s)
      if (c == ',' || c == '\n' || c == '\r') c = ';';
    return s;
  };
  std::string csv = o.flag("--stamp") ? "# generated_at " + utc_now() + "\n" : "";
  csv += "kind,pipeline_size,stages_per_device,micro_batches,segments,seq_len,partition,status,"
         "makespan,bubble_ratio,peak_memory,throughput\n";
  for (const std::string& kname : kinds) {
    const ScheduleKind kind = parse_schedule_kind(kname);
    for (auto P : Ps)
      for (auto nv : NVs)
        for (auto M : Ms)
          for (auto k : Ks)
            for (auto T : Ts) {
              ScenarioConfig cfg = base;
              cfg.pipeline_size = static_cast<int>(P);
              cfg.stages_per_device = static_cast<int>(nv);
              cfg.micro_batches = static_cast<int>(M);
              cfg.segments = static_cast<int>(k);
              cfg.seq_len = T;
              csv += std::string(schedule_kind_name(kind)) + ',' + std::to_string(P) + ',' + std::to_string(nv) + ',' +
                     std::to_string(M) + ',' + std::to_string(k) + ',' + std::to_string(T) + ',' +
                     partition_mode_name(mode) + ',';
              try {
                cfg.validate();
                const SequencePartition part = partition_for(cfg, mode);
                const SimReport r = simulate(generate(cfg, kind, part), part);
                csv += "ok," + format_decimal(r.makespan, 6) + ',' + format_decimal(r.aggregate_bubble_ratio, 6) +
                       ',' + format_decimal(r.max_peak_memory, 6) + ',' + format_decimal(r.modeled_throughput, 6) +
                       '\n';
              } catch (const std::invalid_argument& e) {  // includes UnsupportedScheduleError
                csv += "skip:" + safe(e.what()) + ",,,,\n";
              } catch (const std::domain_error& e) {
                csv += "skip:" + safe(e.what()) + ",,,,\n";
              }
            }
  }
  emit(o.str("--out"), csv);
  return kOk;
}

// ---------------------------------------------------------------- partition

int cmd_partition(const std::vector<std::string>& args) {
  Options o("partition", with_config({{"--segments", "-k", false, false, "segment count override"},
                                      {"--mode", "", false, false, "partitioner", {"even", "cwp", "oracle"}},
                                      {"--json", "", true, false, "emit JSON instead of a table"}}));
  o.parse(args);
  ScenarioConfig cfg = resolve_config(o);
  const long long k = o.integer("--segments", 0);
  if (k > 0) cfg.segments = static_cast<int>(k);
  cfg.validate();
  const SequencePartition part = partition_for(cfg, parse_partition_mode(o.str("--mode", "cwp")));
  const BalanceReport bal = balance_report(part, cfg);
  std::string out;
  if (o.flag("--json")) {
    out = "{\n  \"lengths\": [";
    for (std::size_t i = 0; i < part.lengths.size(); ++i) out += (i ? ", " : "") + std::to_string(part.lengths[i]);
    out += "],\n  \"imbalance\": \"" + part.imbalance.str() + "\",\n  \"segment_costs\": [";
    for (std::size_t i = 0; i < bal.segment_costs.size(); ++i)
      out += std::string(i ? ", " : "") + '"' + bal.segment_costs[i].str() + '"';
    out += "]\n}\n";
  } else {
    out = "segment  tokens  forward_cost\n";
    for (std::size_t i = 0; i < part.lengths.size(); ++i)
      out += std::to_string(i + 1) + "  " + std::to_string(part.lengths[i]) + "  " + bal.segment_costs[i].str() + '\n';
    out += "imbalance = " + part.imbalance.str() + " (" + format_decimal(part.imbalance, 6) + ")\n";
  }
  std::cout << out;
  return kOk;
}

// ---------------------------------------------------------------- validate

int cmd_validate(const std::vector<std::string>& args) {
  Options o("validate", {}, {"schedule"});
  o.parse(args);
  std::ifstream f(o.positional(0), std::ios::binary);
  if (!f) throw std::runtime_error("cannot open '" + o.positional(0) + "'");
  std::ostringstream text;
  text << f.rdbuf();
  const auto v = check_schedule(schedule_from_json(text.str()));
  if (!v.empty()) throw ValidationFailure(violations_to_string(v));
  std::cout << "ok\n";
  return kOk;
}

// ---------------------------------------------------------------- execute (B200)

void sp_ok(int code) {
  if (code != SP_OK) throw std::runtime_error(sp_last_error());
}

std::string engine_text(const std::function<int(char*, size_t*)>& fn) {
  size_t n = 0;
  sp_ok(fn(nullptr, &n));
  std::string buf(n, '\0');
  sp_ok(fn(buf.data(), &n));
  buf.resize(n ? n - 1 : 0);
  return buf;
}

std::uint64_t splitmix64(std::uint64_t& s) {
  std::uint64_t z = (s += 0x9E3779B97F4A7C15ull);
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

int cmd_execute(const std::vector<std::string>& args) {
  Options o("execute", with_config({{"--kind", "", false, false, "schedule kind", {"gpipe", "1f1b", "1f1b-i", "seq1f1b", "seq1f1b-i", "zb1p", "seqzb1p"}, true},
                                    {"--partition", "", false, false, "sequence partitioner", {"even", "cwp"}},
                                    {"--family", "", false, false, "model family (default gpt)", {"gpt", "llama"}},
                                    {"--heads", "", false, false, "attention heads (default hidden/80 for gpt, /128 llama)"},
                                    {"--ffn", "", false, false, "FFN width (default 4h gpt, 8h/3 rounded to 256 llama)"},
                                    {"--vocab", "", false, false, "vocabulary (default 50257 gpt, 32000 llama)"},
                                    {"--dtype", "", false, false, "bf16 production (default) | f32 validation mode", {"bf16", "f32"}},
                                    {"--steps", "", false, false, "steps to run; the last one is reported (default 2)"},
                                    {"--device", "", false, false, "CUDA device (default 0)"},
                                    {"--seed", "", false, false, "token seed (default 1234)"},
                                    {"--out", "", false, false, "measured report JSON path ('-' = stdout)"},
                                    {"--gantt", "", false, false, "render the measured timeline", {"ascii", "svg"}},
                                    {"--gantt-out", "", false, false, "timeline path ('-' = stdout)"},
                                    {"--gantt-width", "", false, false, "ascii timeline width in columns"},
                                    {"--memory-downsample", "", false, false, "keep every n-th memory point"},
                                    {"--summary", "", true, false, "print a one-line summary to stderr"}}));
  o.parse(args);
  if (!o.has("--kind")) throw UsageError("--kind is required\n" + o.usage());
  const ScenarioConfig cfg = resolve_config(o);
  const SequencePartition part = partition_for(cfg, parse_partition_mode(o.str("--partition", "even")));
  const ScheduleKind kind = parse_schedule_kind(o.str("--kind"));
  generate(cfg, kind, part);  // feasibility / UnsupportedScheduleError before any device work

  const std::string fam = o.str("--family", "gpt");
  const bool llama = fam == "llama";
  const std::string dt = o.str("--dtype", "bf16");
  sp_model m{};
  m.family = llama ? SP_MODEL_LLAMA : SP_MODEL_GPT;
  m.dtype = dt == "bf16" ? SP_DTYPE_BF16 : SP_DTYPE_F32;
  m.hidden = static_cast<int32_t>(cfg.hidden_dim);
  m.layers = cfg.layers;
  m.heads = static_cast<int32_t>(o.integer("--heads", llama ? m.hidden / 128 : m.hidden / 80));
  if (m.heads <= 0 || m.hidden % m.heads) throw UsageError("--heads must divide hidden_dim");
  m.head_dim = m.hidden / m.heads;
  m.ffn = static_cast<int32_t>(o.integer("--ffn", llama ? (8 * m.hidden / 3 + 255) / 256 * 256 : 4 * m.hidden));
  m.vocab = static_cast<int32_t>(o.integer("--vocab", llama ? 32000 : 50257));
  m.max_seq = cfg.seq_len;
  m.seed = 42;
  m.init_std = 0.02f;
  m.norm_eps = 1e-5f;
  m.rope_theta = 10000.f;
  m.lr = 1e-4f;
  m.beta1 = 0.9f;
  m.beta2 = 0.95f;
  m.adam_eps = 1e-8f;
  m.weight_decay = 0.1f;
  m.flags = SP_FLAG_TIMELINE;

  sp_scenario c{};
  spc::to_c(cfg, &c);  // the C-ABI's own conversion (csrc/capi)
  std::vector<int64_t> lengths(part.lengths.begin(), part.lengths.end());
  sp_engine* eng = nullptr;
  sp_ok(sp_engine_create(&c, static_cast<int32_t>(kind), lengths.data(), &m, 0, 1,
                         static_cast<int32_t>(o.integer("--device", 0)), &eng));
  struct Guard {
    sp_engine* e;
    ~Guard() { sp_engine_destroy(e); }
  } guard{eng};

  // Synthetic tokens: uniform in [0, vocab), splitmix64 counter stream.
  std::uint64_t state = static_cast<std::uint64_t>(o.integer("--seed", 1234));
  std::vector<int32_t> tokens(static_cast<std::size_t>(cfg.micro_batches) * static_cast<std::size_t>(cfg.seq_len + 1));
  for (int32_t& t : tokens) t = static_cast<int32_t>(splitmix64(state) % static_cast<std::uint64_t>(m.vocab));
  sp_step_report rep{};
  const long long steps = o.integer("--steps", 2);
  if (steps < 1) throw UsageError("--steps must be >= 1");
  for (long long s = 0; s < steps; ++s) sp_ok(sp_engine_step(eng, tokens.data(), 0, &rep));

  const int64_t ds = o.integer("--memory-downsample", 0);
  emit(o.str("--out"), engine_text([&](char* b, size_t* n) { return sp_engine_report_json(eng, 2, ds, b, n); }));
  if (o.has("--gantt")) {
    const int32_t fmt = o.str("--gantt") == "svg" ? SP_RENDER_SVG : SP_RENDER_ASCII;
    const int32_t w = static_cast<int32_t>(o.integer("--gantt-width", 120));
    emit(o.str("--gantt-out"), engine_text([&](char* b, size_t* n) { return sp_engine_render_gantt(eng, fmt, w, b, n); }));
  }
  if (o.flag("--summary")) {
    const double tokens_per_s = static_cast<double>(cfg.micro_batches) * static_cast<double>(cfg.seq_len) / (rep.step_ms * 1e-3);
    std::cerr << "step_ms=" << rep.step_ms << " tokens_per_s=" << tokens_per_s << " loss=" << rep.loss
              << " bubble_ratio=" << rep.bubble_ratio << " peak_activation_gb=" << rep.peak_activation_bytes / 1e9
              << " ops=" << rep.ops_executed << "\n";
  }
  return kOk;
}

const std::map<std::string, std::function<int(const std::vector<std::string>&)>>& commands() {
  static const std::map<std::string, std::function<int(const std::vector<std::string>&)>> m{
      {"simulate", cmd_simulate}, {"sweep", cmd_sweep},     {"partition", cmd_partition},
      {"validate", cmd_validate}, {"execute", cmd_execute}};
  return m;
}

std::string top_usage() {
  return "seqpipe_b200: generate, simulate, validate, sweep and EXECUTE (on a B200) pipeline-parallel schedules\n"
         "Usage: seqpipe_b200 SUBCOMMAND [OPTIONS]\n"
         "Subcommands: simulate, sweep, partition, validate, execute (--help for each)\n";
}

}  // namespace

int main(int argc, char** argv) {
  const std::vector<std::string> all(argv + 1, argv + argc);
  if (all.empty()) {
    std::cerr << top_usage() << "A subcommand is required\n";
    return kUsage;
  }
  if (all[0] == "--help" || all[0] == "-h") {
    std::cout << top_usage();
    return kOk;
  }
  const auto it = commands().find(all[0]);
  if (it == commands().end()) {
    std::cerr << top_usage() << "The following argument was not expected: " << all[0] << "\n";
    return kUsage;
  }
  try {
    return it->second(std::vector<std::string>(all.begin() + 1, all.end()));
  } catch (const UsageError& e) {
    const std::string w = e.what();
    const bool help = w.rfind("Usage:", 0) == 0;
    (help ? std::cout : std::cerr) << w << (w.empty() || w.back() == '\n' ? "" : "\n");
    return help ? kOk : kUsage;
  } catch (const ValidationFailure& e) {
    std::cerr << e.what();
    return kValidation;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << '\n';
    return kRuntime;
  }
}
