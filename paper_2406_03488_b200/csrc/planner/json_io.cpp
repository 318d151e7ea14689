// seqpipe.schedule.v1 / seqpipe.simreport.v1 documents (reference
// core/src/json_io.cpp:59-159) with a self-contained JSON value, writer and
// parser. The writer reproduces the reference's canonical form byte for byte:
// object keys in lexicographic order, `indent` spaces per nesting level,
// `"key": value`, empty containers as `{}` / `[]`, integers in decimal,
// rationals as their exact `n` or `n/d` strings, and a trailing newline.
#include "seqpipe/json_io.hpp"

#include <algorithm>
#include <cstdint>
#include <map>
#include <memory>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace seqpipe {
namespace {

struct JValue {
  enum class Type { kNull, kBool, kInt, kString, kArray, kObject } type = Type::kNull;
  bool b = false;
  std::int64_t i = 0;
  std::string s;
  std::vector<JValue> arr;
  std::map<std::string, JValue> obj;  // sorted keys: the canonical order

  static JValue Int(std::int64_t v) {
    JValue j;
    j.type = Type::kInt;
    j.i = v;
    return j;
  }
  static JValue Str(std::string v) {
    JValue j;
    j.type = Type::kString;
    j.s = std::move(v);
    return j;
  }
  static JValue Arr() {
    JValue j;
    j.type = Type::kArray;
    return j;
  }
  static JValue Obj() {
    JValue j;
    j.type = Type::kObject;
    return j;
  }
  JValue& operator[](const std::string& k) { return obj[k]; }
  void push(JValue v) { arr.push_back(std::move(v)); }

  const JValue& at(const std::string& k) const {
    if (type != Type::kObject) throw std::invalid_argument("json: not an object (key '" + k + "')");
    auto it = obj.find(k);
    if (it == obj.end()) throw std::invalid_argument("json: missing key '" + k + "'");
    return it->second;
  }
  const JValue& at(std::size_t idx) const {
    if (type != Type::kArray || idx >= arr.size()) throw std::invalid_argument("json: array index out of range");
    return arr[idx];
  }
  std::int64_t as_int() const {
    if (type != Type::kInt) throw std::invalid_argument("json: expected an integer");
    return i;
  }
  const std::string& as_str() const {
    if (type != Type::kString) throw std::invalid_argument("json: expected a string");
    return s;
  }
  const std::vector<JValue>& as_arr() const {
    if (type != Type::kArray) throw std::invalid_argument("json: expected an array");
    return arr;
  }
};

void put_string(std::string& out, const std::string& s) {
  out += '"';
  static const char* hex = "0123456789abcdef";
  for (unsigned char c : s) {
    switch (c) {
      case '"': out += "\\\""; break;
      case '\\': out += "\\\\"; break;
      case '\b': out += "\\b"; break;
      case '\f': out += "\\f"; break;
      case '\n': out += "\\n"; break;
      case '\r': out += "\\r"; break;
      case '\t': out += "\\t"; break;
      default:
        if (c < 0x20) {
          out += "\\u00";
          out += hex[c >> 4];
          out += hex[c & 15];
        } else {
          out += static_cast<char>(c);
        }
    }
  }
  out += '"';
}

void dump(const JValue& v, std::string& out, int indent, int level) {
  switch (v.type) {
    case JValue::Type::kNull: out += "null"; return;
    case JValue::Type::kBool: out += v.b ? "true" : "false"; return;
    case JValue::Type::kInt: out += std::to_string(v.i); return;
    case JValue::Type::kString: put_string(out, v.s); return;
    case JValue::Type::kArray: {
      if (v.arr.empty()) {
        out += "[]";
        return;
      }
      // The nlohmann/json header the reference is built with here (the copy shipped in
      // the image's cudnn_frontend wheel, json_io.cpp:6) prints an array whose
      // elements are all integers on one line without spaces: `[16,16]`. Matched
      // so that documents are byte-identical with the compiled reference.
      const bool all_int = std::all_of(v.arr.begin(), v.arr.end(),
                                       [](const JValue& e) { return e.type == JValue::Type::kInt; });
      if (indent < 0 || all_int) {
        out += '[';
        for (std::size_t k = 0; k < v.arr.size(); ++k) {
          if (k) out += ',';
          dump(v.arr[k], out, indent, level + 1);
        }
        out += ']';
        return;
      }
      out += "[\n";
      const std::string pad(static_cast<std::size_t>(indent * (level + 1)), ' ');
      for (std::size_t k = 0; k < v.arr.size(); ++k) {
        out += pad;
        dump(v.arr[k], out, indent, level + 1);
        out += k + 1 < v.arr.size() ? ",\n" : "\n";
      }
      out += std::string(static_cast<std::size_t>(indent * level), ' ');
      out += ']';
      return;
    }
    case JValue::Type::kObject: {
      if (v.obj.empty()) {
        out += "{}";
        return;
      }
      if (indent < 0) {
        out += '{';
        bool first = true;
        for (const auto& [k, x] : v.obj) {
          if (!first) out += ',';
          first = false;
          put_string(out, k);
          out += ':';
          dump(x, out, indent, level + 1);
        }
        out += '}';
        return;
      }
      out += "{\n";
      const std::string pad(static_cast<std::size_t>(indent * (level + 1)), ' ');
      std::size_t k = 0;
      for (const auto& [key, x] : v.obj) {
        out += pad;
        put_string(out, key);
        out += ": ";
        dump(x, out, indent, level + 1);
        out += ++k < v.obj.size() ? ",\n" : "\n";
      }
      out += std::string(static_cast<std::size_t>(indent * level), ' ');
      out += '}';
      return;
    }
  }
}

std::string dump_doc(const JValue& v, int indent) {
  std::string out;
  dump(v, out, indent, 0);
  return out + "\n";
}

// ---------------------------------------------------------------- parser
class Parser {
 public:
  explicit Parser(const std::string& t) : t_(t) {}
  JValue parse() {
    JValue v = value();
    ws();
    if (p_ != t_.size()) fail("trailing characters");
    return v;
  }

 private:
  [[noreturn]] void fail(const char* what) const {
    throw std::invalid_argument(std::string("json parse error at offset ") + std::to_string(p_) + ": " + what);
  }
  void ws() {
    while (p_ < t_.size() && (t_[p_] == ' ' || t_[p_] == '\n' || t_[p_] == '\t' || t_[p_] == '\r')) ++p_;
  }
  bool eat(char c) {
    ws();
    if (p_ < t_.size() && t_[p_] == c) {
      ++p_;
      return true;
    }
    return false;
  }
  void expect(char c) {
    if (!eat(c)) fail("unexpected character");
  }
  JValue value() {
    ws();
    if (p_ >= t_.size()) fail("unexpected end");
    const char c = t_[p_];
    if (c == '{' || c == '[') {
      // Bounded nesting: schedule files come from users (`validate`), so deep
      // input must be an error, not a stack overflow.
      if (++depth_ > kMaxDepth) fail("nesting deeper than 256");
      JValue v = c == '{' ? object() : array();
      --depth_;
      return v;
    }
    if (c == '"') return JValue::Str(string());
    if (c == '-' || (c >= '0' && c <= '9')) return number();
    if (t_.compare(p_, 4, "true") == 0) {
      p_ += 4;
      JValue v;
      v.type = JValue::Type::kBool;
      v.b = true;
      return v;
    }
    if (t_.compare(p_, 5, "false") == 0) {
      p_ += 5;
      JValue v;
      v.type = JValue::Type::kBool;
      return v;
    }
    if (t_.compare(p_, 4, "null") == 0) {
      p_ += 4;
      return JValue{};
    }
    fail("unexpected token");
  }
  JValue object() {
    expect('{');
    JValue o = JValue::Obj();
    if (eat('}')) return o;
    do {
      ws();
      std::string k = string();
      expect(':');
      o.obj[k] = value();
    } while (eat(','));
    expect('}');
    return o;
  }
  JValue array() {
    expect('[');
    JValue a = JValue::Arr();
    if (eat(']')) return a;
    do a.arr.push_back(value());
    while (eat(','));
    expect(']');
    return a;
  }
  std::string string() {
    if (p_ >= t_.size() || t_[p_] != '"') fail("expected a string");
    ++p_;
    std::string out;
    while (true) {
      if (p_ >= t_.size()) fail("unterminated string");
      char c = t_[p_++];
      if (c == '"') break;
      if (c != '\\') {
        out += c;
        continue;
      }
      if (p_ >= t_.size()) fail("bad escape");
      c = t_[p_++];
      switch (c) {
        case '"': out += '"'; break;
        case '\\': out += '\\'; break;
        case '/': out += '/'; break;
        case 'b': out += '\b'; break;
        case 'f': out += '\f'; break;
        case 'n': out += '\n'; break;
        case 'r': out += '\r'; break;
        case 't': out += '\t'; break;
        case 'u': {
          unsigned cp = hex4();
          if (cp >= 0xD800 && cp < 0xDC00) {  // high surrogate: a low one must follow
            if (p_ + 2 > t_.size() || t_[p_] != '\\' || t_[p_ + 1] != 'u') fail("unpaired surrogate");
            p_ += 2;
            const unsigned lo = hex4();
            if (lo < 0xDC00 || lo >= 0xE000) fail("unpaired surrogate");
            cp = 0x10000 + ((cp - 0xD800) << 10) + (lo - 0xDC00);
          } else if (cp >= 0xDC00 && cp < 0xE000) {
            fail("unpaired surrogate");
          }
          if (cp < 0x80) {
            out += static_cast<char>(cp);
          } else if (cp < 0x800) {
            out += static_cast<char>(0xC0 | (cp >> 6));
            out += static_cast<char>(0x80 | (cp & 0x3F));
          } else if (cp < 0x10000) {
            out += static_cast<char>(0xE0 | (cp >> 12));
            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            out += static_cast<char>(0x80 | (cp & 0x3F));
          } else {
            out += static_cast<char>(0xF0 | (cp >> 18));
            out += static_cast<char>(0x80 | ((cp >> 12) & 0x3F));
            out += static_cast<char>(0x80 | ((cp >> 6) & 0x3F));
            out += static_cast<char>(0x80 | (cp & 0x3F));
          }
          break;
        }
        default: fail("bad escape");
      }
    }
    return out;
  }
  // Exactly four hex digits (stoul would accept a partial "\u12G4").
  unsigned hex4() {
    if (p_ + 4 > t_.size()) fail("bad \\u escape");
    unsigned v = 0;
    for (int i = 0; i < 4; ++i) {
      const char h = t_[p_++];
      v <<= 4;
      if (h >= '0' && h <= '9') v |= static_cast<unsigned>(h - '0');
      else if (h >= 'a' && h <= 'f') v |= static_cast<unsigned>(h - 'a' + 10);
      else if (h >= 'A' && h <= 'F') v |= static_cast<unsigned>(h - 'A' + 10);
      else fail("bad \\u escape");
    }
    return v;
  }
  JValue number() {
    const std::size_t b = p_;
    if (t_[p_] == '-') ++p_;
    while (p_ < t_.size() && t_[p_] >= '0' && t_[p_] <= '9') ++p_;
    if (p_ < t_.size() && (t_[p_] == '.' || t_[p_] == 'e' || t_[p_] == 'E')) fail("only integers are used by seqpipe");
    if (p_ == b || (p_ == b + 1 && t_[b] == '-')) fail("bad number");
    return JValue::Int(std::stoll(t_.substr(b, p_ - b)));
  }
  static constexpr int kMaxDepth = 256;
  const std::string& t_;
  std::size_t p_ = 0;
  int depth_ = 0;
};

// ---------------------------------------------------------------- documents
JValue config_to_json(const ScenarioConfig& cfg) {
  JValue j = JValue::Obj();
  j["pipeline_size"] = JValue::Int(cfg.pipeline_size);
  j["stages_per_device"] = JValue::Int(cfg.stages_per_device);
  j["micro_batches"] = JValue::Int(cfg.micro_batches);
  j["segments"] = JValue::Int(cfg.segments);
  j["seq_len"] = JValue::Int(cfg.seq_len);
  j["layers"] = JValue::Int(cfg.layers);
  j["hidden_dim"] = JValue::Int(cfg.hidden_dim);
  j["param_count"] = JValue::Int(cfg.param_count);
  j["backward_ratio"] = JValue::Str(cfg.backward_ratio.str());
  JValue split = JValue::Arr();
  split.push(JValue::Str(cfg.bw_input_ratio.str()));
  split.push(JValue::Str(cfg.bw_weight_ratio.str()));
  j["bw_split_ratio"] = std::move(split);
  j["comm_latency"] = JValue::Str(cfg.comm_latency.str());
  j["activation_cost_per_token"] = JValue::Str(cfg.activation_cost_per_token.str());
  j["time_per_flop"] = JValue::Str(cfg.time_per_flop.str());
  j["cost_model"] = JValue::Str(cost_model_name(cfg.cost_model));
  j["uniform_forward"] = JValue::Str(cfg.uniform_forward.str());
  return j;
}

int to_i32(std::int64_t v) {
  if (v < INT32_MIN || v > INT32_MAX) throw std::invalid_argument("json: integer out of range");
  return static_cast<int>(v);
}

ScenarioConfig config_from_json(const JValue& j) {
  ScenarioConfig cfg;
  cfg.pipeline_size = to_i32(j.at("pipeline_size").as_int());
  cfg.stages_per_device = to_i32(j.at("stages_per_device").as_int());
  cfg.micro_batches = to_i32(j.at("micro_batches").as_int());
  cfg.segments = to_i32(j.at("segments").as_int());
  cfg.seq_len = j.at("seq_len").as_int();
  cfg.layers = to_i32(j.at("layers").as_int());
  cfg.hidden_dim = j.at("hidden_dim").as_int();
  cfg.param_count = j.at("param_count").as_int();
  cfg.backward_ratio = Rational::parse(j.at("backward_ratio").as_str());
  const JValue& split = j.at("bw_split_ratio");
  cfg.bw_input_ratio = Rational::parse(split.at(0).as_str());
  cfg.bw_weight_ratio = Rational::parse(split.at(1).as_str());
  cfg.comm_latency = Rational::parse(j.at("comm_latency").as_str());
  cfg.activation_cost_per_token = Rational::parse(j.at("activation_cost_per_token").as_str());
  cfg.time_per_flop = Rational::parse(j.at("time_per_flop").as_str());
  cfg.cost_model = parse_cost_model(j.at("cost_model").as_str());
  cfg.uniform_forward = Rational::parse(j.at("uniform_forward").as_str());
  return cfg;
}

JValue rational_pair(const Rational& a, const Rational& b) {
  JValue p = JValue::Arr();
  p.push(JValue::Str(a.str()));
  p.push(JValue::Str(b.str()));
  return p;
}

}  // namespace

std::string schedule_to_json(const Schedule& schedule, int indent) {
  JValue j = JValue::Obj();
  j["schema"] = JValue::Str("seqpipe.schedule.v1");
  j["kind"] = JValue::Str(schedule_kind_name(schedule.kind));
  j["config"] = config_to_json(schedule.config);
  JValue orders = JValue::Arr();
  for (const auto& order : schedule.device_orders) {
    JValue tasks = JValue::Arr();
    for (const Task& t : order) {
      JValue e = JValue::Arr();
      e.push(JValue::Str(task_kind_name(t.kind)));
      e.push(JValue::Int(t.micro_batch));
      e.push(JValue::Int(t.segment));
      e.push(JValue::Int(t.stage));
      tasks.push(std::move(e));
    }
    orders.push(std::move(tasks));
  }
  j["device_orders"] = std::move(orders);
  return dump_doc(j, indent);
}

Schedule schedule_from_json(const std::string& text) {
  const JValue j = Parser(text).parse();
  if (j.at("schema").as_str() != "seqpipe.schedule.v1") throw std::invalid_argument("unexpected schedule schema");
  Schedule schedule;
  schedule.kind = parse_schedule_kind(j.at("kind").as_str());
  schedule.config = config_from_json(j.at("config"));
  for (const JValue& order : j.at("device_orders").as_arr()) {
    std::vector<Task> tasks;
    tasks.reserve(order.as_arr().size());
    for (const JValue& e : order.as_arr()) {
      tasks.push_back(make_task(parse_task_kind(e.at(0).as_str()), to_i32(e.at(1).as_int()), to_i32(e.at(2).as_int()),
                                to_i32(e.at(3).as_int()), schedule.config.pipeline_size));
    }
    schedule.device_orders.push_back(std::move(tasks));
  }
  return schedule;
}

std::string report_to_json(const SimReport& report, int indent, std::size_t memory_downsample) {
  JValue j = JValue::Obj();
  j["schema"] = JValue::Str("seqpipe.simreport.v1");
  j["kind"] = JValue::Str(schedule_kind_name(report.kind));
  j["config"] = config_to_json(report.config);
  JValue part = JValue::Arr();
  for (std::int64_t n : report.partition_lengths) part.push(JValue::Int(n));
  j["partition"] = std::move(part);
  j["makespan"] = JValue::Str(report.makespan.str());
  j["modeled_throughput"] = JValue::Str(report.modeled_throughput.str());
  JValue agg = JValue::Obj();
  agg["bubble_ratio"] = JValue::Str(report.aggregate_bubble_ratio.str());
  agg["bubble_ratio_in_makespan"] = JValue::Str(report.aggregate_bubble_ratio_in_makespan.str());
  agg["max_peak_memory"] = JValue::Str(report.max_peak_memory.str());
  j["aggregate"] = std::move(agg);
  JValue devices = JValue::Arr();
  for (std::size_t d = 0; d < report.devices.size(); ++d) {
    const DeviceReport& dev = report.devices[d];
    JValue jd = JValue::Obj();
    jd["device"] = JValue::Int(dev.device);
    jd["first_start"] = JValue::Str(dev.first_start.str());
    jd["last_end"] = JValue::Str(dev.last_end.str());
    jd["busy"] = JValue::Str(dev.busy.str());
    jd["idle"] = JValue::Str(dev.idle.str());
    jd["bubble_ratio"] = JValue::Str(dev.bubble_ratio.str());
    jd["idle_in_makespan"] = JValue::Str(dev.idle_in_makespan.str());
    jd["bubble_ratio_in_makespan"] = JValue::Str(dev.bubble_ratio_in_makespan.str());
    jd["peak_memory"] = JValue::Str(dev.peak_memory.str());
    jd["peak_allocations"] = JValue::Int(dev.peak_allocations);
    jd["warmup_forward_tasks"] = JValue::Int(dev.warmup_forward_tasks);
    JValue series = JValue::Arr();
    const auto& pts = dev.memory_series;
    std::size_t stride = 1;
    if (memory_downsample > 0 && pts.size() > memory_downsample)
      stride = (pts.size() + memory_downsample - 1) / memory_downsample;
    for (std::size_t i = 0; i < pts.size(); i += stride) series.push(rational_pair(pts[i].first, pts[i].second));
    if (!pts.empty() && stride > 1 && (pts.size() - 1) % stride != 0)
      series.push(rational_pair(pts.back().first, pts.back().second));
    jd["memory_series"] = std::move(series);
    JValue tasks = JValue::Arr();
    if (d < report.task_times.size()) {
      for (const TaskTiming& t : report.task_times[d]) {
        JValue jt = JValue::Obj();
        jt["kind"] = JValue::Str(task_kind_name(t.task.kind));
        jt["m"] = JValue::Int(t.task.micro_batch);
        jt["s"] = JValue::Int(t.task.segment);
        jt["stage"] = JValue::Int(t.task.stage);
        jt["start"] = JValue::Str(t.start.str());
        jt["end"] = JValue::Str(t.end.str());
        tasks.push(std::move(jt));
      }
    }
    jd["tasks"] = std::move(tasks);
    devices.push(std::move(jd));
  }
  j["devices"] = std::move(devices);
  return dump_doc(j, indent);
}

}  // namespace seqpipe
