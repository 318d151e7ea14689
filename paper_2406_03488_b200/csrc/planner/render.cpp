// Timeline renderers (reference behaviour: core/src/render.cpp:46-124).
//
// Geometry is computed in double from Rational::to_double, exactly as the
// reference does, so the cell / pixel positions and the "%.2f" coordinates
// agree byte for byte.
#include "seqpipe/render.hpp"

#include <algorithm>
#include <array>
#include <cstdio>
#include <string>

namespace seqpipe {
namespace {

struct KindStyle {
  TaskKind kind;
  char glyph;
  const char* colour;
  const char* legend_name;
};

// Fixed kind table: glyphs render.cpp:20-28, colours :30-38, legend order :94-95.
constexpr std::array<KindStyle, 4> kStyles{{
    {TaskKind::kForward, 'F', "#4e79a7", "forward"},
    {TaskKind::kFusedBackward, 'B', "#f28e2b", "fused backward"},
    {TaskKind::kInputGrad, 'I', "#e15759", "input-grad"},
    {TaskKind::kWeightGrad, 'W', "#76b7b2", "weight-grad"},
}};

const KindStyle& style(TaskKind k) {
  for (const KindStyle& s : kStyles)
    if (s.kind == k) return s;
  static const KindStyle unknown{TaskKind::kForward, '?', "#000000", "?"};
  return unknown;
}

std::string label_of(const Task& t) { return std::to_string(t.micro_batch) + "." + std::to_string(t.segment); }

std::string two_dp(double v) {
  char b[64];
  std::snprintf(b, sizeof b, "%.2f", v);
  return b;
}

// Minimal appender: out << a << b ... without iostreams.
struct Out {
  std::string s;
  Out& operator<<(const std::string& x) { s += x; return *this; }
  Out& operator<<(const char* x) { s += x; return *this; }
  Out& operator<<(char x) { s += x; return *this; }
  Out& operator<<(int x) { s += std::to_string(x); return *this; }
  Out& operator<<(long x) { s += std::to_string(x); return *this; }
  Out& operator<<(long long x) { s += std::to_string(x); return *this; }
  Out& operator<<(std::size_t x) { s += std::to_string(x); return *this; }
};

}  // namespace

std::string render_ascii_gantt(const SimReport& report, int width) {
  const int W = std::max(width, 10);
  Out out;
  out << "kind=" << schedule_kind_name(report.kind) << " makespan=" << report.makespan.str()
      << "  [F forward, B backward, I input-grad, W weight-grad, . idle]\n";
  const double span = report.makespan.to_double();
  auto cell = [&](const Rational& t) { return span <= 0.0 ? 0 : static_cast<int>(t.to_double() / span * W); };
  for (std::size_t d = 0; d < report.task_times.size(); ++d) {
    std::string row(static_cast<std::size_t>(W), '.');
    for (const TaskTiming& tt : report.task_times[d]) {
      const int a = std::clamp(cell(tt.start), 0, W - 1);
      const int b = std::clamp(cell(tt.end), a + 1, W);
      std::fill(row.begin() + a, row.begin() + b, style(tt.task.kind).glyph);
      const std::string lab = label_of(tt.task);
      const int n = static_cast<int>(lab.size());
      if (b - a >= n + 2) row.replace(static_cast<std::size_t>(a + (b - a - n) / 2), lab.size(), lab);
    }
    out << "device " << (d + 1) << " |" << row << "|\n";
  }
  return out.s;
}

std::string render_svg_gantt(const SimReport& report) {
  constexpr int kRowH = 26, kGap = 6, kLeft = 70, kTop = 40, kChartW = 1200;
  const int ndev = static_cast<int>(report.task_times.size());
  const double span = report.makespan.to_double();
  const double px_per_unit = span > 0.0 ? kChartW / span : 0.0;
  const char* kind = schedule_kind_name(report.kind);

  Out out;
  out << "<?xml version=\"1.0\" encoding=\"UTF-8\"?>\n<!-- timeline for " << kind << "; colors:";
  for (std::size_t i = 0; i < kStyles.size(); ++i)
    out << (i ? ", " : " ") << kStyles[i].legend_name << ' ' << kStyles[i].colour;
  out << " -->\n<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" << kLeft + kChartW + 20 << "\" height=\""
      << kTop + ndev * (kRowH + kGap) + 30 << "\" font-family=\"monospace\" font-size=\"11\">\n";
  out << "<text x=\"10\" y=\"18\">" << kind << " P=" << report.config.pipeline_size
      << " M=" << report.config.micro_batches << " k=" << report.config.segments
      << " makespan=" << report.makespan.str() << "</text>\n";
  for (std::size_t i = 0; i < kStyles.size(); ++i) {
    const int x = 10 + 40 * static_cast<int>(i);
    out << "<rect x=\"" << x << "\" y=\"24\" width=\"10\" height=\"10\" fill=\"" << kStyles[i].colour
        << "\"/>\n<text x=\"" << x + 14 << "\" y=\"33\">" << kStyles[i].glyph << "</text>\n";
  }
  for (int d = 0; d < ndev; ++d) {
    const int y = kTop + d * (kRowH + kGap);
    out << "<text x=\"10\" y=\"" << y + kRowH - 8 << "\">dev " << d + 1 << "</text>\n"
        << "<rect x=\"" << kLeft << "\" y=\"" << y << "\" width=\"" << kChartW << "\" height=\"" << kRowH
        << "\" fill=\"#f0f0f0\"/>\n";
    for (const TaskTiming& tt : report.task_times[static_cast<std::size_t>(d)]) {
      const double x = kLeft + tt.start.to_double() * px_per_unit;
      const double w = (tt.end.to_double() - tt.start.to_double()) * px_per_unit;
      const char* fill = style(tt.task.kind).colour;
      out << "<rect x=\"" << two_dp(x) << "\" y=\"" << y << "\" width=\"" << two_dp(w) << "\" height=\"" << kRowH
          << "\" fill=\"" << fill << "\" stroke=\"#ffffff\" stroke-width=\"0.5\"/>\n";
      if (w >= 26.0)
        out << "<text x=\"" << two_dp(x + w / 2.0) << "\" y=\"" << y + kRowH - 8
            << "\" text-anchor=\"middle\" fill=\"#ffffff\">" << label_of(tt.task) << "</text>\n";
    }
  }
  out << "</svg>\n";
  return out.s;
}

}  // namespace seqpipe
