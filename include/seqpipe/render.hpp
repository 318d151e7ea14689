// Timeline rendering of a SimReport (modeled by simulate(), or measured by the
// engine with ns times): an ASCII Gantt chart and an SVG timeline.
// Mirrors core/include/seqpipe/render.hpp:15-21; output is byte-identical to
// core/src/render.cpp:46-124 for the same report (tests/test_render.py).
#pragma once

#include <string>

#include "seqpipe/sim.hpp"

namespace seqpipe {

// One row per device of `width` cells (>= 10): F / B / I / W per task kind,
// '.' idle, and an "m.s" label centred in spans at least label + 2 wide.
std::string render_ascii_gantt(const SimReport& report, int width = 120);

// SVG timeline: one row per device, x scaled to the makespan, a rect per task
// (colour by kind, legend drawn) and an "m.s" label when the rect is >= 26 px.
// Deterministic: identical reports give identical bytes.
std::string render_svg_gantt(const SimReport& report);

}  // namespace seqpipe
