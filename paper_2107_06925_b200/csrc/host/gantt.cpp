// Gantt rendering (pipesim::gantt, reference proj/src/gantt.cpp:35-125) and the
// `pipesim simulate -o` timeline document (reference proj/tools/main.cpp:134-170),
// plus its inverse so measured GPU timelines in that schema can be rendered.
//
// Output is byte-identical to the reference: numbers in the SVG use the iostream
// default float layout (6 significant digits, %g), the timeline JSON the nlohmann
// ordered_json dump of chimera::json.
#include "pipesim/gantt.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <string>

#include "json_io.hpp"
#include "timeline.hpp"

namespace pipesim::gantt {

namespace {

// iostream default formatting of a double (precision 6, %g)
std::string g6(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%g", v);
  return buf;
}

const char* pipeline_color(int p) {
  static const char* kColors[8] = {"#4e79a7", "#f28e2b", "#59a14f", "#e15759",
                                   "#b07aa1", "#76b7b2", "#edc948", "#ff9da7"};
  return kColors[((p % 8) + 8) % 8];
}

}  // namespace

std::string render_svg(const dessim::SimResult& r, const CostProfile& profile) {
  const Schedule& s = r.timed;
  if (!s.timed()) throw UntimedScheduleError("svg rendering requires a timed schedule");
  const int nw = int(s.per_worker.size());
  const double scale = std::max(4.0, 640.0 / std::max(1.0, r.makespan));  // px per time unit
  constexpr int kRow = 26, kGap = 6, kLeft = 46, kTop = 26;
  const int width = kLeft + int(r.makespan * scale) + 20;
  const int height = kTop + nw * (kRow + kGap) + 30;
  std::string o;
  o += "<svg xmlns=\"http://www.w3.org/2000/svg\" width=\"" + std::to_string(width) + "\" height=\"" +
       std::to_string(height) + "\" font-family=\"monospace\" font-size=\"11\">\n";
  o += "  <defs>\n"
       "    <pattern id=\"hatch\" width=\"5\" height=\"5\" patternTransform=\"rotate(45)\" "
       "patternUnits=\"userSpaceOnUse\">\n"
       "      <line x1=\"0\" y1=\"0\" x2=\"0\" y2=\"5\" stroke=\"#00000055\" stroke-width=\"2\"/>\n"
       "    </pattern>\n"
       "  </defs>\n";
  // grid lines + labels every max(1, floor(makespan / 16)) time units
  const double step = std::max(1.0, std::floor(r.makespan / 16.0));
  for (double t = 0; t <= r.makespan + 1e-9; t += step) {
    const double x = kLeft + t * scale;
    o += "  <line x1=\"" + g6(x) + "\" y1=\"" + std::to_string(kTop - 6) + "\" x2=\"" + g6(x) + "\" y2=\"" +
         std::to_string(height - 24) + "\" stroke=\"#dddddd\"/>\n";
    o += "  <text x=\"" + g6(x + 2) + "\" y=\"" + std::to_string(kTop - 10) + "\" fill=\"#666666\">" + g6(t) +
         "</text>\n";
  }
  for (int w = 0; w < nw; ++w) {
    const int y = kTop + w * (kRow + kGap);
    o += "  <text x=\"4\" y=\"" + std::to_string(y + kRow - 8) + "\">P" + std::to_string(w) + "</text>\n";
    for (size_t i = 0; i < s.per_worker[w].size(); ++i) {
      const Task& t = s.per_worker[w][i];
      const TimeSpan& sp = (*s.timing)[w][i];
      const double x = kLeft + sp.start * scale;
      const double len = std::max(1.0, (sp.end - sp.start) * scale - 0.5);
      const std::string box = "  <rect x=\"" + g6(x) + "\" y=\"" + std::to_string(y) + "\" width=\"" + g6(len) +
                              "\" height=\"" + std::to_string(kRow) + "\" fill=\"";
      o += box + pipeline_color(t.pipeline_id) + "\" stroke=\"#333333\" stroke-width=\"0.5\"/>\n";
      if (t.kind == TaskKind::Backward) o += box + "url(#hatch)\"/>\n";
      if (len > 11)
        o += "  <text x=\"" + g6(x + len / 2 - 3) + "\" y=\"" + std::to_string(y + kRow - 8) +
             "\" fill=\"#ffffff\">" + std::to_string(t.micro_batch) + "</text>\n";
    }
  }
  for (const auto& e : r.allreduce_events) {
    const int y = kTop + e.worker * (kRow + kGap) + kRow - 5;
    const double x = kLeft + e.start * scale;
    const double len = std::max(1.0, (e.end - e.start) * scale);
    o += "  <rect x=\"" + g6(x) + "\" y=\"" + std::to_string(y) + "\" width=\"" + g6(len) +
         "\" height=\"5\" fill=\"none\" stroke=\"" + (e.eager ? "#d62728" : "#555555") +
         "\" stroke-width=\"1\"/>\n";
  }
  o += "  <text x=\"4\" y=\"" + std::to_string(height - 8) + "\" fill=\"#666666\">makespan " + g6(r.makespan) +
       " (F_t=" + g6(profile.F_t) + ")</text>\n";
  o += "</svg>\n";
  return o;
}

std::string render_ascii(const dessim::SimResult& r, const CostProfile& profile) {
  const Schedule& s = r.timed;
  if (!s.timed()) throw UntimedScheduleError("ascii rendering requires a timed schedule");
  const double u = profile.F_t;
  const int cols = int(std::llround(r.compute_makespan / u));
  std::string o;
  for (int w = 0; w < int(s.per_worker.size()); ++w) {
    std::string line(size_t(std::max(cols, 1)), '.');
    for (size_t i = 0; i < s.per_worker[w].size(); ++i) {
      const Task& t = s.per_worker[w][i];
      const TimeSpan& sp = (*s.timing)[w][i];
      const int a = int(std::llround(sp.start / u));
      const int b = std::max(a + 1, int(std::llround(sp.end / u)));
      const char c = t.kind == TaskKind::Backward ? char('A' + t.micro_batch % 26) : char('0' + t.micro_batch % 10);
      for (int k = a; k < b && k < cols; ++k) line[size_t(k)] = c;
    }
    o += "P" + std::to_string(w) + (w < 10 ? " " : "") + "|" + line + "|\n";
  }
  return o;
}

}  // namespace pipesim::gantt

namespace chimera::timeline {

using chimera::json::Value;
using namespace pipesim;

std::string to_json(const dessim::SimResult& r, dessim::SyncPolicy policy, int indent) {
  Value j = Value::object();
  j.set("policy", Value::string(dessim::to_string(policy)));
  j.set("makespan", Value::number(r.makespan));
  j.set("compute_makespan", Value::number(r.compute_makespan));
  j.set("allreduce_exposed", Value::number(r.allreduce_exposed));
  Value idle = Value::array();
  for (double x : r.per_worker_idle) idle.push(Value::number(x));
  j.set("per_worker_idle", std::move(idle));
  Value ev = Value::array();
  const Schedule& s = r.timed;
  if (!s.timed()) throw UntimedScheduleError("timeline requires a timed schedule");
  for (size_t w = 0; w < s.per_worker.size(); ++w)
    for (size_t i = 0; i < s.per_worker[w].size(); ++i) {
      const Task& t = s.per_worker[w][i];
      const TimeSpan& sp = (*s.timing)[w][i];
      Value e = Value::object();
      e.set("worker", Value::integer(t.worker));
      e.set("kind", Value::string(pipesim::to_string(t.kind)));
      e.set("pipeline_id", Value::integer(t.pipeline_id));
      e.set("micro_batch", Value::integer(t.micro_batch));
      e.set("stage", Value::integer(t.stage));
      e.set("start", Value::number(sp.start));
      e.set("end", Value::number(sp.end));
      ev.push(std::move(e));
    }
  j.set("events", std::move(ev));
  Value ar = Value::array();
  for (const auto& a : r.allreduce_events) {
    Value e = Value::object();
    e.set("worker", Value::integer(a.worker));
    e.set("stage", Value::integer(a.stage));
    e.set("eager", Value::boolean(a.eager));
    e.set("start", Value::number(a.start));
    e.set("end", Value::number(a.end));
    ar.push(std::move(e));
  }
  j.set("allreduce", std::move(ar));
  return chimera::json::dump(j, indent);
}

dessim::SimResult from_json(const std::string& text) {
  const Value j = chimera::json::parse(text);
  dessim::SimResult r;
  r.makespan = j.at("makespan").as_double();
  r.compute_makespan = j.at("compute_makespan").as_double();
  r.allreduce_exposed = j.has("allreduce_exposed") ? j.at("allreduce_exposed").as_double() : 0.0;
  int nw = 0;
  if (j.has("per_worker_idle")) {
    for (const Value& x : j.at("per_worker_idle").arr) r.per_worker_idle.push_back(x.as_double());
    nw = int(r.per_worker_idle.size());
  }
  const auto& evs = j.at("events").arr;
  for (const Value& e : evs) nw = std::max(nw, int(e.at("worker").as_int()) + 1);
  r.timed.per_worker.assign(size_t(nw), {});
  std::vector<std::vector<TimeSpan>> timing(static_cast<size_t>(nw));
  for (const Value& e : evs) {
    Task t;
    const auto kind = task_kind_from_string(e.at("kind").as_string());
    if (!kind) throw InvalidConfigError("timeline: unknown task kind " + e.at("kind").as_string());
    t.kind = *kind;
    t.worker = int(e.at("worker").as_int());
    if (t.worker < 0) throw InvalidConfigError("timeline: negative worker");
    t.pipeline_id = int(e.at("pipeline_id").as_int());
    t.micro_batch = int(e.at("micro_batch").as_int());
    t.stage = int(e.at("stage").as_int());
    r.timed.per_worker[size_t(t.worker)].push_back(t);
    timing[size_t(t.worker)].push_back(TimeSpan{e.at("start").as_double(), e.at("end").as_double()});
  }
  r.timed.timing = std::move(timing);
  if (j.has("allreduce"))
    for (const Value& e : j.at("allreduce").arr) {
      dessim::AllReduceEvent a;
      a.worker = int(e.at("worker").as_int());
      a.stage = int(e.at("stage").as_int());
      a.eager = e.at("eager").as_bool();
      a.start = e.at("start").as_double();
      a.end = e.at("end").as_double();
      r.allreduce_events.push_back(a);
    }
  return r;
}

}  // namespace chimera::timeline
