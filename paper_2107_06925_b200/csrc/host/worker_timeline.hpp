// Chimera-B200 host layer -- per-worker views of a timed schedule.
//
// dessim (eager-sync decision, idle), perfmodel (free regions, Eq. 1's hidden
// allreduce) and analysis (bubble, stash peaks) all ask the same few questions of
// one worker's spans: when did each held stage receive its last gradient, how much
// idle lies after an instant, where are the gaps.  They are answered here once, on
// a start-ordered copy of the worker's spans.
//
// Numerical contract: every sum below accumulates in start order and every
// maximum is strict-first, because the reference's timeline JSON / predicted
// times are compared byte-for-byte (proj/src/dessim.cpp:64-95,
// proj/src/perfmodel.cpp:137-160,214-260).
#pragma once

#include <algorithm>
#include <utility>
#include <vector>

#include "pipesim/core.hpp"

namespace pipesim::timeline {

// One worker's spans ordered by start time.  Equal starts can only come from
// zero-length tasks; every query below is independent of their relative order.
class Track {
 public:
  explicit Track(std::vector<TimeSpan> spans) : s_(std::move(spans)) {
    std::sort(s_.begin(), s_.end(), [](const TimeSpan& a, const TimeSpan& b) { return a.start < b.start; });
  }

  const std::vector<TimeSpan>& spans() const { return s_; }

  // Idle time strictly after `t` up to the worker's last busy instant: the spans
  // that still run after t are walked with a busy cursor starting at t.
  double idle_after(double t) const {
    double idle = 0, cur = t;
    for (const TimeSpan& x : s_) {
      if (x.end <= t) continue;
      if (x.start > cur) idle += x.start - cur;
      cur = std::max(cur, x.end);
    }
    return idle;
  }

  // Maximal idle intervals between the first start and the last end.
  std::vector<std::pair<double, double>> gaps() const {
    std::vector<std::pair<double, double>> g;
    if (s_.empty()) return g;
    double cur = s_.front().start;
    for (const TimeSpan& x : s_) {
      if (x.start > cur) g.emplace_back(cur, x.start);
      cur = std::max(cur, x.end);
    }
    return g;
  }

 private:
  std::vector<TimeSpan> s_;
};

// When each stage a worker holds received its final weight gradient: the latest
// end of its backwards and the index of the first backward reaching it.  `index`
// stays -1 (and `at` 0) for a stage whose backwards all end at time 0.  Ordered by
// stage id, which is the order the reference visits held stages in.
struct StageDone {
  int stage = 0;
  double at = 0;
  int index = -1;
};

inline std::vector<StageDone> stages_done(const std::vector<Task>& tasks, const std::vector<TimeSpan>& spans) {
  std::vector<StageDone> out;
  for (int i = 0; i < int(tasks.size()); ++i) {
    if (tasks[i].kind != TaskKind::Backward) continue;
    auto it = std::lower_bound(out.begin(), out.end(), tasks[i].stage,
                               [](const StageDone& d, int st) { return d.stage < st; });
    if (it == out.end() || it->stage != tasks[i].stage) it = out.insert(it, StageDone{tasks[i].stage, 0.0, -1});
    if (spans[i].end > it->at) {
      it->at = spans[i].end;
      it->index = i;
    }
  }
  return out;
}

inline double busy_time(const std::vector<TimeSpan>& spans) {
  double b = 0;
  for (const TimeSpan& x : spans) b += x.end - x.start;
  return b;
}

inline double last_end(const std::vector<TimeSpan>& spans) {
  double e = 0;
  for (const TimeSpan& x : spans) e = std::max(e, x.end);
  return e;
}

}  // namespace pipesim::timeline
