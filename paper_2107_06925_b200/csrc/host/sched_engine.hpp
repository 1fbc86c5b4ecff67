// Chimera-B200 host layer -- the list-scheduling engine shared by schedgen
// (order settling), analysis (exact tick timing), dessim (timing model) and the
// GPU executor (replay order and eager-sync decision).
//
// Semantics follow proj/src/listsched.hpp:52-197 exactly, because the settled
// Chimera order (and therefore bit-exact schedule parity) depends on them:
//   * data edges F(p,m,s-1)->F(p,m,s), B(p,m,s+1)->B(p,m,s), stash edge
//     F(p,m,s)->B(p,m,s) (cost 0); edge costs only across workers;
//   * a missing predecessor does not constrain; a pending one blocks;
//   * relaxed mode: the first not-yet-run Forward behind the worker's head may
//     overtake queued Backwards; nothing else reorders;
//   * ties (1e-12) go to the earlier candidate: head first, lower worker first.
// Implementation differs: tasks live in flat arrays, predecessors are resolved
// once up front through a hash index, and the per-step scan touches only each
// worker's head window.
#pragma once

#include <array>
#include <cmath>
#include <cstdint>
#include <limits>
#include <map>
#include <unordered_map>
#include <utility>
#include <vector>

#include "pipesim/core.hpp"

namespace pipesim::engine {

struct Params {
  double f_dur = 1.0;
  double b_dur = 2.0;
  double p2p_fwd = 0.0;
  double p2p_bwd = 0.0;
  bool relaxed = false;
  // extra busy time after task (worker, index) completes (eager-sync epsilon)
  const std::map<std::pair<int, int>, double>* post_delays = nullptr;
};

struct Timeline {
  std::vector<std::vector<TimeSpan>> spans;  // index-aligned with per_worker
  double makespan = 0;
};

inline std::uint64_t task_key(bool backward, int pipeline, int micro, int stage) {
  return (std::uint64_t(backward) << 63) | (std::uint64_t(std::uint32_t(pipeline) & 0x7FFF) << 48) |
         (std::uint64_t(std::uint32_t(micro) & 0xFFFFFF) << 24) |
         std::uint64_t(std::uint32_t(stage) & 0xFFFFFF);
}

// (worker, index) of every Forward/Backward; the first occurrence of a key wins.
inline std::unordered_map<std::uint64_t, std::pair<int, int>> index_tasks(const Schedule& s) {
  std::unordered_map<std::uint64_t, std::pair<int, int>> where;
  for (int w = 0; w < int(s.per_worker.size()); ++w)
    for (int i = 0; i < int(s.per_worker[w].size()); ++i) {
      const Task& t = s.per_worker[w][i];
      if (t.kind != TaskKind::Forward && t.kind != TaskKind::Backward) continue;
      where.emplace(task_key(t.kind == TaskKind::Backward, t.pipeline_id, t.micro_batch, t.stage),
                    std::make_pair(w, i));
    }
  return where;
}

inline Timeline list_schedule(const Schedule& s, const Params& prm) {
  constexpr double kInf = std::numeric_limits<double>::infinity();
  constexpr double kEps = 1e-12;
  const int nw = int(s.per_worker.size());

  // Flatten: task id = base[w] + i.
  std::vector<int> base(nw + 1, 0);
  for (int w = 0; w < nw; ++w) base[w + 1] = base[w] + int(s.per_worker[w].size());
  const int total = base[nw];
  std::vector<int> owner(total);
  for (int w = 0; w < nw; ++w)
    for (int t = base[w]; t < base[w + 1]; ++t) owner[t] = w;

  // Resolved predecessor edges: up to two per task {task id, cost if cross-worker}.
  struct Edge {
    int pred = -1;
    double cost = 0;
  };
  std::vector<std::array<Edge, 2>> preds(total);
  {
    const auto where = index_tasks(s);
    auto resolve = [&](int me, std::uint64_t key, double cost) -> Edge {
      auto it = where.find(key);
      if (it == where.end()) return {};
      const int id = base[it->second.first] + it->second.second;
      if (id == me) return {};
      return {id, cost};
    };
    for (int w = 0; w < nw; ++w)
      for (int i = 0; i < int(s.per_worker[w].size()); ++i) {
        const Task& t = s.per_worker[w][i];
        const int me = base[w] + i;
        if (t.kind == TaskKind::Forward && t.stage > 0) {
          preds[me][0] = resolve(me, task_key(false, t.pipeline_id, t.micro_batch, t.stage - 1),
                                 prm.p2p_fwd);
        } else if (t.kind == TaskKind::Backward) {
          preds[me][0] = resolve(me, task_key(true, t.pipeline_id, t.micro_batch, t.stage + 1),
                                 prm.p2p_bwd);
          preds[me][1] = resolve(me, task_key(false, t.pipeline_id, t.micro_batch, t.stage), 0.0);
        }
      }
  }

  Timeline out;
  out.spans.resize(nw);
  for (int w = 0; w < nw; ++w) out.spans[w].assign(s.per_worker[w].size(), TimeSpan{-1, -1});
  std::vector<char> done(total, 0);
  std::vector<double> end_of(total, 0.0), free_at(nw, 0.0);
  std::vector<int> head(nw, 0);

  auto earliest = [&](int w, int id) -> double {
    double est = free_at[w];
    for (const Edge& e : preds[id]) {
      if (e.pred < 0) continue;
      if (!done[e.pred]) return kInf;
      est = std::max(est, end_of[e.pred] + (owner[e.pred] == w ? 0.0 : e.cost));
    }
    return est;
  };

  for (int left = total; left > 0; --left) {
    int best = -1;
    double best_est = kInf;
    for (int w = 0; w < nw; ++w) {
      const int n = int(s.per_worker[w].size());
      while (head[w] < n && done[base[w] + head[w]]) ++head[w];
      if (head[w] >= n) continue;
      int cand = -1;
      double cand_est = kInf;
      bool fwd_seen = false;  // a pending Forward has been reached in this window
      for (int i = head[w]; i < n; ++i) {
        const int id = base[w] + i;
        if (done[id]) continue;
        const bool is_fwd = s.per_worker[w][i].kind == TaskKind::Forward;
        if (i == head[w] || (prm.relaxed && is_fwd && !fwd_seen)) {
          const double est = earliest(w, id);
          if (est < cand_est - kEps) cand = id, cand_est = est;
        }
        fwd_seen |= is_fwd;
        if (!prm.relaxed || (fwd_seen && i > head[w])) break;
      }
      if (cand >= 0 && cand_est < best_est - kEps) best = cand, best_est = cand_est;
    }
    if (best < 0) throw CyclicDependencyError("no schedulable task; dependency cycle in schedule");

    const int w = owner[best], i = best - base[w];
    const TaskKind kind = s.per_worker[w][i].kind;
    const double dur = kind == TaskKind::Backward ? prm.b_dur
                       : kind == TaskKind::Forward ? prm.f_dur
                                                   : 0.0;
    out.spans[w][i] = {best_est, best_est + dur};
    done[best] = 1;
    end_of[best] = best_est + dur;
    free_at[w] = best_est + dur;
    if (prm.post_delays) {
      auto it = prm.post_delays->find({w, i});
      if (it != prm.post_delays->end()) free_at[w] += it->second;
    }
    out.makespan = std::max(out.makespan, best_est + dur);
  }
  return out;
}

// Integer tick lengths from the rationalized backward/forward ratio
// (listsched.hpp:172-188): forward = den (x2 when backwards are halved), backward = num.
struct Ticks {
  long long f = 1;
  long long b = 2;
};

inline bool halved_backward(const PipelineConfig& c) {
  return c.scheme == Scheme::Chimera && c.scaling == ScalingStrategy::BackwardHalving && c.N > c.D;
}

inline Ticks tick_durations(const CostProfile& profile, bool halved) {
  const Rational r = rationalize(profile.backward_ratio);
  return {halved ? 2 * r.den : r.den, r.num};
}

inline Timeline tick_schedule(const Schedule& s, const CostProfile& profile) {
  const Ticks t = tick_durations(profile, halved_backward(s.config));
  Params p;
  p.f_dur = double(t.f);
  p.b_dur = double(t.b);
  return list_schedule(s, p);
}

}  // namespace pipesim::engine
