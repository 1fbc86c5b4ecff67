// Shared helpers for the extern "C" layer: error capture and the schedule replay
// order used by every executor (host tests and the GPU runtime).
#pragma once

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "pipesim/analysis.hpp"
#include "pipesim/core.hpp"
#include "pipesim/oracle.hpp"
#include "sched_engine.hpp"

namespace chimera::capi {

inline std::string& last_error() {
  static thread_local std::string msg;
  return msg;
}

// Status convention of the C boundary: 0 ok, 2 invalid input,
// 3 internal (CUDA / NCCL failure, missing activation, deadlock timeout).
// Device-side failures surface to C++ callers as pipesim::oracle::DeviceError.
using InternalError = pipesim::oracle::DeviceError;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const pipesim::InvalidConfigError& e) {
    last_error() = e.what();
    return 2;
  } catch (const std::invalid_argument& e) {
    last_error() = e.what();
    return 2;
  } catch (const std::exception& e) {
    last_error() = e.what();
    return 3;
  } catch (...) {
    last_error() = "unknown error";
    return 3;
  }
}

inline char* dup_string(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

// Precondition of every executed schedule: the schedule must
// pass analysis::validate_dependencies.  Violations map to the exception the
// reference Engine would raise executing it (proj/src/oracle.cpp:210-280): a backward
// whose forward never runs -> MissingActivationError, a dependency cycle ->
// CyclicDependencyError (from the replay-order timing); anything else (duplicate
// tasks, stage order) -> InvalidConfigError listing the violations.
inline void require_executable(const pipesim::Schedule& s) {
  const auto bad = pipesim::analysis::validate_dependencies(s);
  if (bad.empty()) return;
  std::string all;
  for (const auto& v : bad) all += (all.empty() ? "" : "; ") + v;
  for (const auto& v : bad)
    if (v.rfind("backward without matching forward", 0) == 0) throw pipesim::oracle::MissingActivationError(all);
  for (const auto& v : bad)
    if (v.rfind("cyclic dependency", 0) == 0) throw pipesim::CyclicDependencyError(all);
  throw pipesim::InvalidConfigError("schedule fails validate_dependencies: " + all);
}

// Global issue order of a schedule's tasks: unit-profile tick timing, sorted by
// (start, worker, index) -- the reference oracle's replay order
// (proj/src/oracle.cpp:312-327).  Every producer precedes its consumers in it, so a
// host thread issuing in this order never waits on an unrecorded event.
inline std::vector<std::pair<int, int>> replay_order(const pipesim::Schedule& s) {
  const auto tl = pipesim::engine::tick_schedule(s, pipesim::CostProfile{});
  struct Item {
    double start;
    int w, i;
  };
  std::vector<Item> items;
  for (int w = 0; w < int(s.per_worker.size()); ++w)
    for (int i = 0; i < int(s.per_worker[w].size()); ++i) items.push_back({tl.spans[w][i].start, w, i});
  std::sort(items.begin(), items.end(), [](const Item& a, const Item& b) {
    if (a.start != b.start) return a.start < b.start;
    if (a.w != b.w) return a.w < b.w;
    return a.i < b.i;
  });
  std::vector<std::pair<int, int>> out;
  out.reserve(items.size());
  for (const auto& it : items) out.emplace_back(it.w, it.i);
  return out;
}

}  // namespace chimera::capi
