// Chimera-B200 host layer -- discrete-event timing model and gradient-sync policy.
// Drop-in for proj/include/pipesim/dessim.hpp:24-68 (same declarations).  On the
// GPU the executor *measures* timing; simulate() supplies (a) the eager-sync-opt
// decision the launcher obeys and (b) the predicted timeline shown beside the
// measured one.
#pragma once

#include <optional>
#include <string>
#include <vector>

#include "pipesim/core.hpp"

namespace pipesim::dessim {

enum class SyncPolicy { EndOfIteration, EagerSync, EagerSyncOpt };

std::string to_string(SyncPolicy p);
std::optional<SyncPolicy> sync_policy_from_string(const std::string& s);

struct AllReduceEvent {
  int worker = 0;
  int stage = 0;
  bool eager = false;
  double start = 0;
  double end = 0;
};

struct SimResult {
  Schedule timed;
  double makespan = 0;
  double compute_makespan = 0;
  std::vector<double> per_worker_idle;
  double allreduce_exposed = 0;
  std::vector<AllReduceEvent> allreduce_events;
};

struct SimOptions {
  SyncPolicy policy = SyncPolicy::EndOfIteration;
  double eager_overhead = -1.0;  // < 0: 0.02 * F_t
  bool zero_comm = false;
};

SimResult simulate(const Schedule& s, const CostProfile& profile, const SimOptions& opts = {});

struct MemorySample {
  double time = 0;
  double bytes = 0;
};

std::vector<std::vector<MemorySample>> memory_trace(const SimResult& result,
                                                    const CostProfile& profile);

}  // namespace pipesim::dessim
