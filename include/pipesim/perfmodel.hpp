// Chimera-B200 host layer -- communication cost model and stage-replica groups.
// Drop-in for proj/include/pipesim/perfmodel.hpp:26-82 (same declarations).
#pragma once

#include <vector>

#include "pipesim/core.hpp"

namespace pipesim::perfmodel {

struct CriticalPath {
  int C_f = 0;
  int C_b = 0;
  std::vector<Task> path;
};

struct StageSlack {
  int stage = 0;
  double slack = 0;
};

struct FreeRegions {
  std::vector<std::vector<StageSlack>> per_worker;
};

struct PlanEntry {
  int W = 0;
  int D = 0;
  int B = 0;
  int N = 0;
  ScalingStrategy scaling = ScalingStrategy::Direct;
  bool recompute = false;
  double T_predicted = 0;
};

double p2p_cost(double payload_bytes, const CostProfile& profile);
double allreduce_cost(double L_bytes, int replicas, const CostProfile& profile);
bool is_power_of_two(int n);
// Number of processes holding one stage: the allreduce group size (2f*W for Chimera).
int replicas_per_stage(const PipelineConfig& config);
CriticalPath critical_path(const Schedule& s, const CostProfile& profile);
FreeRegions free_regions(const Schedule& s, const CostProfile& profile);
double predict_T(const PipelineConfig& config, const CostProfile& profile);
std::vector<PlanEntry> plan(int P, long long B_hat, const CostProfile& profile, Scheme scheme);

}  // namespace pipesim::perfmodel
