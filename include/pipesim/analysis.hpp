// Chimera-B200 host layer -- schedule metrics.
// Drop-in for proj/include/pipesim/analysis.hpp:26-60 (same declarations).
#pragma once

#include <string>
#include <vector>

#include "pipesim/core.hpp"
#include "pipesim/rational.hpp"

namespace pipesim::analysis {

struct MemoryProfile {
  std::vector<int> weight_counts;
  std::vector<int> act_counts;
  std::vector<double> weight_bytes;
  std::vector<double> act_bytes;
  int peak_worker = 0;
  double peak_bytes = 0;
};

std::vector<std::string> validate_dependencies(const Schedule& s);
Rational bubble_ratio(const Schedule& s, const CostProfile& profile);
std::vector<Rational> bubble_ratio_per_worker(const Schedule& s, const CostProfile& profile);
double steady_state_idle(const Schedule& s, const CostProfile& profile);
MemoryProfile memory_profile(const Schedule& s, const CostProfile& profile);
bool fits_memory(const PipelineConfig& config, const CostProfile& profile);

}  // namespace pipesim::analysis
