// Chimera-B200 host layer -- Gantt rendering of a timed schedule.
// Drop-in for proj/include/pipesim/gantt.hpp:23-33 (same declarations).  Renders both
// dessim predictions and measured GPU timelines (pipesim_gantt_timeline).
#pragma once

#include <string>

#include "pipesim/dessim.hpp"

namespace pipesim::gantt {

/// One row per worker, time left to right, colored by pipeline id, hatched for
/// backward passes; allreduce events as outlined bars (red when eager).
std::string render_svg(const dessim::SimResult& result, const CostProfile& profile);

/// One column per F_t: forwards '0'+micro%10, backwards 'A'+micro%26, '.' idle.
std::string render_ascii(const dessim::SimResult& result, const CostProfile& profile);

}  // namespace pipesim::gantt
