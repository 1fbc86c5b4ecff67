// The `pipesim simulate -o` timeline document (reference proj/tools/main.cpp:134-170):
// {policy, makespan, compute_makespan, allreduce_exposed, per_worker_idle,
//  events:[{worker, kind, pipeline_id, micro_batch, stage, start, end}],
//  allreduce:[{worker, stage, eager, start, end}]}.
#pragma once

#include <string>

#include "pipesim/dessim.hpp"

namespace chimera::timeline {

std::string to_json(const pipesim::dessim::SimResult& r, pipesim::dessim::SyncPolicy policy, int indent);
// Inverse (events grouped per worker in document order): lets measured GPU timelines
// in the same schema go through pipesim::gantt.
pipesim::dessim::SimResult from_json(const std::string& text);

}  // namespace chimera::timeline
