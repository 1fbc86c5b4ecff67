// Internal entry into the GPU ToyModel executor (cuda/toy.cu).
#pragma once

#include <vector>

#include "pipesim/core.hpp"

namespace chimera::toy {
// sched == nullptr runs plain mini-batch SGD (sequential_sgd).
void run(const pipesim::Schedule* sched, const std::vector<int>& dims, const double* params_in,
         const double* inputs, const double* targets, int batch, double lr, double* params_out,
         int* peak_stash, int cap);
// oracle::check_gradients on the GPU: max relative error of central finite differences.
double check_gradients(const std::vector<int>& dims, const double* params, const double* inputs,
                       const double* targets, int batch, double step);
}  // namespace chimera::toy
