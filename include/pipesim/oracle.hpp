// Chimera-B200 -- ToyModel training API, executed on the GPU.
// Drop-in for proj/include/pipesim/oracle.hpp:26-82: same types and signatures.  In the
// reference these run a CPU fp64 engine; here run_iteration / run_iteration_traced /
// sequential_sgd execute sm_100a kernels (one CUDA stream per logical worker, events
// for the schedule's data edges).  make_model / make_batch are host-side and
// bit-identical to the reference (same libstdc++ mt19937_64 + uniform_real_distribution).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <vector>

#include "pipesim/core.hpp"

namespace pipesim::oracle {

struct ToyModel {
  std::vector<int> dims;
  std::vector<std::vector<double>> weights;
  std::vector<std::vector<double>> biases;

  int stages() const { return static_cast<int>(weights.size()); }
  int in_dim() const { return dims.front(); }
  int out_dim() const { return dims.back(); }
};

struct Batch {
  int size = 0;
  std::vector<double> inputs;
  std::vector<double> targets;
};

ToyModel make_model(const std::vector<int>& dims, std::uint64_t seed);
Batch make_batch(const ToyModel& model, int size, std::uint64_t seed);

struct MissingActivationError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct VersionMismatchError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
/// Chimera-B200 extension (not in the reference): the GPU could not run the request --
/// no sm_100 device, a CUDA / NCCL failure, out of device memory.  Every GPU-executed
/// entry point below reports device trouble with this type (C boundary: status 3).
struct DeviceError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

ToyModel sequential_sgd(const ToyModel& model, const Batch& batch, double lr);
ToyModel run_iteration(const Schedule& s, const ToyModel& model, const Batch& batch, double lr);

struct IterationTrace {
  ToyModel model;
  std::vector<int> peak_stash_per_worker;
};

IterationTrace run_iteration_traced(const Schedule& s, const ToyModel& model, const Batch& batch,
                                    double lr);
/// Central finite differences of the mean squared-error loss on every weight and bias
/// against the analytic gradient (proj/src/oracle.cpp:358-410); returns the maximum
/// relative error max|fd - g| / max(1, |fd|, |g|).  Both sides run on the GPU in fp64.
double check_gradients(const ToyModel& model, const Batch& batch, double step = 1e-5);

double max_relative_diff(const ToyModel& a, const ToyModel& b);

}  // namespace pipesim::oracle
