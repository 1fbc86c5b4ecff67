// pipesim::oracle API of the Chimera-B200 build (include/pipesim/oracle.hpp).
// Host-side generators follow proj/src/oracle.cpp:94-123 (same engine, same
// distribution, same draw order => bit-identical models and batches); the training
// entry points run on the GPU through chimera::toy::run (cuda/toy.cu).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <random>

#include "capi_util.hpp"
#include "chimera_ck.h"
#include "pipesim/oracle.hpp"
#include "toy_exec.hpp"

namespace pipesim::oracle {

ToyModel make_model(const std::vector<int>& dims, std::uint64_t seed) {
  if (dims.size() < 2) throw InvalidConfigError("model needs at least one stage");
  ToyModel m;
  m.dims = dims;
  std::mt19937_64 gen(seed);
  std::uniform_real_distribution<double> u(-0.5, 0.5);
  for (std::size_t s = 0; s + 1 < dims.size(); ++s) {
    const double w_scale = 1.0 / std::sqrt(double(dims[s]));
    std::vector<double> w(std::size_t(dims[s]) * dims[s + 1]), b(dims[s + 1]);
    for (auto& v : w) v = u(gen) * w_scale;
    for (auto& v : b) v = u(gen) * 0.1;
    m.weights.push_back(std::move(w));
    m.biases.push_back(std::move(b));
  }
  return m;
}

Batch make_batch(const ToyModel& model, int size, std::uint64_t seed) {
  Batch b;
  b.size = size;
  std::mt19937_64 gen(seed ^ 0x9e3779b97f4a7c15ull);
  std::uniform_real_distribution<double> u(-1.0, 1.0);
  b.inputs.resize(std::size_t(size) * model.in_dim());
  b.targets.resize(std::size_t(size) * model.out_dim());
  for (auto& v : b.inputs) v = u(gen);
  for (auto& v : b.targets) v = u(gen) * 0.5;
  return b;
}

namespace {

std::vector<double> flat(const ToyModel& m) {
  std::vector<double> out;
  for (int s = 0; s < m.stages(); ++s) {
    out.insert(out.end(), m.weights[s].begin(), m.weights[s].end());
    out.insert(out.end(), m.biases[s].begin(), m.biases[s].end());
  }
  return out;
}

ToyModel unflat(const ToyModel& shape, const std::vector<double>& v) {
  ToyModel m = shape;
  std::size_t off = 0;
  for (int s = 0; s < m.stages(); ++s) {
    std::copy_n(v.begin() + off, m.weights[s].size(), m.weights[s].begin());
    off += m.weights[s].size();
    std::copy_n(v.begin() + off, m.biases[s].size(), m.biases[s].begin());
    off += m.biases[s].size();
  }
  return m;
}

}  // namespace

ToyModel sequential_sgd(const ToyModel& model, const Batch& batch, double lr) {
  auto p = flat(model);
  std::vector<double> out(p.size());
  chimera::toy::run(nullptr, model.dims, p.data(), batch.inputs.data(), batch.targets.data(),
                    batch.size, lr, out.data(), nullptr, 0);
  return unflat(model, out);
}

IterationTrace run_iteration_traced(const Schedule& s, const ToyModel& model, const Batch& batch,
                                    double lr) {
  auto p = flat(model);
  std::vector<double> out(p.size());
  IterationTrace tr;
  tr.peak_stash_per_worker.assign(s.per_worker.size(), 0);
  chimera::toy::run(&s, model.dims, p.data(), batch.inputs.data(), batch.targets.data(), batch.size,
                    lr, out.data(), tr.peak_stash_per_worker.data(), int(s.per_worker.size()));
  tr.model = unflat(model, out);
  return tr;
}

ToyModel run_iteration(const Schedule& s, const ToyModel& model, const Batch& batch, double lr) {
  return run_iteration_traced(s, model, batch, lr).model;
}

double check_gradients(const ToyModel& model, const Batch& batch, double step) {
  const auto p = flat(model);
  return chimera::toy::check_gradients(model.dims, p.data(), batch.inputs.data(), batch.targets.data(), batch.size,
                                       step);
}

double max_relative_diff(const ToyModel& a, const ToyModel& b) {
  const auto x = flat(a), y = flat(b);
  double worst = 0;
  for (std::size_t i = 0; i < x.size(); ++i)
    worst = std::max(worst, std::abs(x[i] - y[i]) /
                                std::max({1e-9, std::abs(x[i]), std::abs(y[i])}));
  return worst;
}

}  // namespace pipesim::oracle

extern "C" {

CK_API int ck_toy_make_model(const int* dims, int n_dims, uint64_t seed, double* params) {
  return chimera::capi::guarded([&] {
    const auto m = pipesim::oracle::make_model(std::vector<int>(dims, dims + n_dims), seed);
    const auto f = pipesim::oracle::flat(m);
    std::memcpy(params, f.data(), f.size() * sizeof(double));
  });
}

CK_API int ck_toy_make_batch(const int* dims, int n_dims, int size, uint64_t seed, double* inputs,
                             double* targets) {
  return chimera::capi::guarded([&] {
    pipesim::oracle::ToyModel m;
    m.dims.assign(dims, dims + n_dims);
    const auto b = pipesim::oracle::make_batch(m, size, seed);
    std::memcpy(inputs, b.inputs.data(), b.inputs.size() * sizeof(double));
    std::memcpy(targets, b.targets.data(), b.targets.size() * sizeof(double));
  });
}

}  // extern "C"
