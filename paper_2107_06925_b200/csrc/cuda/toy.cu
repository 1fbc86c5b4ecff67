// ToyModel stage executor on the GPU: the reference oracle's Engine
// (proj/src/oracle.cpp:162-356) re-designed as a multi-stream CUDA executor.
//
// * every logical worker (replica r, worker w) owns a CUDA stream; tasks are issued
//   in the reference replay order (unit-tick start, worker, index), so each
//   cross-worker data edge -- F(p,m,s-1)->F(p,m,s), B(p,m,s+1)->B(p,m,s) -- is a
//   cudaStreamWaitEvent on an event that was recorded before the wait is issued;
// * forward = y = tanh(W x + b) over the B samples of the micro-batch; backward =
//   gz = g (1 - y^2); gW += gz^T x / B_hat; gb += gz / B_hat; gx = W^T gz;
// * gradients accumulate per (replica, pipeline) copy exactly like the reference
//   (oracle.cpp:170-181) and are summed over all 2f*W copies before one SGD step
//   (apply_stage_update, oracle.cpp:283-299);
// * arithmetic is fp64 with explicit round-to-nearest mul/add (no FMA contraction)
//   so the only differences to the CPU oracle are libm-vs-CUDA tanh ulps and the
//   reference's Kahan compensation; the parity bound is 1e-10 relative.
// The peak number of live stashes per worker is counted on the issue path and must
// equal analysis::memory_profile().act_counts (test_oracle.cpp:147-157).
#include <array>
#include <map>
#include <vector>

#include "chimera_ck.h"
#include "common.cuh"
#include "pipesim/core.hpp"
#include "toy_exec.hpp"

namespace chimera::toy {

namespace {

using pipesim::Schedule;
using pipesim::Task;
using pipesim::TaskKind;

__global__ void k_forward(const double* __restrict__ w, const double* __restrict__ b,
                          const double* __restrict__ x, double* __restrict__ y, int rows, int in,
                          int out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * out) return;
  const int i = idx / out, o = idx % out;
  double acc = b[o];
  for (int k = 0; k < in; ++k) acc = __dadd_rn(acc, __dmul_rn(w[o * in + k], x[i * in + k]));
  y[idx] = tanh(acc);
}

// gz = g_y * (1 - y^2); at the last stage g_y = y - target.
__global__ void k_gz(const double* __restrict__ y, const double* __restrict__ gy,
                     const double* __restrict__ target, double* __restrict__ gz, int n) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= n) return;
  const double g = target ? __dadd_rn(y[idx], -target[idx]) : gy[idx];
  gz[idx] = __dmul_rn(g, __dadd_rn(1.0, -__dmul_rn(y[idx], y[idx])));
}

// gW[o][k] += sum_i gz[i][o] * x[i][k] * scale ; gb[o] += sum_i gz[i][o] * scale
__global__ void k_wgrad(const double* __restrict__ gz, const double* __restrict__ x,
                        double* __restrict__ gw, double* __restrict__ gb, int rows, int in, int out,
                        double scale) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx < out * in) {
    const int o = idx / in, k = idx % in;
    double acc = gw[idx];
    for (int i = 0; i < rows; ++i)
      acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(gz[i * out + o], x[i * in + k]), scale));
    gw[idx] = acc;
  } else if (idx < out * in + out) {
    const int o = idx - out * in;
    double acc = gb[o];
    for (int i = 0; i < rows; ++i) acc = __dadd_rn(acc, __dmul_rn(gz[i * out + o], scale));
    gb[o] = acc;
  }
}

// gx[i][k] = sum_o W[o][k] * gz[i][o]
__global__ void k_dgrad(const double* __restrict__ w, const double* __restrict__ gz,
                        double* __restrict__ gx, int rows, int in, int out) {
  const int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= rows * in) return;
  const int i = idx / in, k = idx % in;
  double acc = 0.0;
  for (int o = 0; o < out; ++o) acc = __dadd_rn(acc, __dmul_rn(w[o * in + k], gz[i * out + o]));
  gx[idx] = acc;
}

// params -= lr * sum_c grads[c]  (c = replica * P + pipeline, fixed order)
__global__ void k_sgd(double* __restrict__ params, const double* __restrict__ grads, int copies,
                      long long n, double lr) {
  const long long idx = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= n) return;
  double tot = 0.0;
  for (int c = 0; c < copies; ++c) tot = __dadd_rn(tot, grads[c * n + idx]);
  params[idx] = __dadd_rn(params[idx], -__dmul_rn(lr, tot));
}

constexpr int kThreads = 128;
inline int blocks(long long n) { return int((n + kThreads - 1) / kThreads); }

struct DeviceBuf {
  double* p = nullptr;
  explicit DeviceBuf(size_t n) { CK_CUDA(cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double))); }
  ~DeviceBuf() { cudaFree(p); }
  DeviceBuf(const DeviceBuf&) = delete;
  DeviceBuf& operator=(const DeviceBuf&) = delete;
};

struct Layout {
  std::vector<long long> w_off, b_off;
  long long n = 0;
  explicit Layout(const std::vector<int>& dims) {
    for (size_t s = 0; s + 1 < dims.size(); ++s) {
      w_off.push_back(n);
      n += (long long)dims[s] * dims[s + 1];
      b_off.push_back(n);
      n += dims[s + 1];
    }
  }
};

}  // namespace

// One full iteration on the current device.  sched == nullptr runs plain mini-batch
// SGD instead (the reference's sequential_sgd, oracle.cpp:125-151).
void run(const Schedule* sched, const std::vector<int>& dims, const double* params_in,
         const double* inputs, const double* targets, int batch, double lr, double* params_out,
         int* peak_stash, int cap) {
  const int D = int(dims.size()) - 1;
  const Layout L(dims);
  int maxd = 0;
  for (int d : dims) maxd = std::max(maxd, d);

  int W = 1, N = batch, B = 1, P = 1, nw = 1;
  if (sched) {
    const auto& c = sched->config;
    if (c.D != D) throw pipesim::InvalidConfigError("model stage count must equal D");
    if ((long long)batch != c.mini_batch())
      throw pipesim::InvalidConfigError("batch size must equal B*N*W");
    W = c.W, N = c.N, B = c.B, nw = int(sched->per_worker.size());
    for (const auto& wl : sched->per_worker)
      for (const Task& t : wl) P = std::max(P, t.pipeline_id + 1);
  }

  cuda::require_sm100();
  DeviceBuf d_params(L.n), d_grads((size_t)W * P * L.n), d_in((size_t)batch * dims[0]),
      d_tg((size_t)batch * dims[D]);
  CK_CUDA(cudaMemcpy(d_params.p, params_in, L.n * sizeof(double), cudaMemcpyHostToDevice));
  CK_CUDA(cudaMemset(d_grads.p, 0, (size_t)W * P * L.n * sizeof(double)));
  CK_CUDA(cudaMemcpy(d_in.p, inputs, (size_t)batch * dims[0] * sizeof(double), cudaMemcpyHostToDevice));
  CK_CUDA(cudaMemcpy(d_tg.p, targets, (size_t)batch * dims[D] * sizeof(double), cudaMemcpyHostToDevice));
  // pageable uploads may still be in flight: order them before the non-blocking streams
  CK_CUDA(cudaDeviceSynchronize());

  if (!sched) {  // sequential SGD: one stream, all stages on the whole batch
    DeviceBuf acts((size_t)(D + 1) * batch * maxd), gy((size_t)batch * maxd), gx((size_t)batch * maxd),
        gz((size_t)batch * maxd);
    auto act = [&](int s) { return s == 0 ? d_in.p : acts.p + (size_t)s * batch * maxd; };
    for (int s = 0; s < D; ++s)
      k_forward<<<blocks((long long)batch * dims[s + 1]), kThreads>>>(
          d_params.p + L.w_off[s], d_params.p + L.b_off[s], act(s), act(s + 1), batch, dims[s], dims[s + 1]);
    const double scale = 1.0 / batch;
    for (int s = D - 1; s >= 0; --s) {
      const int in = dims[s], out = dims[s + 1];
      k_gz<<<blocks((long long)batch * out), kThreads>>>(act(s + 1), gy.p, s == D - 1 ? d_tg.p : nullptr,
                                                         gz.p, batch * out);
      k_wgrad<<<blocks((long long)out * in + out), kThreads>>>(gz.p, act(s), d_grads.p + L.w_off[s],
                                                               d_grads.p + L.b_off[s], batch, in, out, scale);
      k_dgrad<<<blocks((long long)batch * in), kThreads>>>(d_params.p + L.w_off[s], gz.p, gx.p, batch, in, out);
      std::swap(gy.p, gx.p);
    }
    k_sgd<<<blocks(L.n), kThreads>>>(d_params.p, d_grads.p, 1, L.n, lr);
    CK_CUDA(cudaGetLastError());
    CK_CUDA(cudaMemcpy(params_out, d_params.p, L.n * sizeof(double), cudaMemcpyDeviceToHost));
    return;
  }

  // Activation stash / upstream-gradient buffers keyed by (r, p, m, s).
  const size_t slot = (size_t)B * maxd;
  const size_t keys = (size_t)W * P * N * D;
  DeviceBuf st_in(keys * slot), st_out(keys * slot), g_in(keys * slot), gz_buf(keys * slot);
  auto key = [&](int r, int p, int m, int s) { return (((size_t)r * P + p) * N + m) * D + s; };

  std::vector<cudaStream_t> streams((size_t)W * nw);
  for (auto& s : streams) CK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  std::map<std::array<int, 5>, cudaEvent_t> done;  // (r, is_bwd, p, m, s) -> completion
  auto event_of = [&](int r, bool bwd, const Task& t) {
    cudaEvent_t e;
    CK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    done[{r, int(bwd), t.pipeline_id, t.micro_batch, t.stage}] = e;
    return e;
  };
  auto wait_for = [&](cudaStream_t st, int r, bool bwd, int p, int m, int s) {
    auto it = done.find({r, int(bwd), p, m, s});
    if (it != done.end()) CK_CUDA(cudaStreamWaitEvent(st, it->second, 0));
  };

  std::vector<int> live(nw, 0), peak(nw, 0);
  const double scale = 1.0 / batch;
  for (const auto& [w, i] : capi::replay_order(*sched)) {
    const Task& t = sched->per_worker[w][i];
    if (t.kind != TaskKind::Forward && t.kind != TaskKind::Backward) continue;
    const int p = t.pipeline_id, m = t.micro_batch, s = t.stage;
    if (m < 0 || m >= N || s < 0 || s >= D) throw pipesim::InvalidConfigError("task out of range");
    const int in = dims[s], out = dims[s + 1];
    for (int r = 0; r < W; ++r) {
      cudaStream_t st = streams[(size_t)r * nw + w];
      const size_t k = key(r, p, m, s) * slot;
      if (t.kind == TaskKind::Forward) {
        const double* x;
        if (s == 0) {
          x = d_in.p + (size_t)(r * N + m) * B * dims[0];
        } else {
          wait_for(st, r, false, p, m, s - 1);
          x = st_out.p + key(r, p, m, s - 1) * slot;
        }
        // stash the input rows (contiguous, stride `in`) and the output
        CK_CUDA(cudaMemcpyAsync(st_in.p + k, x, (size_t)B * in * sizeof(double), cudaMemcpyDeviceToDevice, st));
        k_forward<<<blocks((long long)B * out), kThreads, 0, st>>>(d_params.p + L.w_off[s], d_params.p + L.b_off[s],
                                                                 st_in.p + k, st_out.p + k, B, in, out);
        CK_CUDA(cudaEventRecord(event_of(r, false, t), st));
        if (r == 0) peak[w] = std::max(peak[w], ++live[w]);
      } else {
        if (s < D - 1) wait_for(st, r, true, p, m, s + 1);
        wait_for(st, r, false, p, m, s);
        const double* target = s == D - 1 ? d_tg.p + (size_t)(r * N + m) * B * dims[D] : nullptr;
        double* grads = d_grads.p + ((size_t)r * P + p) * L.n;
        k_gz<<<blocks((long long)B * out), kThreads, 0, st>>>(st_out.p + k, g_in.p + k, target, gz_buf.p + k, B * out);
        k_wgrad<<<blocks((long long)out * in + out), kThreads, 0, st>>>(gz_buf.p + k, st_in.p + k,
                                                                         grads + L.w_off[s], grads + L.b_off[s],
                                                                         B, in, out, scale);
        if (s > 0)
          k_dgrad<<<blocks((long long)B * in), kThreads, 0, st>>>(d_params.p + L.w_off[s], gz_buf.p + k,
                                                                  g_in.p + key(r, p, m, s - 1) * slot, B, in, out);
        CK_CUDA(cudaEventRecord(event_of(r, true, t), st));
        if (r == 0) --live[w];
      }
    }
  }
  CK_CUDA(cudaGetLastError());
  // flush: the update waits for every worker stream
  cudaStream_t main = streams[0];
  for (size_t k = 1; k < streams.size(); ++k) {
    cudaEvent_t e;
    CK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK_CUDA(cudaEventRecord(e, streams[k]));
    CK_CUDA(cudaStreamWaitEvent(main, e, 0));
    done[{-1, 0, 0, 0, int(k)}] = e;
  }
  k_sgd<<<blocks(L.n), kThreads, 0, main>>>(d_params.p, d_grads.p, W * P, L.n, lr);
  CK_CUDA(cudaGetLastError());
  CK_CUDA(cudaStreamSynchronize(main));
  CK_CUDA(cudaMemcpy(params_out, d_params.p, L.n * sizeof(double), cudaMemcpyDeviceToHost));
  for (auto& kv : done) cudaEventDestroy(kv.second);
  for (auto& s : streams) cudaStreamDestroy(s);
  for (int w = 0; w < nw && w < cap; ++w) peak_stash[w] = peak[w];
}

}  // namespace chimera::toy

extern "C" {

CK_API int ck_toy_run_iteration(const char* schedule_json, const int* dims, int n_dims,
                                const double* params_in, const double* inputs,
                                const double* targets, int batch, double lr, double* params_out,
                                int* peak_stash, int cap) {
  return chimera::capi::guarded([&] {
    if (n_dims < 2) throw pipesim::InvalidConfigError("model needs at least one stage");
    const pipesim::Schedule s = pipesim::schedule_from_json(schedule_json);
    chimera::toy::run(&s, std::vector<int>(dims, dims + n_dims), params_in, inputs, targets, batch,
                      lr, params_out, peak_stash, cap);
  });
}

CK_API int ck_toy_sequential_sgd(const int* dims, int n_dims, const double* params_in,
                                 const double* inputs, const double* targets, int batch, double lr,
                                 double* params_out) {
  return chimera::capi::guarded([&] {
    if (n_dims < 2) throw pipesim::InvalidConfigError("model needs at least one stage");
    chimera::toy::run(nullptr, std::vector<int>(dims, dims + n_dims), params_in, inputs, targets,
                      batch, lr, params_out, nullptr, 0);
  });
}

}  // extern "C"
