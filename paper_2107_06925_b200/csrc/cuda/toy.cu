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
// PipeDream (oracle.cpp:205-214,337-345) runs as the reference defines it: every
// forward snapshots its stage's weights (at most D versions per stage, else
// VersionMismatchError), the backward uses the snapshot, and each backward task is
// followed by that stage's update over all replicas with gradient scale 1/(B*W); this
// mode issues everything on one stream.  Other schemes are synchronous (one update
// per stage at the end).  check_gradients (oracle.cpp:358-410) is a finite-difference
// kernel: one CTA per (parameter, +/-step) re-runs the perturbed forward from the
// stored activations of the parameter's stage.
#include <array>
#include <map>
#include <vector>

#include <set>

#include "chimera_ck.h"
#include "common.cuh"
#include "pipesim/core.hpp"
#include "pipesim/oracle.hpp"
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

// params[i] -= lr * sum_c grads[c][i] for i in [lo, hi)  (c = replica * P + pipeline,
// fixed order, copy stride n); `zero` clears the consumed gradients (PipeDream).
__global__ void k_sgd(double* __restrict__ params, double* __restrict__ grads, int copies, long long n,
                      long long lo, long long hi, double lr, bool zero) {
  const long long idx = lo + blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (idx >= hi) return;
  double tot = 0.0;
  for (int c = 0; c < copies; ++c) tot = __dadd_rn(tot, grads[c * n + idx]);
  if (zero)
    for (int c = 0; c < copies; ++c) grads[c * n + idx] = 0.0;
  params[idx] = __dadd_rn(params[idx], -__dmul_rn(lr, tot));
}

constexpr int kMaxToyStages = 32;
struct StageTable {
  int n;                            // stages
  int dims[kMaxToyStages + 1];
  long long w_off[kMaxToyStages];   // flat offsets of W_s and b_s
  long long b_off[kMaxToyStages];
  long long act_stride;             // doubles per activation row block (batch x maxd)
};

// Finite-difference loss probe: CTA (j, side) evaluates the mean loss with parameter j
// moved to value(j) + step (side 0) or value(j) - step (side 1), starting from the
// stored unperturbed input activations of j's stage.  loss[2j + side].
__global__ void k_fd_loss(const double* __restrict__ params, const double* __restrict__ acts,
                          const double* __restrict__ targets, StageTable T, int batch, double step,
                          double* __restrict__ loss) {
  extern __shared__ double sm[];
  const long long j = blockIdx.x;
  const int side = blockIdx.y;
  int s0 = 0;
  while (s0 + 1 < T.n && j >= T.w_off[s0 + 1]) ++s0;
  const long long local = j - T.w_off[s0];
  const long long nw = (long long)T.dims[s0] * T.dims[s0 + 1];
  int pert_o = -1, pert_k = -1;  // perturbed W[o][k] (k = -1: bias o)
  if (local < nw) pert_o = int(local / T.dims[s0]), pert_k = int(local % T.dims[s0]);
  else pert_o = int(local - nw);
  const double base = params[j];
  const double moved = side == 0 ? __dadd_rn(base, step) : __dadd_rn(base, -step);
  int maxd = 0;
  for (int s = 0; s <= T.n; ++s) maxd = max(maxd, T.dims[s]);
  double* x = sm;
  double* y = sm + maxd;
  double* red = sm + 2 * maxd;
  double acc_loss = 0.0;
  for (int i = 0; i < batch; ++i) {
    for (int k = threadIdx.x; k < T.dims[s0]; k += blockDim.x) x[k] = acts[s0 * T.act_stride + (long long)i * maxd + k];
    __syncthreads();
    for (int s = s0; s < T.n; ++s) {
      const int in = T.dims[s], out = T.dims[s + 1];
      const double* w = params + T.w_off[s];
      const double* b = params + T.b_off[s];
      for (int o = threadIdx.x; o < out; o += blockDim.x) {
        double a = (s == s0 && o == pert_o && pert_k < 0) ? moved : b[o];
        for (int k = 0; k < in; ++k) {
          const double wv = (s == s0 && o == pert_o && k == pert_k) ? moved : w[(long long)o * in + k];
          a = __dadd_rn(a, __dmul_rn(wv, x[k]));
        }
        y[o] = tanh(a);
      }
      __syncthreads();
      double* t = x;
      x = y;
      y = t;
    }
    const int out = T.dims[T.n];
    for (int o = threadIdx.x; o < out; o += blockDim.x) {
      const double d = __dadd_rn(x[o], -targets[(long long)i * out + o]);
      acc_loss = __dadd_rn(acc_loss, __dmul_rn(0.5, __dmul_rn(d, d)));
    }
    __syncthreads();
  }
  red[threadIdx.x] = acc_loss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double tot = 0.0;
    for (int t = 0; t < blockDim.x; ++t) tot = __dadd_rn(tot, red[t]);
    loss[2 * j + side] = __dmul_rn(tot, 1.0 / batch);
  }
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

namespace {

// Whole-batch forward + backward of the unpipelined model (the reference's
// sequential_sgd / check_gradients gradient, oracle.cpp:125-151,358-372): activations
// of every layer into `acts` (layer s at acts + s*batch*maxd, row stride = width),
// gradients summed (x 1/batch) into `grads`.
void whole_batch_grads(const std::vector<int>& dims, const Layout& L, const double* params, const double* in,
                       const double* tg, int batch, int maxd, double* acts, double* grads) {
  const int D = int(dims.size()) - 1;
  DeviceBuf gy((size_t)batch * maxd), gx((size_t)batch * maxd), gz((size_t)batch * maxd);
  auto act = [&](int s) { return s == 0 ? in : acts + (size_t)s * batch * maxd; };
  CK_CUDA(cudaMemcpy(acts, in, (size_t)batch * dims[0] * sizeof(double), cudaMemcpyDeviceToDevice));
  for (int s = 0; s < D; ++s)
    k_forward<<<blocks((long long)batch * dims[s + 1]), kThreads>>>(params + L.w_off[s], params + L.b_off[s], act(s),
                                                                   acts + (size_t)(s + 1) * batch * maxd, batch,
                                                                   dims[s], dims[s + 1]);
  const double scale = 1.0 / batch;
  for (int s = D - 1; s >= 0; --s) {
    const int i_ = dims[s], o_ = dims[s + 1];
    k_gz<<<blocks((long long)batch * o_), kThreads>>>(act(s + 1), gy.p, s == D - 1 ? tg : nullptr, gz.p, batch * o_);
    k_wgrad<<<blocks((long long)o_ * i_ + o_), kThreads>>>(gz.p, act(s), grads + L.w_off[s], grads + L.b_off[s], batch,
                                                          i_, o_, scale);
    k_dgrad<<<blocks((long long)batch * i_), kThreads>>>(params + L.w_off[s], gz.p, gx.p, batch, i_, o_);
    std::swap(gy.p, gx.p);
  }
  CK_CUDA(cudaGetLastError());
}

using StashKey = std::array<int, 4>;  // (replica, pipeline, micro, stage) as Engine::stash

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
  bool pipedream = false;
  if (sched) {
    const auto& c = sched->config;
    if (c.D != D) throw pipesim::InvalidConfigError("model stage count must equal D");
    if ((long long)batch != c.mini_batch())
      throw pipesim::InvalidConfigError("batch size must equal B*N*W");
    capi::require_executable(*sched);
    W = c.W, N = c.N, B = c.B, nw = int(sched->per_worker.size());
    pipedream = c.scheme == pipesim::Scheme::PipeDream;
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
    DeviceBuf acts((size_t)(D + 1) * batch * maxd);
    whole_batch_grads(dims, L, d_params.p, d_in.p, d_tg.p, batch, maxd, acts.p, d_grads.p);
    k_sgd<<<blocks(L.n), kThreads>>>(d_params.p, d_grads.p, 1, L.n, 0, L.n, lr, false);
    CK_CUDA(cudaGetLastError());
    CK_CUDA(cudaMemcpy(params_out, d_params.p, L.n * sizeof(double), cudaMemcpyDeviceToHost));
    return;
  }

  // Activation stash / upstream-gradient buffers keyed by (r, p, m, s); PipeDream also
  // keeps the stage weights each stashed forward used.
  const size_t slot = (size_t)B * maxd;
  const size_t keys = (size_t)W * P * N * D;
  long long stage_max = 0;
  for (int s = 0; s < D; ++s) stage_max = std::max(stage_max, (long long)dims[s] * dims[s + 1] + dims[s + 1]);
  DeviceBuf st_in(keys * slot), st_out(keys * slot), g_in(keys * slot), gz_buf(keys * slot),
      snap(pipedream ? keys * stage_max : 0);
  auto key = [&](int r, int p, int m, int s) { return (((size_t)r * P + p) * N + m) * D + s; };

  // One stream per (replica, worker); PipeDream's per-task updates serialise on one.
  std::vector<cudaStream_t> streams(pipedream ? 1 : (size_t)W * nw);
  for (auto& s : streams) CK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
  auto stream_of = [&](int r, int w) { return pipedream ? streams[0] : streams[(size_t)r * nw + w]; };
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

  // Host mirror of Engine::stash / Engine::grad_in (oracle.cpp:174-175): what the
  // reference would find at each step, so misuse raises the same exceptions.
  std::set<StashKey> stash, grad_in;
  std::vector<int> live(nw, 0), peak(nw, 0);
  const double scale = pipedream ? 1.0 / (double(B) * W) : 1.0 / batch;
  for (const auto& [w, i] : capi::replay_order(*sched)) {
    const Task& t = sched->per_worker[w][i];
    if (t.kind != TaskKind::Forward && t.kind != TaskKind::Backward) continue;
    const int p = t.pipeline_id, m = t.micro_batch, s = t.stage;
    if (m < 0 || m >= N || s < 0 || s >= D) throw pipesim::InvalidConfigError("task out of range");
    const int in = dims[s], out = dims[s + 1];
    const long long wn = (long long)in * out + out;
    for (int r = 0; r < W; ++r) {
      cudaStream_t st = stream_of(r, w);
      const size_t k = key(r, p, m, s) * slot;
      if (t.kind == TaskKind::Forward) {
        if (pipedream) {
          int depth = 0;
          for (const StashKey& e : stash) depth += e[0] == r && e[1] == p && e[3] == s;
          if (depth >= D)
            throw pipesim::oracle::VersionMismatchError("weight version stash exhausted on stage " + std::to_string(s));
        }
        const double* x;
        if (s == 0) {
          x = d_in.p + (size_t)(r * N + m) * B * dims[0];
        } else {
          if (!stash.count({r, p, m, s - 1}))
            throw pipesim::oracle::MissingActivationError("missing upstream activation for micro " + std::to_string(m));
          wait_for(st, r, false, p, m, s - 1);
          x = st_out.p + key(r, p, m, s - 1) * slot;
        }
        // stash the input rows (contiguous, stride `in`) and the output
        CK_CUDA(cudaMemcpyAsync(st_in.p + k, x, (size_t)B * in * sizeof(double), cudaMemcpyDeviceToDevice, st));
        if (pipedream)
          CK_CUDA(cudaMemcpyAsync(snap.p + key(r, p, m, s) * stage_max, d_params.p + L.w_off[s], wn * sizeof(double),
                                  cudaMemcpyDeviceToDevice, st));
        k_forward<<<blocks((long long)B * out), kThreads, 0, st>>>(d_params.p + L.w_off[s], d_params.p + L.b_off[s],
                                                                 st_in.p + k, st_out.p + k, B, in, out);
        CK_CUDA(cudaEventRecord(event_of(r, false, t), st));
        stash.insert({r, p, m, s});
        if (r == 0) peak[w] = std::max(peak[w], ++live[w]);
      } else {
        if (!stash.count({r, p, m, s}))
          throw pipesim::oracle::MissingActivationError("backward without stashed activation, micro " +
                                                        std::to_string(m));
        if (s < D - 1 && !grad_in.count({r, p, m, s}))
          throw pipesim::oracle::MissingActivationError("missing upstream gradient, micro " + std::to_string(m));
        stash.erase({r, p, m, s});
        grad_in.erase({r, p, m, s});
        if (s < D - 1) wait_for(st, r, true, p, m, s + 1);
        wait_for(st, r, false, p, m, s);
        const double* target = s == D - 1 ? d_tg.p + (size_t)(r * N + m) * B * dims[D] : nullptr;
        double* grads = d_grads.p + ((size_t)r * P + p) * L.n;
        const double* w_used = pipedream ? snap.p + key(r, p, m, s) * stage_max : d_params.p + L.w_off[s];
        k_gz<<<blocks((long long)B * out), kThreads, 0, st>>>(st_out.p + k, g_in.p + k, target, gz_buf.p + k, B * out);
        k_wgrad<<<blocks((long long)out * in + out), kThreads, 0, st>>>(gz_buf.p + k, st_in.p + k,
                                                                         grads + L.w_off[s], grads + L.b_off[s],
                                                                         B, in, out, scale);
        if (s > 0) {
          k_dgrad<<<blocks((long long)B * in), kThreads, 0, st>>>(w_used, gz_buf.p + k,
                                                                  g_in.p + key(r, p, m, s - 1) * slot, B, in, out);
          grad_in.insert({r, p, m, s - 1});
        }
        CK_CUDA(cudaEventRecord(event_of(r, true, t), st));
        if (r == 0) --live[w];
      }
    }
    if (pipedream && t.kind == TaskKind::Backward)  // Engine::apply_stage_update after each backward
      k_sgd<<<blocks(wn), kThreads, 0, streams[0]>>>(d_params.p, d_grads.p, W * P, L.n, L.w_off[s], L.w_off[s] + wn,
                                                      lr, true);
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
  if (!pipedream) k_sgd<<<blocks(L.n), kThreads, 0, main>>>(d_params.p, d_grads.p, W * P, L.n, 0, L.n, lr, false);
  CK_CUDA(cudaGetLastError());
  CK_CUDA(cudaStreamSynchronize(main));
  CK_CUDA(cudaMemcpy(params_out, d_params.p, L.n * sizeof(double), cudaMemcpyDeviceToHost));
  for (auto& kv : done) cudaEventDestroy(kv.second);
  for (auto& s : streams) cudaStreamDestroy(s);
  for (int w = 0; w < nw && w < cap; ++w) peak_stash[w] = peak[w];
}

double check_gradients(const std::vector<int>& dims, const double* params, const double* inputs,
                       const double* targets, int batch, double step) {
  const int D = int(dims.size()) - 1;
  if (D < 1) throw pipesim::InvalidConfigError("model needs at least one stage");
  if (D > kMaxToyStages) throw pipesim::InvalidConfigError("check_gradients supports at most 32 stages");
  const Layout L(dims);
  int maxd = 0;
  for (int d : dims) maxd = std::max(maxd, d);
  if (batch < 1) return 0.0;
  cuda::require_sm100();
  DeviceBuf d_params(L.n), d_grads(L.n), d_in((size_t)batch * dims[0]), d_tg((size_t)batch * dims[D]),
      acts((size_t)(D + 1) * batch * maxd), loss(2 * (size_t)L.n);
  CK_CUDA(cudaMemcpy(d_params.p, params, L.n * sizeof(double), cudaMemcpyHostToDevice));
  CK_CUDA(cudaMemset(d_grads.p, 0, L.n * sizeof(double)));
  CK_CUDA(cudaMemcpy(d_in.p, inputs, (size_t)batch * dims[0] * sizeof(double), cudaMemcpyHostToDevice));
  CK_CUDA(cudaMemcpy(d_tg.p, targets, (size_t)batch * dims[D] * sizeof(double), cudaMemcpyHostToDevice));
  // activations are laid out with row stride maxd for the probe kernel
  DeviceBuf in_pad((size_t)batch * maxd);
  CK_CUDA(cudaMemset(in_pad.p, 0, (size_t)batch * maxd * sizeof(double)));
  CK_CUDA(cudaMemcpy2D(in_pad.p, maxd * sizeof(double), d_in.p, dims[0] * sizeof(double), dims[0] * sizeof(double),
                       batch, cudaMemcpyDeviceToDevice));
  whole_batch_grads(dims, L, d_params.p, d_in.p, d_tg.p, batch, maxd, acts.p, d_grads.p);
  // whole_batch_grads packs layer s rows with stride dims[s]; re-pack with stride maxd
  DeviceBuf acts_pad((size_t)(D + 1) * batch * maxd);
  CK_CUDA(cudaMemcpy(acts_pad.p, in_pad.p, (size_t)batch * maxd * sizeof(double), cudaMemcpyDeviceToDevice));
  for (int s = 1; s <= D; ++s)
    CK_CUDA(cudaMemcpy2D(acts_pad.p + (size_t)s * batch * maxd, maxd * sizeof(double),
                         acts.p + (size_t)s * batch * maxd, dims[s] * sizeof(double), dims[s] * sizeof(double), batch,
                         cudaMemcpyDeviceToDevice));
  StageTable T{};
  T.n = D;
  for (int s = 0; s <= D; ++s) T.dims[s] = dims[s];
  for (int s = 0; s < D; ++s) T.w_off[s] = L.w_off[s], T.b_off[s] = L.b_off[s];
  T.act_stride = (long long)batch * maxd;
  const int threads = 128;
  const size_t smem = (2 * (size_t)maxd + threads) * sizeof(double);
  if (smem > 200 * 1024) throw pipesim::InvalidConfigError("check_gradients: layer too wide");
  if (smem > 48 * 1024)
    CK_CUDA(cudaFuncSetAttribute(k_fd_loss, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
  k_fd_loss<<<dim3(unsigned(L.n), 2), threads, smem>>>(d_params.p, acts_pad.p, d_tg.p, T, batch, step, loss.p);
  CK_CUDA(cudaGetLastError());
  std::vector<double> g(L.n), lo(2 * L.n), p(params, params + L.n);
  CK_CUDA(cudaMemcpy(g.data(), d_grads.p, L.n * sizeof(double), cudaMemcpyDeviceToHost));
  CK_CUDA(cudaMemcpy(lo.data(), loss.p, 2 * L.n * sizeof(double), cudaMemcpyDeviceToHost));
  double worst = 0;
  for (long long j = 0; j < L.n; ++j) {
    const double fd = (lo[2 * j] - lo[2 * j + 1]) / (2.0 * step);
    const double denom = std::max({1.0, std::abs(fd), std::abs(g[j])});
    worst = std::max(worst, std::abs(fd - g[j]) / denom);
  }
  return worst;
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

CK_API int ck_toy_check_gradients(const int* dims, int n_dims, const double* params, const double* inputs,
                                  const double* targets, int batch, double step, double* max_rel_err) {
  return chimera::capi::guarded([&] {
    *max_rel_err = chimera::toy::check_gradients(std::vector<int>(dims, dims + n_dims), params, inputs, targets,
                                                 batch, step);
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
