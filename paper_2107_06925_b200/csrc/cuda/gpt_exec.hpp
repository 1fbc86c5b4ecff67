// GPT-2 Chimera trainer (cuda/gpt.cu).
#pragma once

#include "pipesim/oracle.hpp"

#include <cstdint>
#include <memory>
#include <stdexcept>
#include <string>

#include <cuda_bf16.h>

#include "gpt_model.hpp"
#include "pipesim/core.hpp"

namespace chimera::gpt {

struct Stash;

// oracle::MissingActivationError itself (status 3 at the C-ABI)
using MissingActivation = pipesim::oracle::MissingActivationError;

class Trainer {
 public:
  Trainer(const ModelShape& shape, const pipesim::Schedule& sched, float lr, int first_rank, int n_ranks);
  ~Trainer();
  float step();          // one full iteration, returns the loss
  void launch_async();   // enqueue one iteration (graph replay) without host sync
  std::string profile_step();  // one eager iteration with per-task GPU timestamps (JSON)
  void upload_batch(const int32_t* tokens, const int32_t* labels, bool from_host, void* stream);
  void set_params(int stage, const float* host);
  void get_params(int stage, float* host) const;
  long long stage_numel(int stage) const;
  std::string layout_json() const;
  std::string stats_json() const;
  void* stream() const;
  void set_use_graph(bool on);
  void set_sync_policy(int policy);  // 0 end-of-iteration, 1 eager-sync, 2 eager-sync-opt
  // The measured CostProfile (F_t, backward_ratio, alpha, beta, L_act, L_grad) the
  // eager-sync-opt decision and the collective order are planned on (dessim::simulate).
  void set_cost_profile(const pipesim::CostProfile& p);
  std::string sync_plan_json() const;  // per stage: eager?, planned launch time
  // Optimizer of the stage update (the reference has SGD only):
  // kind 0 = SGD (default, proj/src/oracle.cpp:283-299), 1 = AdamW with (beta1, beta2,
  // eps, weight_decay).  zero = ZeRO-1: each process holding a stage keeps only its
  // 1/R share of the AdamW moments and updates that share of the weights (gradient
  // reduce-scatter + fp32 weight all-gather over the stage communicator instead of one
  // allreduce).  Multi-process trainers call it after connect().
  void set_optimizer(int kind, float beta1, float beta2, float eps, float weight_decay, bool zero);
  // multi-process: this process's IPC handles (inbox, outbox), then connect with the
  // handles of all processes (ordered by process index) and an NCCL unique id.
  std::string ipc_export() const;
  void connect(const std::string& all_handles, const std::string& nccl_id);
  // Engine-style driving (oracle.cpp:304-356): begin, run_task for every task in a
  // dependency-respecting order (each covers all local replicas), end -> loss.
  // Out-of-order tasks throw MissingActivation before anything is enqueued.
  void begin_iteration();
  void run_task(const pipesim::Task& t);
  void end_iteration();
  float finish_step();  // wait for the iteration, ++steps, return the loss
  bool connected() const;

 public:
  struct Impl;

 private:
  void issue_iteration();
  void forward_task(int rank, int p, int mb, int s);
  void backward_task(int rank, int p, int mb, int s, int pairs = 1);
  void stage_forward(int rank, int s, Stash& X, const __nv_bfloat16* x, __nv_bfloat16* out_final,
                     size_t tok0, float* loss, int pairs = 1);
  // Forward doubling: micro-batches mb, mb+1 (adjacent forwards of one copy) as one 2B-row pass
  void forward_pair(int rank, int p, int mb, int s);
  bool fuse_forward_pair(const pipesim::Task& t, const pipesim::Task& next);
  bool fuse_backward_pair(const pipesim::Task& t, const pipesim::Task& next);
  std::unique_ptr<Impl> d_;
};

}  // namespace chimera::gpt
