// GPT-2 stage executor: runs a pipesim Schedule (Chimera, or the GPipe / 1F1B
// baselines) as real transformer training on B200.
//
// Mapping: logical rank = r*D + w for data-parallel replica r and
// pipeline worker w; this process hosts a contiguous range of ranks (all of them on
// one GPU, or one per GPU under torchrun).  Each rank owns a CUDA stream; tasks are
// issued in the reference replay order (oracle.cpp:312-327) looping replicas inside
// each task, exactly like oracle::Engine, so every cross-rank data edge is a wait on
// an event recorded earlier in program order.  Per task:
//   Forward(p,m,s):  [embed] -> L/D x (LN, QKV GEMM, flash-attn, O-proj GEMM + bias +
//                    residual, LN, FC1 GEMM + bias + GELU, FC2 GEMM + bias + residual)
//                    -> [final LN, LM-head GEMM, fused softmax-xent fwd+bwd]; the last
//                    layer's epilogue writes straight into the consumer's receive slot.
//   Backward(p,m,s): reverse, dgrad GEMMs (MN-major weights, GELU' fused), wgrad
//                    GEMMs accumulating in fp32 (both operands MN-major), bias grads,
//                    LN backward with the residual gradient fused, flash-attn bwd.
// Gradients accumulate per (rank, pipeline) stage copy (oracle.cpp:170-181); at the
// iteration end every stage's copies are summed (locally, then NCCL across
// processes) and one SGD step updates the fp32 master and the bf16 working copy
// (apply_stage_update, oracle.cpp:283-299).  Activation stashes come from per-copy
// slot pools whose live peak per worker equals analysis::memory_profile().act_counts.
// The whole iteration is captured once into a CUDA graph and replayed.
#include <algorithm>
#include <cstdio>
#include <array>
#include <cstdlib>
#include <cstring>
#include <map>
#include <memory>
#include <numeric>
#include <set>
#include <string>
#include <vector>

#include "nccl_rt.hpp"

#include "chimera_ck.h"
#include "common.cuh"
#include "gemm.cuh"
#include "gpt_exec.hpp"
#include "json_io.hpp"
#include "link_plan.hpp"
#include "links.hpp"
#include "ops.cuh"
#include "pipesim/analysis.hpp"
#include "pipesim/dessim.hpp"
#include "sched_engine.hpp"
#include "pipesim/core.hpp"

namespace chimera::gpt {

using ops::bf16;
using pipesim::Task;
using pipesim::TaskKind;

// ------------------------------------------------------------------- arena --
struct Arena {
  std::vector<void*> blocks;
  size_t bytes = 0;
  ~Arena() {
    for (void* p : blocks) cudaFree(p);
  }
  template <class T>
  T* alloc(size_t n) {
    void* p = nullptr;
    const size_t b = std::max<size_t>(n * sizeof(T), 256);
    CK_CUDA(cudaMalloc(&p, b));
    blocks.push_back(p);
    bytes += b;
    return static_cast<T*>(p);
  }
};

struct LayerStash {
  bf16 *h1, *qkv, *a, *x2, *h2, *u, *g, *xo;
  float *mean1, *rstd1, *mean2, *rstd2, *lse;
};

struct Stash {
  bf16* x0 = nullptr;  // stage-0 embedding output (stage input)
  std::vector<LayerStash> layers;
  bf16* xfinal = nullptr;  // last stage: input of the final LN
  bf16* hf = nullptr;
  float *meanf = nullptr, *rstdf = nullptr;
  bf16* logits = nullptr;  // dlogits after the fused cross-entropy
};

// Backward temporaries of one rank.  Weight / bias gradients run on a side stream one
// layer behind the activation-gradient chain, so the buffers that stream reads rotate:
// the chain's dx over 3 (written at layer l, read by the side stream at layer l-1), the
// per-layer du / dx2 / dqkv over 2; the chain at layer l first waits for the side
// stream's layer l+2, the last reader of the buffers it is about to overwrite.
struct Scratch {
  bf16 *dx[3], *dx2[2], *du[2], *dqkv[2], *dh, *da;
  bf16 *gin2 = nullptr, *gout2 = nullptr;  // backward pairs: gathered input / scattered output gradient
  float* attn;
  float* ws = nullptr;  // split-K workspace of the chain stream's bf16 GEMMs (gemm.cuh EpiArgs::ws)
  long long ws_elems = 0;
  cudaStream_t side = nullptr;  // weight-gradient stream (== the rank stream when serialised)
  cudaEvent_t fork[4], join[3];
};

struct StageState {
  StageLayout L;
  float* w32 = nullptr;
  bf16* w16 = nullptr;
  std::vector<float*> grads;  // gradient buffers of the local copies (one, shared, by default)
  int copies = 0;             // local copies (rank, pipeline) holding this stage
};

struct Copy {  // one (local rank, pipeline) stage replica
  int rank, pipeline, stage;
  float* grad;
  std::vector<Stash> slots;
  std::vector<int> free_slots;
};

struct Trainer::Impl {
  ModelShape m;
  pipesim::Schedule sched;
  float lr;
  int D, W, N, B, P, first, nlocal;
  int M;  // tokens per micro-batch = B * seq
  Arena arena;
  std::vector<cudaStream_t> streams;  // per local rank
  cudaStream_t main_stream;
  std::map<int, StageState> stages;              // stage -> state (stages held locally)
  std::map<std::array<int, 2>, Copy> copies;     // (rank, pipeline) -> copy
  std::vector<Scratch> scratch;                  // per local rank
  std::map<long long, Msg> msgs;                 // messages touching a local rank
  std::vector<int> micro_pipeline;               // micro-batch -> pipeline id
  std::map<std::array<int, 2>, int> worker_of;   // (pipeline, stage) -> worker
  // cross-process plumbing (one process per GPU under torchrun)
  int procs = 1, proc = 0, per = 1;
  void* inbox = nullptr;   // receive buffers + flags of locally consumed messages
  void* outbox = nullptr;  // acks of locally produced, remotely consumed messages
  std::vector<void*> peer_inbox, peer_outbox;  // IPC mappings, indexed by process
  bool connected = false;
  ncclComm_t world_comm = nullptr;
  std::map<int, ncclComm_t> stage_comm;  // stage -> communicator over its holder processes
  // stage -> (flag in a peer holder's inbox to raise, own inbox flag that peer raises):
  // the rendezvous before the stage collective (LinkPlan::ready_flag)
  std::map<int, std::vector<std::pair<uint32_t*, uint32_t*>>> stage_ready;
  std::vector<cudaEvent_t> rank_done;
  cudaEvent_t start_ev, upd_ev;
  int32_t *tokens = nullptr, *labels = nullptr;
  float* loss = nullptr;
  std::vector<std::pair<int, int>> order;
  std::map<std::array<int, 4>, int> slot_of;  // (rank, p, m, s) -> slot index during issue
  std::vector<int> peak_live;                  // per local rank
  // activation recomputation (config.recompute, forced by forward doubling): slots keep
  // only the stage input; one full per-rank workspace is rebuilt by each backward
  bool recompute = false;
  // forward doubling: adjacent forwards of micro-batches (m, m+1) of one copy run as one
  // 2B-row pass (the recompute workspace holds 2M rows; fd_in / fd_out per rank gather the
  // two stage inputs and scatter the two outputs).  CK_FD_FUSE=0 disables.
  bool fd_fuse = false;
  bool bwd_fuse = false;  // backward pairs under forward doubling (CK_BWD_FUSE=0 disables)
  int fwd_pairs = 0, bwd_pairs = 0, bwd_tasks = 0;  // fused pairs / backward tasks issued (last iteration)
  std::vector<bf16*> fd_in, fd_out;
  std::vector<Stash> rscratch;  // per local rank
  float* loss_dummy = nullptr;  // sink for the recomputed last-stage loss
  std::map<std::array<int, 2>, long long> slot_bytes;  // (rank, pipeline) -> bytes of one stash
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t graph_exec = nullptr;
  bool use_graph = true;
  // gradient synchronisation policy (dessim::SyncPolicy): 0 end-of-iteration,
  // 1 eager-sync, 2 eager-sync-opt (eager iff the reference's slack rule says so)
  int sync_policy = 1;
  // CostProfile the gradient-sync plan is computed on (set_cost_profile: the measured
  // B200 profile; default: unit compute with a small alpha-beta allreduce, under which
  // only "slack > 0" decides eager-sync-opt)
  pipesim::CostProfile sync_profile = [] {
    pipesim::CostProfile p;
    p.alpha = 0.01, p.beta = 0.001, p.L_grad = 100.0;
    return p;
  }();
  std::map<int, double> sync_time;  // stage -> planned allreduce start (profile time units)
  // optimizer (set_optimizer): 0 SGD, 1 AdamW; per held stage the moments of its shard
  int optimizer = 0;
  ops::AdamHP adam;
  struct OptState {
    float *m = nullptr, *v = nullptr;
    int* step = nullptr;
    long long lo = 0, hi = 0;  // this process's ZeRO shard of the stage (whole stage if unsharded)
    int pos = 0, holders = 1;  // position in / size of the stage communicator when sharded
  };
  std::map<int, OptState> opt;
  cudaStream_t comm_stream = nullptr;
  std::vector<int> coll_order;                   // stages in the global collective order
  std::map<int, bool> stage_eager;               // stage -> launched at its completion
  std::map<int, int> bwd_total;                  // stage -> local backward tasks per iteration
  std::map<int, std::vector<cudaEvent_t>> stage_done_ev;  // per local copy, after its last bwd
  // profiled iteration: timing events around every task on its rank's stream
  bool profiling = false;
  struct TaskSpan {
    int rank, kind, pipeline, micro, stage;
    cudaEvent_t a, b;
    std::vector<std::pair<cudaEvent_t, cudaEvent_t>> stalls;  // waits for an incoming message
  };
  std::vector<TaskSpan> spans;
  TaskSpan* cur_span = nullptr;  // the span being issued (profiling)
  bool capturing_profile = false;  // profile_step captures its iteration into a graph
  // A timing event: recorded as an event-record NODE when the profiled iteration is
  // being captured (cudaEventRecordExternal), a plain record otherwise.
  void mark(cudaEvent_t e, cudaStream_t st) {
    if (capturing_profile) CK_CUDA(cudaEventRecordWithFlags(e, st, cudaEventRecordExternal));
    else CK_CUDA(cudaEventRecord(e, st));
  }
  // Stream wait for a message, bracketed by events while profiling: the bracket's
  // length is time the rank's stream sat idle inside the task (not busy), so the
  // measured bubble uses busy = span - stalls (dessim's busy = compute only).
  void consume(const Msg& in, cudaStream_t st);
  struct CollSpan {  // one stage's allreduce + SGD on the comm stream
    int stage;
    bool eager;
    cudaEvent_t a, b;
  };
  std::vector<CollSpan> coll_spans;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_next = 0;
  cudaEvent_t timed_event() {
    if (ev_next == ev_pool.size()) {
      cudaEvent_t e;
      CK_CUDA(cudaEventCreate(&e));
      ev_pool.push_back(e);
    }
    return ev_pool[ev_next++];
  }
  int steps = 0;
  long long launches_per_step = 0;
  long long graph_kernels = 0;  // kernel nodes of the captured iteration graph
  // issue state of the open iteration (begin_iteration .. end_iteration)
  struct IterState {
    bool open = false;
    std::map<int, int> bwd_left;                       // stage -> local backwards not yet issued
    std::map<int, int> copy_done;                      // stage -> local copies fully issued
    std::map<std::array<int, 2>, int> copy_bwd_left;   // (rank, pipeline) -> backwards left
    std::set<std::array<int, 4>> issued;               // (kind, pipeline, micro, stage)
    size_t next_coll = 0;
  } it;

  bool local(int rank) const { return rank >= first && rank < first + nlocal; }
  cudaStream_t stream_of(int rank) const { return streams[rank - first]; }
  long long msg_key(int r, int mb, int s, int dir) const {
    return (((long long)r * N + mb) * D + s) * 2 + dir;
  }
  std::unique_ptr<plan::LinkPlan> lp;  // cross-process message plan (host/link_plan.hpp)
  int proc_of(int rank) const { return lp->proc_of(rank); }
};

namespace {

int stage_of(const pipesim::Schedule& s, int w, int p) {
  for (const Task& t : s.per_worker[w])
    if (t.pipeline_id == p) return t.stage;
  return -1;
}

}  // namespace

Trainer::Trainer(const ModelShape& shape, const pipesim::Schedule& sched, float lr, int first_rank,
                 int n_ranks)
    : d_(new Impl) {
  Impl& I = *d_;
  I.m = shape;
  I.sched = sched;
  I.lr = lr;
  const auto& c = sched.config;
  I.D = c.D, I.W = c.W, I.N = c.N, I.B = c.B;
  I.P = 1;
  for (const auto& wl : sched.per_worker)
    for (const Task& t : wl) I.P = std::max(I.P, t.pipeline_id + 1);
  I.first = first_rank;
  I.nlocal = n_ranks;
  I.M = I.B * shape.seq;
  if (shape.stage_layers.empty()) {
    if (shape.n_layer % I.D) throw pipesim::InvalidConfigError("n_layer must be divisible by D");
  } else {
    int sum = 0;
    for (int v : shape.stage_layers) sum += v, v < 1 ? throw pipesim::InvalidConfigError("empty stage") : 0;
    if (int(shape.stage_layers.size()) != I.D || sum != shape.n_layer)
      throw pipesim::InvalidConfigError("stage_layers must have D entries summing to n_layer");
  }
  if (shape.hidden != shape.heads * 64) throw pipesim::InvalidConfigError("head dim must be 64");
  if (shape.hidden % 256) throw pipesim::InvalidConfigError("hidden must be a multiple of 256");
  if (shape.vocab_padded % 8 || shape.vocab_padded < shape.vocab)
    throw pipesim::InvalidConfigError("vocab_padded must be >= vocab and a multiple of 8");
  if (first_rank < 0 || n_ranks < 1 || first_rank + n_ranks > I.W * I.D)
    throw pipesim::InvalidConfigError("rank range outside W*D");
  if (int(sched.per_worker.size()) != I.D) throw pipesim::InvalidConfigError("schedule must have D workers");
  if ((I.W * I.D) % n_ranks || first_rank % n_ranks)
    throw pipesim::InvalidConfigError("ranks must split evenly over processes (contiguous blocks)");
  I.per = n_ranks;
  I.procs = I.W * I.D / n_ranks;
  I.proc = first_rank / n_ranks;
  I.lp = std::make_unique<plan::LinkPlan>(sched, n_ranks, ((size_t)I.M * shape.hidden * 2 + 255) / 256 * 256);
  I.micro_pipeline = I.lp->micro_pipeline;
  I.worker_of = I.lp->worker_of;
  cuda::require_sm100();

  const int h = shape.hidden, f = shape.ffn, M = I.M;
  int Lmax = 0;
  for (int st = 0; st < I.D; ++st) Lmax = std::max(Lmax, shape.layers_of(I.D, st));
  const int H = shape.heads;
  // ---- stage weights and per-copy state
  for (int rank = first_rank; rank < first_rank + n_ranks; ++rank) {
    const int w = rank % I.D;
    for (int p = 0; p < I.P; ++p) {
      const int s = stage_of(sched, w, p);
      if (s < 0) continue;
      if (!I.stages.count(s)) {
        StageState st;
        st.L = make_stage_layout(shape, I.D, s);
        st.w32 = I.arena.alloc<float>(st.L.total);
        st.w16 = I.arena.alloc<bf16>(st.L.total);
        CK_CUDA(cudaMemset(st.w32, 0, st.L.total * sizeof(float)));
        CK_CUDA(cudaMemset(st.w16, 0, st.L.total * sizeof(bf16)));
        I.stages[s] = std::move(st);
      }
      // The local copies of a stage accumulate into ONE fp32 gradient buffer (every
      // gradient accumulation is atomic: TMA reduce-add / vector red in the GEMMs,
      // atomics in LayerNorm, bias, embedding backward), so the optimizer step reads one
      // gradient per parameter instead of one per copy -- Engine::apply_stage_update's
      // sum over copies (oracle.cpp:283-299) happens as the gradients are produced.
      // CK_SHARED_GRADS=0: one buffer per copy, summed by the update kernel.
      static const bool shared = [] {
        const char* e = std::getenv("CK_SHARED_GRADS");
        return !(e && e[0] == '0');
      }();
      StageState& S = I.stages[s];
      Copy cp{rank, p, s, nullptr, {}, {}};
      if (shared && !S.grads.empty()) {
        cp.grad = S.grads[0];
      } else {
        cp.grad = I.arena.alloc<float>(S.L.total);
        CK_CUDA(cudaMemset(cp.grad, 0, S.L.total * sizeof(float)));
        S.grads.push_back(cp.grad);
      }
      S.copies++;
      I.copies[{rank, p}] = std::move(cp);
    }
  }
  // ---- replay order and stash slot counts (simulated issue => per-copy peaks)
  I.order = capi::replay_order(sched);
  std::map<std::array<int, 2>, int> live, peak;
  I.peak_live.assign(n_ranks, 0);
  std::vector<int> live_rank(n_ranks, 0);
  for (const auto& [w, i] : I.order) {
    const Task& t = sched.per_worker[w][i];
    if (t.kind != TaskKind::Forward && t.kind != TaskKind::Backward) continue;
    for (int r = 0; r < I.W; ++r) {
      const int rank = r * I.D + w;
      if (!I.local(rank)) continue;
      auto& l = live[{rank, t.pipeline_id}];
      if (t.kind == TaskKind::Forward) {
        l++;
        live_rank[rank - first_rank]++;
      } else {
        l--;
        live_rank[rank - first_rank]--;
      }
      peak[{rank, t.pipeline_id}] = std::max(peak[{rank, t.pipeline_id}], l);
      I.peak_live[rank - first_rank] = std::max(I.peak_live[rank - first_rank], live_rank[rank - first_rank]);
    }
  }
  I.recompute = c.recompute;
  {
    const char* e = std::getenv("CK_FD_FUSE");
    I.fd_fuse = I.recompute && c.scaling == pipesim::ScalingStrategy::ForwardDoubling && !(e && e[0] == '0');
    const char* b = std::getenv("CK_BWD_FUSE");
    I.bwd_fuse = I.fd_fuse && !(b && b[0] == '0');
  }
  auto alloc_full = [&](Stash& st, bool embed, bool head, int Ls, int pairs = 1) {
      const int M = I.M * pairs;  // rows
      if (embed) st.x0 = I.arena.alloc<bf16>((size_t)M * h);
      for (int l = 0; l < Ls; ++l) {
        LayerStash ls;
        ls.h1 = I.arena.alloc<bf16>((size_t)M * h);
        ls.qkv = I.arena.alloc<bf16>((size_t)M * 3 * h);
        ls.a = I.arena.alloc<bf16>((size_t)M * h);
        ls.x2 = I.arena.alloc<bf16>((size_t)M * h);
        ls.h2 = I.arena.alloc<bf16>((size_t)M * h);
        ls.u = I.arena.alloc<bf16>((size_t)M * f);
        ls.g = I.arena.alloc<bf16>((size_t)M * f);
        ls.xo = (l + 1 < Ls) ? I.arena.alloc<bf16>((size_t)M * h) : nullptr;
        ls.mean1 = I.arena.alloc<float>(M);
        ls.rstd1 = I.arena.alloc<float>(M);
        ls.mean2 = I.arena.alloc<float>(M);
        ls.rstd2 = I.arena.alloc<float>(M);
        ls.lse = I.arena.alloc<float>((size_t)pairs * I.B * H * shape.seq);
        st.layers.push_back(ls);
      }
      if (head) {
        st.xfinal = I.arena.alloc<bf16>((size_t)M * h);
        st.hf = I.arena.alloc<bf16>((size_t)M * h);
        st.meanf = I.arena.alloc<float>(M);
        st.rstdf = I.arena.alloc<float>(M);
        st.logits = I.arena.alloc<bf16>((size_t)M * shape.vocab_padded);
      }
  };
  if (I.recompute) {  // one full workspace per rank; xo of the last layer is a sink
    for (int k = 0; k < n_ranks; ++k) {
      Stash st;
      alloc_full(st, false, true, Lmax, I.fd_fuse ? 2 : 1);
      if (I.fd_fuse) {
        I.fd_in.push_back(I.arena.alloc<bf16>((size_t)2 * M * h));
        I.fd_out.push_back(I.arena.alloc<bf16>((size_t)2 * M * h));
      }
      st.layers.back().xo = I.arena.alloc<bf16>((size_t)(I.fd_fuse ? 2 : 1) * M * h);  // pairs: 2M rows
      I.rscratch.push_back(std::move(st));
    }
    I.loss_dummy = I.arena.alloc<float>(1);
  }
  for (auto& [key, cp] : I.copies) {
    const StageLayout& L = I.stages[cp.stage].L;
    const int nslots = peak[key];
    const size_t before = I.arena.bytes;
    for (int k = 0; k < nslots; ++k) {
      Stash st;
      if (I.recompute) {
        if (L.has_embed) st.x0 = I.arena.alloc<bf16>((size_t)M * h);  // the only stashed tensor
      } else {
        alloc_full(st, L.has_embed, L.has_head, L.n_layers);
      }
      cp.slots.push_back(std::move(st));
    }
    I.slot_bytes[key] = nslots ? (long long)((I.arena.bytes - before) / nslots) : 0;
  }
  // ---- per-rank scratch and streams
  for (int k = 0; k < n_ranks; ++k) {
    Scratch sc;
    const int pm = I.fd_fuse ? 2 : 1;  // backward pairs run on 2M rows
    for (auto& b : sc.dx) b = I.arena.alloc<bf16>((size_t)pm * M * h);
    for (int j = 0; j < 2; ++j) {
      sc.dx2[j] = I.arena.alloc<bf16>((size_t)pm * M * h);
      sc.du[j] = I.arena.alloc<bf16>((size_t)pm * M * f);
      sc.dqkv[j] = I.arena.alloc<bf16>((size_t)pm * M * 3 * h);
    }
    sc.dh = I.arena.alloc<bf16>((size_t)pm * M * h);
    sc.da = I.arena.alloc<bf16>((size_t)pm * M * h);
    if (I.fd_fuse) {
      sc.gin2 = I.arena.alloc<bf16>((size_t)2 * M * h);
      sc.gout2 = I.arena.alloc<bf16>((size_t)2 * M * h);
    }
    sc.attn = I.arena.alloc<float>(ops::attn_bwd_scratch_floats(pm * I.B, shape.seq, H));
    // split-K workspace: the widest chain GEMM output (fused forward pairs: 2M rows)
    sc.ws_elems = (long long)(I.fd_fuse ? 2 : 1) * M * std::max(3 * h, f);
    if (std::getenv("CK_GEMM_SPLIT_BF16") && std::string(std::getenv("CK_GEMM_SPLIT_BF16")) == "0") sc.ws_elems = 0;
    if (sc.ws_elems) {
      sc.ws = I.arena.alloc<float>((size_t)sc.ws_elems);
      CK_CUDA(cudaMemset(sc.ws, 0, (size_t)sc.ws_elems * sizeof(float)));
    }
    cudaStream_t s;
    // CK_STREAM_PRIO=1: the activation / gradient chain streams at the highest priority,
    // the weight-gradient side streams at the lowest (off the pipeline's critical path)
    static const int prio_mode = [] {
      const char* e = std::getenv("CK_STREAM_PRIO");
      return e ? atoi(e) : 0;
    }();
    int prio_lo = 0, prio_hi = 0;
    CK_CUDA(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
    if (prio_mode) cuda::node_priority_flag() = true;
    // CK_SERIALIZE=1: every rank issues on one stream (debug: rules out cross-stream races)
    const bool serial = std::getenv("CK_SERIALIZE") != nullptr;
    if (k > 0 && serial) s = I.streams[0];
    else CK_CUDA(cudaStreamCreateWithPriority(&s, cudaStreamNonBlocking, prio_mode ? prio_hi : 0));
    I.streams.push_back(s);
    // CK_WGRAD_SIDE=0: weight gradients stay on the rank stream (default under CK_SERIALIZE
    // unless CK_WGRAD_SIDE=1: one chain stream + side streams, the one-rank-per-GPU shape)
    const char* ws = std::getenv("CK_WGRAD_SIDE");
    const bool on = ws ? std::string(ws) != "0" : !serial;
    if (!on) sc.side = s;
    else CK_CUDA(cudaStreamCreateWithPriority(&sc.side, cudaStreamNonBlocking, prio_mode ? prio_lo : 0));
    for (auto& e : sc.fork) CK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto& e : sc.join) CK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    I.scratch.push_back(sc);
    cudaEvent_t e;
    CK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    I.rank_done.push_back(e);
  }
  CK_CUDA(cudaStreamCreateWithFlags(&I.main_stream, cudaStreamNonBlocking));
  CK_CUDA(cudaEventCreateWithFlags(&I.start_ev, cudaEventDisableTiming));
  CK_CUDA(cudaEventCreateWithFlags(&I.upd_ev, cudaEventDisableTiming));
  // ---- messages: fwd (r, m, s) feeds stage s+1; bwd (r, m, s) feeds stage s.
  //      Receive buffers + flags live in this process's inbox, acks in its outbox.
  size_t in_bytes = 0, out_bytes = 0;
  const auto in_lay = I.lp->inbox_layout(I.proc, &in_bytes);
  const auto out_lay = I.lp->outbox_layout(I.proc, &out_bytes);
  CK_CUDA(cudaMalloc(&I.inbox, in_bytes));
  CK_CUDA(cudaMalloc(&I.outbox, out_bytes));
  CK_CUDA(cudaMemset(I.inbox, 0, in_bytes));  // flags start at 0
  {
    std::vector<uint32_t> ones(out_bytes / 4, 1u);  // acks start at 1
    CK_CUDA(cudaMemcpy(I.outbox, ones.data(), out_bytes, cudaMemcpyHostToDevice));
  }
  for (int r = 0; r < I.W; ++r)
    for (int mb = 0; mb < I.N; ++mb)
      for (int s = 0; s + 1 < I.D; ++s)
        for (int dir = 0; dir < 2; ++dir) {
          Msg g;
          g.producer = I.lp->producer_of(r, mb, s, dir);
          g.consumer = I.lp->consumer_of(r, mb, s, dir);
          g.prod_local = I.local(g.producer);
          g.cons_local = I.local(g.consumer);
          if (!g.prod_local && !g.cons_local) continue;
          const long long k = I.msg_key(r, mb, s, dir);
          if (g.cons_local) {
            const auto& sl = in_lay.at(k);
            g.buf = reinterpret_cast<bf16*>(static_cast<char*>(I.inbox) + sl.buf);
            g.flag = reinterpret_cast<uint32_t*>(static_cast<char*>(I.inbox) + sl.flag);
          }
          if (g.prod_local && !g.cons_local)
            g.ack = reinterpret_cast<uint32_t*>(static_cast<char*>(I.outbox) + out_lay.at(k));
          if (g.prod_local && g.cons_local)
            CK_CUDA(cudaEventCreateWithFlags(&g.ev, cudaEventDisableTiming));
          I.msgs[k] = g;
        }
  I.connected = I.procs == 1;
  const size_t toks = (size_t)I.W * I.N * I.B * shape.seq;
  I.tokens = I.arena.alloc<int32_t>(toks);
  I.labels = I.arena.alloc<int32_t>(toks);
  I.loss = I.arena.alloc<float>(1);
  CK_CUDA(cudaMemset(I.tokens, 0, toks * 4));
  CK_CUDA(cudaMemset(I.labels, 0, toks * 4));
  CK_CUDA(cudaDeviceSynchronize());
}

Trainer::~Trainer() {
  Impl& I = *d_;
  if (I.graph_exec) cudaGraphExecDestroy(I.graph_exec);
  if (I.graph) cudaGraphDestroy(I.graph);
  for (auto& kv : I.msgs)
    if (kv.second.ev) cudaEventDestroy(kv.second.ev);
  for (auto& kv : I.stage_comm) Nccl::get().CommDestroy(kv.second);
  if (I.world_comm) Nccl::get().CommDestroy(I.world_comm);
  for (void* p : I.peer_inbox)
    if (p) cudaIpcCloseMemHandle(p);
  for (void* p : I.peer_outbox)
    if (p) cudaIpcCloseMemHandle(p);
  cudaFree(I.inbox);
  cudaFree(I.outbox);
  for (auto e : I.rank_done) cudaEventDestroy(e);
  for (auto e : I.ev_pool) cudaEventDestroy(e);
  for (auto& kv : I.stage_done_ev)
    for (auto e : kv.second) cudaEventDestroy(e);
  if (I.comm_stream) cudaStreamDestroy(I.comm_stream);
  cudaEventDestroy(I.start_ev);
  cudaEventDestroy(I.upd_ev);
  for (size_t k = 0; k < I.scratch.size(); ++k) {
    Scratch& sc = I.scratch[k];
    for (auto e : sc.fork) cudaEventDestroy(e);
    for (auto e : sc.join) cudaEventDestroy(e);
    if (sc.side && sc.side != I.streams[k]) cudaStreamDestroy(sc.side);
  }
  for (size_t k = 0; k < I.streams.size(); ++k)
    if (k == 0 || I.streams[k] != I.streams[0]) cudaStreamDestroy(I.streams[k]);
  cudaStreamDestroy(I.main_stream);
}

void Trainer::Impl::consume(const Msg& in, cudaStream_t st) {
  if (!profiling || !cur_span) return in.before_consume(st);
  cudaEvent_t a = timed_event(), b = timed_event();
  mark(a, st);
  in.before_consume(st);
  mark(b, st);
  cur_span->stalls.emplace_back(a, b);
}

// ----------------------------------------------------------- task kernels --
namespace {

using gemm::EpiArgs;

EpiArgs epi(void* out, long long ldo, const bf16* bias = nullptr, const bf16* aux = nullptr,
            long long ld_aux = 0, bf16* out2 = nullptr, long long ld_out2 = 0) {
  EpiArgs e;
  e.out = out, e.ldo = ldo, e.bias = bias, e.aux = aux, e.ld_aux = ld_aux, e.out2 = out2, e.ld_out2 = ld_out2;
  e.atomic_acc = true;  // weight gradients: copies on concurrent streams share the buffer
  return e;
}

// A bf16-epilogue GEMM on a rank's chain stream may split K through that stream's workspace.
EpiArgs on_chain(EpiArgs e, const Scratch& sc) {
  e.ws = sc.ws;
  e.ws_elems = sc.ws_elems;
  return e;
}

}  // namespace

void Trainer::forward_task(int rank, int p, int mb, int s) {
  Impl& I = *d_;
  const ModelShape& m = I.m;
  const int h = m.hidden, M = I.M, r = rank / I.D;
  cudaStream_t st = I.stream_of(rank);
  Copy& cp = I.copies.at({rank, p});
  StageState& S = I.stages.at(s);
  const StageLayout& L = S.L;
  const bf16* w = S.w16;
  if (cp.free_slots.empty()) throw capi::InternalError("stash pool exhausted");
  const int slot = cp.free_slots.back();
  cp.free_slots.pop_back();
  I.slot_of[{rank, p, mb, s}] = slot;
  Stash& X = cp.slots[slot];
  const size_t tok0 = (size_t)(r * I.N + mb) * I.B * m.seq;

  const bf16* x;
  if (s == 0) {
    ops::embed_fwd(I.tokens + tok0, w + L.wte, w + L.wpe, X.x0, M, m.seq, h, st);
    x = X.x0;
  } else {
    const Msg& in = I.msgs.at(I.msg_key(r, mb, s - 1, 0));
    I.consume(in, st);
    x = in.buf;
  }
  const Msg* out_msg = (s + 1 < I.D) ? &I.msgs.at(I.msg_key(r, mb, s, 0)) : nullptr;
  if (out_msg) out_msg->before_produce(st);
  Stash& Wk = I.recompute ? I.rscratch[rank - I.first] : X;  // activations land here
  bf16* out_final = out_msg ? out_msg->buf : Wk.xfinal;
  stage_forward(rank, s, Wk, x, out_final, tok0, I.loss);
  if (!L.has_head) out_msg->after_produce(st);
  if (s == 0) I.launches_per_step += 1;
}

// Forward doubling (schedgen.cpp:104-111): the two real micro-batches mb, mb+1
// that one virtual micro-batch expands to run as ONE pass of 2B sequences -- GEMMs of 2M
// rows instead of two of M (the 632-row GPT-2 1.3B stage GEMMs fill 3 of their 256-row
// tiles 2.5 times) -- through the 2M-row recompute workspace: the two stage inputs are
// gathered into fd_in, the 2M-row output is scattered to the two outgoing messages (peer
// copies over NVLink when the consumer is remote).  Stash discipline, slot accounting and
// message handshakes are exactly those of two forward_task calls.
void Trainer::forward_pair(int rank, int p, int mb, int s) {
  Impl& I = *d_;
  const ModelShape& m = I.m;
  const int h = m.hidden, M = I.M, r = rank / I.D;
  const size_t bytes = (size_t)M * h * sizeof(bf16);
  cudaStream_t st = I.stream_of(rank);
  Copy& cp = I.copies.at({rank, p});
  const StageLayout& L = I.stages.at(s).L;
  const bf16* w = I.stages.at(s).w16;
  bf16* xin = I.fd_in[rank - I.first];
  const Msg* outs[2] = {nullptr, nullptr};
  for (int k = 0; k < 2; ++k) {
    if (cp.free_slots.empty()) throw capi::InternalError("stash pool exhausted");
    const int slot = cp.free_slots.back();
    cp.free_slots.pop_back();
    I.slot_of[{rank, p, mb + k, s}] = slot;
    Stash& X = cp.slots[slot];
    const size_t tok0 = (size_t)(r * I.N + mb + k) * I.B * m.seq;
    if (s == 0) {
      ops::embed_fwd(I.tokens + tok0, w + L.wte, w + L.wpe, X.x0, M, m.seq, h, st);
      CK_CUDA(cudaMemcpyAsync(xin + (size_t)k * M * h, X.x0, bytes, cudaMemcpyDeviceToDevice, st));
      I.launches_per_step += 1;
    } else {
      const Msg& in = I.msgs.at(I.msg_key(r, mb + k, s - 1, 0));
      I.consume(in, st);
      CK_CUDA(cudaMemcpyAsync(xin + (size_t)k * M * h, in.buf, bytes, cudaMemcpyDeviceToDevice, st));
    }
    if (s + 1 < I.D) {
      outs[k] = &I.msgs.at(I.msg_key(r, mb + k, s, 0));
      outs[k]->before_produce(st);
    }
  }
  Stash& Wk = I.rscratch[rank - I.first];
  bf16* out_final = L.has_head ? Wk.xfinal : I.fd_out[rank - I.first];
  stage_forward(rank, s, Wk, xin, out_final, (size_t)(r * I.N + mb) * I.B * m.seq, I.loss, 2);
  if (!L.has_head)
    for (int k = 0; k < 2; ++k) {
      CK_CUDA(cudaMemcpyAsync(outs[k]->buf, out_final + (size_t)k * M * h, bytes, cudaMemcpyDeviceToDevice, st));
      outs[k]->after_produce(st);
    }
}

// The layers (+ final LN, LM head, fused cross-entropy) of stage s for one
// micro-batch: activations into X, stage output into out_final.
void Trainer::stage_forward(int rank, int s, Stash& X, const bf16* x, bf16* out_final, size_t tok0,
                            float* loss, int pairs) {
  Impl& I = *d_;
  const ModelShape& m = I.m;
  const int h = m.hidden, f = m.ffn, M = I.M * pairs, H = m.heads, Bq = I.B * pairs;  // rows, sequences
  cudaStream_t st = I.stream_of(rank);
  const StageLayout& L = I.stages.at(s).L;
  const bf16* w = I.stages.at(s).w16;
  const Scratch& sc = I.scratch[rank - I.first];
  for (int l = 0; l < L.n_layers; ++l) {
    const LayerOffsets& o = L.layers[l];
    LayerStash& A = X.layers[l];
    bf16* xo = (l + 1 < L.n_layers) ? A.xo : out_final;
    ops::layernorm_fwd(x, w + o.ln1_g, w + o.ln1_b, A.h1, A.mean1, A.rstd1, M, h, st);
    gemm::gemm(gemm::kStoreBF16, false, false, M, 3 * h, h, A.h1, h, w + o.w_qkv, h,
               on_chain(epi(A.qkv, 3 * h, w + o.b_qkv), sc), st);
    ops::attn_fwd_tc(A.qkv, A.a, A.lse, Bq, m.seq, H, m.causal, st);
    gemm::gemm(gemm::kBiasResid, false, false, M, h, h, A.a, h, w + o.w_o, h,
               on_chain(epi(A.x2, h, w + o.b_o, x, h), sc), st);
    ops::layernorm_fwd(A.x2, w + o.ln2_g, w + o.ln2_b, A.h2, A.mean2, A.rstd2, M, h, st);
    gemm::gemm(gemm::kBiasGelu, false, false, M, f, h, A.h2, h, w + o.w_fc1, h,
               on_chain(epi(A.u, f, w + o.b_fc1, nullptr, 0, A.g, f), sc), st);
    gemm::gemm(gemm::kBiasResid, false, false, M, h, f, A.g, f, w + o.w_fc2, f,
               on_chain(epi(xo, h, w + o.b_fc2, A.x2, h), sc), st);
    x = xo;
    I.launches_per_step += 7;
  }
  if (L.has_head) {
    ops::layernorm_fwd(X.xfinal, w + L.lnf_g, w + L.lnf_b, X.hf, X.meanf, X.rstdf, M, h, st);
    gemm::gemm(gemm::kStoreBF16, false, false, M, m.vocab_padded, h, X.hf, h, w + L.w_head, h,
               epi(X.logits, m.vocab_padded), st);
    const float scale = 1.f / float((double)I.W * I.N * I.B * m.seq);
    ops::xent_fwd_bwd(X.logits, m.vocab_padded, I.labels + tok0, M, m.vocab, m.vocab_padded, scale, scale,
                      loss, st);
    I.launches_per_step += 3;
  }
}

// pairs = 2 (forward doubling, backward_pair): the backwards of micro-batches mb, mb+1 --
// adjacent on the worker -- as ONE pass over 2B sequences: the two stashed stage inputs
// are gathered for the recompute, the two incoming gradients gathered, every GEMM runs
// on 2M rows (the weight gradients with K = 2M: one fp32 accumulate instead of two), and
// the 2M-row input gradient is scattered to the two outgoing messages.
void Trainer::backward_task(int rank, int p, int mb, int s, int pairs) {
  Impl& I = *d_;
  const ModelShape& m = I.m;
  const int h = m.hidden, f = m.ffn, M1 = I.M, M = I.M * pairs, H = m.heads, r = rank / I.D;
  const size_t msg_bytes = (size_t)M1 * h * sizeof(bf16);
  cudaStream_t st = I.stream_of(rank);
  Copy& cp = I.copies.at({rank, p});
  StageState& S = I.stages.at(s);
  const StageLayout& L = S.L;
  const bf16* w = S.w16;
  float* gw = cp.grad;
  int slots[2] = {-1, -1};
  for (int k = 0; k < pairs; ++k) {
    const auto it = I.slot_of.find({rank, p, mb + k, s});
    if (it == I.slot_of.end()) throw capi::InternalError("backward without stashed activation");
    slots[k] = it->second;
    I.slot_of.erase(it);
  }
  Stash& Xslot = cp.slots[slots[0]];
  Scratch& sc = I.scratch[rank - I.first];
  const size_t tok0 = (size_t)(r * I.N + mb) * I.B * m.seq;
  const bf16* stage_in = s == 0 ? Xslot.x0 : I.msgs.at(I.msg_key(r, mb, s - 1, 0)).buf;
  if (pairs == 2) {  // gather the two stage inputs (kept until this task: stash / inbox)
    bf16* xin2 = I.fd_in[rank - I.first];
    for (int k = 0; k < 2; ++k) {
      const bf16* src = s == 0 ? cp.slots[slots[k]].x0 : I.msgs.at(I.msg_key(r, mb + k, s - 1, 0)).buf;
      CK_CUDA(cudaMemcpyAsync(xin2 + (size_t)k * M1 * h, src, msg_bytes, cudaMemcpyDeviceToDevice, st));
    }
    stage_in = xin2;
  }
  Stash& X = I.recompute ? I.rscratch[rank - I.first] : Xslot;
  if (I.recompute) {  // rebuild the stage's activations from its stashed input
    Stash& Wk = I.rscratch[rank - I.first];
    stage_forward(rank, s, Wk, stage_in, L.has_head ? Wk.xfinal : Wk.layers.back().xo, tok0, I.loss_dummy, pairs);
  }

  // Activation-gradient chain on the rank stream `st`; weight and bias gradients on the
  // side stream (fork after each producer, join per layer: see Scratch).
  cudaStream_t ws = sc.side;
  const bool side = ws != st;
  int fork_i = 0;
  auto fork = [&] {  // the side stream waits for everything issued so far on st
    if (!side) return;
    cudaEvent_t e = sc.fork[fork_i++ & 3];
    CK_CUDA(cudaEventRecord(e, st));
    CK_CUDA(cudaStreamWaitEvent(ws, e, 0));
  };
  const int top = L.has_head ? L.n_layers : L.n_layers - 1;  // highest side-stream "layer" index
  auto side_done = [&](int l) {
    if (side) CK_CUDA(cudaEventRecord(sc.join[l % 3], ws));
  };
  auto wait_side = [&](int l) {  // the chain is about to overwrite buffers side layer l read
    if (side && l <= top) CK_CUDA(cudaStreamWaitEvent(st, sc.join[l % 3], 0));
  };
  const bf16* dxo;
  if (L.has_head) {
    fork();
    gemm::gemm(gemm::kAccF32, true, true, m.vocab_padded, h, M, X.logits, m.vocab_padded, X.hf, h,
               epi(gw + L.w_head, h), ws);
    side_done(L.n_layers);
    gemm::gemm(gemm::kStoreBF16, false, true, M, h, m.vocab_padded, X.logits, m.vocab_padded, w + L.w_head, h,
               on_chain(epi(sc.dh, h), sc), st);
    bf16* d = sc.dx[L.n_layers % 3];
    // (+ the top layer's FC2 bias gradient: column sums of this dx)
    ops::layernorm_bwd(sc.dh, X.xfinal, X.meanf, X.rstdf, w + L.lnf_g, nullptr, d, gw + L.lnf_g,
                       gw + L.lnf_b, gw + L.layers[L.n_layers - 1].b_fc2, M, h, st);
    dxo = d;
    I.launches_per_step += 3;
  } else if (pairs == 1) {
    const Msg& in = I.msgs.at(I.msg_key(r, mb, s, 1));
    I.consume(in, st);
    dxo = in.buf;
  } else {  // gather the two incoming gradients
    for (int k = 0; k < 2; ++k) {
      const Msg& in = I.msgs.at(I.msg_key(r, mb + k, s, 1));
      I.consume(in, st);
      CK_CUDA(cudaMemcpyAsync(sc.gin2 + (size_t)k * M1 * h, in.buf, msg_bytes, cudaMemcpyDeviceToDevice, st));
    }
    dxo = sc.gin2;
  }
  const Msg* out_msgs[2] = {nullptr, nullptr};
  for (int k = 0; k < pairs && s > 0; ++k) {
    out_msgs[k] = &I.msgs.at(I.msg_key(r, mb + k, s - 1, 1));
    out_msgs[k]->before_produce(st);
  }
  const Msg* out_msg = out_msgs[0];
  // a single message is produced in place; a pair's 2M rows go through scratch, then split
  bf16* dx_stage = out_msg ? (pairs == 1 ? out_msg->buf : sc.gout2) : nullptr;
  for (int l = L.n_layers - 1; l >= 0; --l) {
    const LayerOffsets& o = L.layers[l];
    LayerStash& A = X.layers[l];
    const bf16* xin = (l > 0) ? X.layers[l - 1].xo : stage_in;
    bf16* dxin = (l == 0 && dx_stage) ? dx_stage : sc.dx[l % 3];
    bf16 *du = sc.du[l & 1], *dx2 = sc.dx2[l & 1], *dqkv = sc.dqkv[l & 1];
    wait_side(l + 2);
    // MLP
    // Bias gradients ride on the kernels producing the gradient they sum: FC1's in the
    // GELU' epilogue, O-proj's in LN2-backward, FC2's in the LN1-backward of the layer
    // above (or the final LN's), QKV's in the attention backward (dQ conversion, dK / dV
    // epilogue); only the stage's top layer input gradient, arriving as a message, keeps
    // a separate column-sum pass.
    fork();
    if (l == L.n_layers - 1 && !L.has_head) {
      ops::bias_grad(dxo, gw + o.b_fc2, M, h, ws);
      I.launches_per_step += 1;
    }
    gemm::gemm(gemm::kAccF32, true, true, h, f, M, dxo, h, A.g, f, epi(gw + o.w_fc2, f), ws);
    {
      EpiArgs e = on_chain(epi(du, f, nullptr, A.u, f), sc);
      e.colsum = gw + o.b_fc1;
      gemm::gemm(gemm::kGeluBwd, false, true, M, f, h, dxo, h, w + o.w_fc2, f, e, st);
    }
    fork();
    gemm::gemm(gemm::kAccF32, true, true, f, h, M, du, f, A.h2, h, epi(gw + o.w_fc1, h), ws);
    gemm::gemm(gemm::kStoreBF16, false, true, M, h, f, du, f, w + o.w_fc1, h, on_chain(epi(sc.dh, h), sc), st);
    ops::layernorm_bwd(sc.dh, A.x2, A.mean2, A.rstd2, w + o.ln2_g, dxo, dx2, gw + o.ln2_g, gw + o.ln2_b,
                       gw + o.b_o, M, h, st);
    // attention
    fork();
    gemm::gemm(gemm::kAccF32, true, true, h, h, M, dx2, h, A.a, h, epi(gw + o.w_o, h), ws);
    gemm::gemm(gemm::kStoreBF16, false, true, M, h, h, dx2, h, w + o.w_o, h, on_chain(epi(sc.da, h), sc), st);
    ops::attn_bwd_tc(A.qkv, A.a, sc.da, A.lse, dqkv, sc.attn, I.B * pairs, m.seq, H, m.causal, st, gw + o.b_qkv);
    fork();
    gemm::gemm(gemm::kAccF32, true, true, 3 * h, h, M, dqkv, 3 * h, A.h1, h, epi(gw + o.w_qkv, h), ws);
    side_done(l);
    gemm::gemm(gemm::kStoreBF16, false, true, M, h, 3 * h, dqkv, 3 * h, w + o.w_qkv, h, on_chain(epi(sc.dh, h), sc),
               st);
    ops::layernorm_bwd(sc.dh, xin, A.mean1, A.rstd1, w + o.ln1_g, dx2, dxin, gw + o.ln1_g, gw + o.ln1_b,
                       l > 0 ? gw + L.layers[l - 1].b_fc2 : nullptr, M, h, st);
    dxo = dxin;
    I.launches_per_step += 14;  // attn_bwd = 3 kernels (+ a memset node)
  }
  if (s == 0) {
    ops::embed_bwd(I.tokens + tok0, dxo, gw + L.wte, gw + L.wpe, M, m.seq, h, st);
    I.launches_per_step += 1;
  } else {
    for (int k = 0; k < pairs; ++k) {  // the gradient leaves before the side stream is joined
      if (pairs == 2)
        CK_CUDA(cudaMemcpyAsync(out_msgs[k]->buf, dx_stage + (size_t)k * M1 * h, msg_bytes, cudaMemcpyDeviceToDevice,
                                st));
      out_msgs[k]->after_produce(st);
    }
  }
  if (side) {  // join: the side stream read the input message and the stash
    CK_CUDA(cudaEventRecord(sc.join[0], ws));
    CK_CUDA(cudaStreamWaitEvent(st, sc.join[0], 0));
  }
  // this task was the last reader of its input messages
  for (int k = 0; k < pairs; ++k) {
    if (s > 0) I.msgs.at(I.msg_key(r, mb + k, s - 1, 0)).after_last_use(st);
    if (s + 1 < I.D) I.msgs.at(I.msg_key(r, mb + k, s, 1)).after_last_use(st);
    cp.free_slots.push_back(slots[k]);
  }
}

namespace {

// Global order of the per-stage gradient collectives, identical on every process:
// eager stages by the unit-tick time at which their last backward (over all holders)
// ends, then the end-of-iteration ones by stage id.
void plan_sync(Trainer::Impl& I) {
  // dessim::simulate on the sync profile (proj/src/dessim.cpp:60-135): per (worker, held
  // stage) the reference rule -- eager-sync: always; eager-sync-opt: iff the worker
  // idles after that stage's last backward (interior slack > 0).  A stage launches
  // eagerly iff every holder would; eager stages are ordered by their simulated launch
  // time, the others follow by stage id -- the same order on every process.
  pipesim::dessim::SimOptions o;
  o.policy = I.sync_policy == 2 ? pipesim::dessim::SyncPolicy::EagerSyncOpt : pipesim::dessim::SyncPolicy::EagerSync;
  pipesim::CostProfile prof = I.sync_profile;
  if (prof.L_grad <= 0) prof.L_grad = 1.0;  // the rule needs a non-zero allreduce cost
  const auto sim = pipesim::dessim::simulate(I.sched, prof, o);
  std::map<int, bool> all_eager;
  std::map<int, double> start;
  for (const auto& ev : sim.allreduce_events) {
    auto it = all_eager.emplace(ev.stage, true).first;
    it->second = it->second && ev.eager;
    start[ev.stage] = std::max(start[ev.stage], ev.start);
  }
  I.stage_eager.clear();
  I.sync_time = start;
  for (int s = 0; s < I.D; ++s) I.stage_eager[s] = I.sync_policy == 1 || (I.sync_policy == 2 && all_eager[s]);
  std::vector<std::pair<double, int>> eager, late;
  for (int s = 0; s < I.D; ++s) (I.stage_eager[s] ? eager : late).push_back({I.stage_eager[s] ? start[s] : s, s});
  std::sort(eager.begin(), eager.end());
  std::sort(late.begin(), late.end());
  I.coll_order.clear();
  for (auto& e : eager) I.coll_order.push_back(e.second);
  for (auto& e : late) I.coll_order.push_back(e.second);
  I.bwd_total.clear();
  for (const auto& [w, i] : I.order) {
    const Task& t = I.sched.per_worker[w][i];
    if (t.kind != TaskKind::Backward) continue;
    for (int r = 0; r < I.W; ++r)
      if (I.local(r * I.D + w)) I.bwd_total[t.stage]++;
  }
  for (auto& [st, S] : I.stages) {
    auto& evs = I.stage_done_ev[st];
    while (int(evs.size()) < S.copies) {
      cudaEvent_t e;
      CK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      evs.push_back(e);
    }
  }
  if (!I.comm_stream) CK_CUDA(cudaStreamCreateWithFlags(&I.comm_stream, cudaStreamNonBlocking));
}

// Sum the local copies, allreduce across the processes holding the stage (if any),
// SGD -- on the comm stream, after every local copy's last backward.
void sync_stage_body(Trainer::Impl& I, int s);

// Stage s's gradient sync + SGD on the comm stream; timed when profiling.
void sync_stage(Trainer::Impl& I, int s) {
  if (!I.profiling) return sync_stage_body(I, s);
  Trainer::Impl::CollSpan c{s, I.stage_eager.count(s) && I.stage_eager.at(s), I.timed_event(), nullptr};
  I.mark(c.a, I.comm_stream);
  sync_stage_body(I, s);
  c.b = I.timed_event();
  I.mark(c.b, I.comm_stream);
  I.coll_spans.push_back(c);
}

void sync_stage_body(Trainer::Impl& I, int s) {
  StageState& S = I.stages.at(s);
  cudaStream_t cs = I.comm_stream;
  for (cudaEvent_t e : I.stage_done_ev.at(s)) CK_CUDA(cudaStreamWaitEvent(cs, e, 0));
  const bool adam = I.optimizer == 1;
  auto update = [&](float* const* g, int copies) {  // the optimizer step over this process's range
    if (!adam) return ops::sgd_update(S.w32, S.w16, g, copies, S.L.total, I.lr, cs);
    Trainer::Impl::OptState& o = I.opt.at(s);
    ops::AdamHP hp = I.adam;
    hp.lr = I.lr;
    ops::adamw_update(S.w32, S.w16, g, copies, o.m, o.v, o.step, o.lo, o.hi, hp, cs);
    I.launches_per_step += 1;
  };
  auto it = I.stage_comm.find(s);
  if (it == I.stage_comm.end()) {
    update(S.grads.data(), int(S.grads.size()));
    I.launches_per_step += 1;
    return;
  }
  // Rendezvous with the other holders before the collective kernel launches: raise our
  // flag in each peer's inbox, wait for theirs in ours (stream memory operations -- they
  // hold no SMs).  An NCCL kernel spins on its SMs until every peer has launched; without
  // this, one launched early can keep a persistent GEMM's last CTAs off the GPU while the
  // peer it waits for needs that GEMM's output (a cross-process message) to get there.
  // Reset-before-raise is ordered by the collective itself: a peer raises the next
  // iteration's flag only after this iteration's collective, which runs after our reset.
  for (const auto& [remote, own] : I.stage_ready.at(s)) MemOps::get().write(cs, remote, 1);
  for (const auto& [remote, own] : I.stage_ready.at(s)) {
    MemOps::get().wait(cs, own, 1);
    MemOps::get().write(cs, own, 0);
  }
  float* g0 = S.grads[0];
  if (S.grads.size() > 1) {
    ops::reduce_copies(g0, S.grads.data(), int(S.grads.size()), S.L.total, cs);
    for (size_t c = 1; c < S.grads.size(); ++c)
      CK_CUDA(cudaMemsetAsync(S.grads[c], 0, S.L.total * sizeof(float), cs));
    I.launches_per_step += 1;
  }
  if (adam && I.opt.at(s).holders > 1) {  // ZeRO-1: reduce-scatter, shard update, all-gather
    const Trainer::Impl::OptState& o = I.opt.at(s);
    const size_t chunk = size_t(o.hi - o.lo);
    if (Nccl::get().ReduceScatter(g0, g0 + o.lo, chunk, ncclFloat, ncclSum, it->second, cs) != ncclSuccess)
      throw capi::InternalError("ncclReduceScatter failed");
    update(&g0, 1);
    CK_CUDA(cudaMemsetAsync(g0, 0, S.L.total * sizeof(float), cs));  // the other shards' partial sums
    if (Nccl::get().AllGather(S.w32 + o.lo, S.w32, chunk, ncclFloat, it->second, cs) != ncclSuccess)
      throw capi::InternalError("ncclAllGather failed");
    ops::cast_f32_bf16(S.w32, S.w16, S.L.total, cs);
    I.launches_per_step += 1;
    return;
  }
  if (Nccl::get().AllReduce(g0, g0, S.L.total, ncclFloat, ncclSum, it->second, cs) != ncclSuccess)
    throw capi::InternalError("ncclAllReduce failed");
  update(&g0, 1);
  I.launches_per_step += 1;
}

}  // namespace

// Iteration issue, split Engine-style (oracle.cpp:304-356): begin, one call per task in
// replay order (every local replica of it, like the reference's loop over r), end.
// issue_iteration() drives it from the schedule's replay order; the C-ABI exposes the
// same three calls so a host scheduler can drive the GPU task by task.
void Trainer::begin_iteration() {
  Impl& I = *d_;
  if (I.it.open) throw pipesim::InvalidConfigError("iteration already open");
  if (I.coll_order.empty()) plan_sync(I);
  I.launches_per_step = 0;
  I.fwd_pairs = I.bwd_pairs = I.bwd_tasks = 0;
  I.slot_of.clear();
  for (auto& kv : I.copies) {
    Copy& cp = kv.second;
    cp.free_slots.resize(cp.slots.size());
    std::iota(cp.free_slots.rbegin(), cp.free_slots.rend(), 0);
  }
  CK_CUDA(cudaMemsetAsync(I.loss, 0, sizeof(float), I.main_stream));
  CK_CUDA(cudaEventRecord(I.start_ev, I.main_stream));
  for (auto s : I.streams) CK_CUDA(cudaStreamWaitEvent(s, I.start_ev, 0));
  CK_CUDA(cudaStreamWaitEvent(I.comm_stream, I.start_ev, 0));
  Impl::IterState& S = I.it;
  S = Impl::IterState{};
  S.open = true;
  S.bwd_left = I.bwd_total;
  for (const auto& [w, i] : I.order) {
    const Task& t = I.sched.per_worker[w][i];
    if (t.kind != TaskKind::Backward) continue;
    for (int r = 0; r < I.W; ++r)
      if (I.local(r * I.D + w)) S.copy_bwd_left[{r * I.D + w, t.pipeline_id}]++;
  }
}

// Launch the stage collectives that became ready, in the global order (drain).
static void drain_collectives(Trainer::Impl& I, bool at_end) {
  Trainer::Impl::IterState& S = I.it;
  while (S.next_coll < I.coll_order.size()) {
    const int s = I.coll_order[S.next_coll];
    if (!I.stages.count(s) && !I.stage_comm.count(s)) {  // not held here
      ++S.next_coll;
      continue;
    }
    const bool ready = S.bwd_left[s] == 0;
    if (!ready || (!I.stage_eager[s] && !at_end)) break;
    sync_stage(I, s);
    ++S.next_coll;
  }
}

void Trainer::run_task(const pipesim::Task& t) {
  Impl& I = *d_;
  Impl::IterState& S = I.it;
  if (!S.open) throw pipesim::InvalidConfigError("run_task outside begin_iteration / end_iteration");
  if (t.kind != TaskKind::Forward && t.kind != TaskKind::Backward) return;
  if (t.worker < 0 || t.worker >= I.D || t.stage < 0 || t.stage >= I.D || t.pipeline_id < 0 ||
      t.micro_batch < 0 || t.micro_batch >= I.N || I.worker_of.count({t.pipeline_id, t.stage}) == 0 ||
      I.worker_of.at({t.pipeline_id, t.stage}) != t.worker)
    throw pipesim::InvalidConfigError("task does not belong to this schedule");
  // the reference Engine's stash discipline (oracle.cpp:202-280): a forward needs the
  // previous stage's output, a backward its own forward's stash and the next stage's
  // gradient -- otherwise MissingActivationError, here before anything is enqueued
  const bool fwd = t.kind == TaskKind::Forward;
  const std::array<int, 4> self{fwd ? 0 : 1, t.pipeline_id, t.micro_batch, t.stage};
  if (S.issued.count(self)) throw pipesim::InvalidConfigError("task issued twice in one iteration");
  const bool ok = fwd ? (t.stage == 0 || S.issued.count({0, t.pipeline_id, t.micro_batch, t.stage - 1}))
                      : (S.issued.count({0, t.pipeline_id, t.micro_batch, t.stage}) &&
                         (t.stage == I.D - 1 || S.issued.count({1, t.pipeline_id, t.micro_batch, t.stage + 1})));
  if (!ok) throw MissingActivation("no stashed activation for (pipeline " + std::to_string(t.pipeline_id) +
                                   ", micro " + std::to_string(t.micro_batch) + ", stage " +
                                   std::to_string(t.stage) + ")");
  S.issued.insert(self);
  for (int r = 0; r < I.W; ++r) {
    const int rank = r * I.D + t.worker;
    if (!I.local(rank)) continue;
    Impl::TaskSpan sp{rank, int(t.kind), t.pipeline_id, t.micro_batch, t.stage, nullptr, nullptr, {}};
    if (I.profiling) {
      sp.a = I.timed_event();
      I.mark(sp.a, I.stream_of(rank));
      I.cur_span = &sp;
    }
    if (fwd) forward_task(rank, t.pipeline_id, t.micro_batch, t.stage);
    else backward_task(rank, t.pipeline_id, t.micro_batch, t.stage), I.bwd_tasks++;
    I.cur_span = nullptr;
    if (I.profiling) {
      sp.b = I.timed_event();
      I.mark(sp.b, I.stream_of(rank));
      I.spans.push_back(sp);
    }
    if (!fwd) {
      if (--S.copy_bwd_left[{rank, t.pipeline_id}] == 0) {
        const int c = S.copy_done[t.stage]++;
        CK_CUDA(cudaEventRecord(I.stage_done_ev.at(t.stage).at(c), I.stream_of(rank)));
      }
      if (--S.bwd_left[t.stage] == 0) drain_collectives(I, false);
    }
  }
}

void Trainer::end_iteration() {
  Impl& I = *d_;
  Impl::IterState& S = I.it;
  if (!S.open) throw pipesim::InvalidConfigError("end_iteration without begin_iteration");
  S.open = false;
  for (const auto& kv : S.bwd_left)
    if (kv.second != 0)
      throw pipesim::InvalidConfigError("iteration ended with backward tasks of stage " + std::to_string(kv.first) +
                                        " not issued");
  drain_collectives(I, true);  // end-of-iteration collectives, still in the global order
  if (S.next_coll != I.coll_order.size()) throw capi::InternalError("gradient sync incomplete");
  for (int k = 0; k < I.nlocal; ++k) {
    CK_CUDA(cudaEventRecord(I.rank_done[k], I.streams[k]));
    CK_CUDA(cudaStreamWaitEvent(I.main_stream, I.rank_done[k], 0));
  }
  CK_CUDA(cudaEventRecord(I.upd_ev, I.comm_stream));
  CK_CUDA(cudaStreamWaitEvent(I.main_stream, I.upd_ev, 0));
}

void Trainer::issue_iteration() {
  Impl& I = *d_;
  begin_iteration();
  // CK_TRACE_ISSUE=1 (debug): print every task as it is issued and synchronise after it,
  // so a fault or a hang is pinned to one task; =2: print only (is the host blocked in
  // issue -- a full launch queue -- or the device?)
  static const char* trace_env = std::getenv("CK_TRACE_ISSUE");
  static const bool trace = trace_env != nullptr;
  static const bool trace_sync = trace && trace_env[0] != '2';
  std::set<std::pair<int, int>> fused;  // (worker, index) issued as the second of a pair
  for (const auto& [w, i] : I.order) {
    if (fused.count({w, i})) continue;
    const auto& wl = I.sched.per_worker[w];
    bool mine = false;
    for (int r = 0; r < I.W; ++r) mine = mine || I.local(r * I.D + w);
    if (trace && mine) {
      const Task& t = wl[i];
      std::fprintf(stderr, "[issue] proc %d w%d i%d %s p%d m%d s%d\n", I.proc, w, i,
                   t.kind == TaskKind::Forward ? "F" : "B", t.pipeline_id, t.micro_batch, t.stage);
      std::fflush(stderr);
      if (trace_sync) CK_CUDA(cudaDeviceSynchronize());
    }
    if (I.fd_fuse && i + 1 < int(wl.size()) && fuse_forward_pair(wl[i], wl[i + 1])) {
      fused.insert({w, i + 1});
      continue;
    }
    if (I.bwd_fuse && i + 1 < int(wl.size()) && fuse_backward_pair(wl[i], wl[i + 1])) {
      fused.insert({w, i + 1});
      continue;
    }
    run_task(wl[i]);
  }
  end_iteration();
  if (trace) std::fprintf(stderr, "[issue] proc %d: iteration issued\n", I.proc), std::fflush(stderr);
}

// Adjacent forwards of micro-batches (m, m+1) of the same copy in a worker's order (the
// forward-doubling expansion) run as one forward_pair; same checks and bookkeeping as
// two run_task calls.  Stream order is unchanged -- the two tasks were consecutive on
// the worker -- so no new cross-rank waits arise.  Returns false if (t, next) is no pair.
bool Trainer::fuse_forward_pair(const pipesim::Task& t, const pipesim::Task& next) {
  Impl& I = *d_;
  Impl::IterState& S = I.it;
  if (t.kind != TaskKind::Forward || next.kind != TaskKind::Forward || next.pipeline_id != t.pipeline_id ||
      next.stage != t.stage || next.worker != t.worker || next.micro_batch != t.micro_batch + 1)
    return false;
  for (const pipesim::Task* u : {&t, &next}) {
    const std::array<int, 4> self{0, u->pipeline_id, u->micro_batch, u->stage};
    if (S.issued.count(self)) throw pipesim::InvalidConfigError("task issued twice in one iteration");
    if (u->stage > 0 && !S.issued.count({0, u->pipeline_id, u->micro_batch, u->stage - 1}))
      throw MissingActivation("no stashed activation for (pipeline " + std::to_string(u->pipeline_id) +
                              ", micro " + std::to_string(u->micro_batch) + ", stage " +
                              std::to_string(u->stage) + ")");
  }
  S.issued.insert({0, t.pipeline_id, t.micro_batch, t.stage});
  S.issued.insert({0, next.pipeline_id, next.micro_batch, next.stage});
  for (int r = 0; r < I.W; ++r) {
    const int rank = r * I.D + t.worker;
    if (!I.local(rank)) continue;
    Impl::TaskSpan sp{rank, int(t.kind), t.pipeline_id, t.micro_batch, t.stage, nullptr, nullptr, {}};
    if (I.profiling) {
      sp.a = I.timed_event();
      I.mark(sp.a, I.stream_of(rank));
      I.cur_span = &sp;
    }
    forward_pair(rank, t.pipeline_id, t.micro_batch, t.stage);
    I.fwd_pairs++;
    I.cur_span = nullptr;
    if (I.profiling) {  // the pair's span goes to its first task, the second gets an empty one
      sp.b = I.timed_event();
      I.mark(sp.b, I.stream_of(rank));
      I.spans.push_back(sp);
      Impl::TaskSpan sp2{rank, int(next.kind), next.pipeline_id, next.micro_batch, next.stage, sp.b, sp.b, {}};
      I.spans.push_back(sp2);
    }
  }
  return true;
}

// Adjacent backwards of micro-batches (m, m+1) of the same copy (the forward-doubling
// expansion, whose recompute workspace holds 2M rows) run as one backward pass over 2M
// rows (backward_task with pairs = 2).  Fused only when both incoming gradients have
// been issued already -- otherwise false and the two tasks run one by one -- so the
// pair never waits on a producer the host has not enqueued.  Same checks and
// bookkeeping as two run_task calls.
bool Trainer::fuse_backward_pair(const pipesim::Task& t, const pipesim::Task& next) {
  Impl& I = *d_;
  Impl::IterState& S = I.it;
  if (t.kind != TaskKind::Backward || next.kind != TaskKind::Backward || next.pipeline_id != t.pipeline_id ||
      next.stage != t.stage || next.worker != t.worker || next.micro_batch != t.micro_batch + 1)
    return false;
  for (const pipesim::Task* u : {&t, &next}) {
    const std::array<int, 4> self{1, u->pipeline_id, u->micro_batch, u->stage};
    if (S.issued.count(self)) throw pipesim::InvalidConfigError("task issued twice in one iteration");
    if (!S.issued.count({0, u->pipeline_id, u->micro_batch, u->stage}) ||
        (u->stage < I.D - 1 && !S.issued.count({1, u->pipeline_id, u->micro_batch, u->stage + 1})))
      return false;  // not both ready: issue them separately (run_task raises if truly missing)
  }
  S.issued.insert({1, t.pipeline_id, t.micro_batch, t.stage});
  S.issued.insert({1, next.pipeline_id, next.micro_batch, next.stage});
  for (int r = 0; r < I.W; ++r) {
    const int rank = r * I.D + t.worker;
    if (!I.local(rank)) continue;
    Impl::TaskSpan sp{rank, int(t.kind), t.pipeline_id, t.micro_batch, t.stage, nullptr, nullptr, {}};
    if (I.profiling) {
      sp.a = I.timed_event();
      I.mark(sp.a, I.stream_of(rank));
      I.cur_span = &sp;
    }
    backward_task(rank, t.pipeline_id, t.micro_batch, t.stage, 2);
    I.bwd_pairs++;
    I.bwd_tasks += 2;
    I.cur_span = nullptr;
    if (I.profiling) {  // the pair's span goes to its first task, the second gets an empty one
      sp.b = I.timed_event();
      I.mark(sp.b, I.stream_of(rank));
      I.spans.push_back(sp);
      Impl::TaskSpan sp2{rank, int(next.kind), next.pipeline_id, next.micro_batch, next.stage, sp.b, sp.b, {}};
      I.spans.push_back(sp2);
    }
    for (int k = 0; k < 2; ++k)
      if (--S.copy_bwd_left[{rank, t.pipeline_id}] == 0) {
        const int c = S.copy_done[t.stage]++;
        CK_CUDA(cudaEventRecord(I.stage_done_ev.at(t.stage).at(c), I.stream_of(rank)));
      }
    S.bwd_left[t.stage] -= 2;
    if (S.bwd_left[t.stage] == 0) drain_collectives(I, false);
  }
  return true;
}

float Trainer::finish_step() {
  Impl& I = *d_;
  ++I.steps;
  float loss = 0;
  CK_CUDA(cudaMemcpyAsync(&loss, I.loss, sizeof(float), cudaMemcpyDeviceToHost, I.main_stream));
  CK_CUDA(cudaStreamSynchronize(I.main_stream));
  return loss;
}

void Trainer::set_sync_policy(int policy) {
  Impl& I = *d_;
  if (policy < 0 || policy > 2) throw pipesim::InvalidConfigError("sync policy must be 0, 1 or 2");
  I.sync_policy = policy;
  I.coll_order.clear();
  if (I.graph_exec) {
    cudaGraphExecDestroy(I.graph_exec);
    cudaGraphDestroy(I.graph);
    I.graph_exec = nullptr, I.graph = nullptr;
  }
}

void Trainer::set_cost_profile(const pipesim::CostProfile& p) {
  Impl& I = *d_;
  I.sync_profile = p;
  set_sync_policy(I.sync_policy);  // re-plan, drop the captured graph
}

void Trainer::set_optimizer(int kind, float beta1, float beta2, float eps, float weight_decay, bool zero) {
  Impl& I = *d_;
  if (kind < 0 || kind > 1) throw pipesim::InvalidConfigError("optimizer must be 0 (sgd) or 1 (adamw)");
  if (kind == 1 && !(beta1 >= 0 && beta1 < 1 && beta2 >= 0 && beta2 < 1 && eps > 0 && weight_decay >= 0))
    throw pipesim::InvalidConfigError("adamw: need 0 <= beta < 1, eps > 0, weight_decay >= 0");
  if (!I.connected) throw capi::InternalError("multi-process trainer: call connect() before set_optimizer()");
  I.optimizer = kind;
  I.adam.beta1 = beta1, I.adam.beta2 = beta2, I.adam.eps = eps, I.adam.weight_decay = weight_decay;
  if (kind == 1) {
    for (auto& [s, S] : I.stages) {
      Impl::OptState o;
      o.lo = 0, o.hi = S.L.total;
      if (zero && I.stage_comm.count(s)) {  // shard over the processes holding the stage
        const std::vector<int> holders = I.lp->stage_holders(s);
        const int R = int(holders.size());
        const int pos = int(std::find(holders.begin(), holders.end(), I.proc) - holders.begin());
        if (S.L.total % (4LL * R) == 0) {
          const long long chunk = S.L.total / R;
          o.lo = pos * chunk, o.hi = o.lo + chunk, o.pos = pos, o.holders = R;
        }
      }
      Impl::OptState& cur = I.opt[s];
      if (!cur.m || cur.hi - cur.lo != o.hi - o.lo) {  // (re)allocate this process's moments
        cur.m = I.arena.alloc<float>(size_t(o.hi - o.lo));
        cur.v = I.arena.alloc<float>(size_t(o.hi - o.lo));
        if (!cur.step) cur.step = I.arena.alloc<int>(1);
      }
      CK_CUDA(cudaMemset(cur.m, 0, size_t(o.hi - o.lo) * sizeof(float)));
      CK_CUDA(cudaMemset(cur.v, 0, size_t(o.hi - o.lo) * sizeof(float)));
      CK_CUDA(cudaMemset(cur.step, 0, sizeof(int)));
      cur.lo = o.lo, cur.hi = o.hi, cur.pos = o.pos, cur.holders = o.holders;
    }
  }
  set_sync_policy(I.sync_policy);  // drop the captured graph
}

std::string Trainer::sync_plan_json() const {
  Impl& I = *d_;
  if (I.coll_order.empty()) plan_sync(I);
  using json::Value;
  Value arr = Value::array();
  for (int s : I.coll_order) {
    Value e = Value::object();
    e.set("stage", Value::integer(s));
    e.set("eager", Value::boolean(I.stage_eager.at(s)));
    e.set("planned_start", Value::number(I.sync_time.count(s) ? I.sync_time.at(s) : 0.0));
    arr.push(std::move(e));
  }
  Value j = Value::object();
  j.set("policy", Value::string(I.sync_policy == 0 ? "end-of-iteration" : I.sync_policy == 1 ? "eager-sync"
                                                                                            : "eager-sync-opt"));
  j.set("profile", json::parse(pipesim::to_json(I.sync_profile, -1)));
  j.set("order", std::move(arr));
  return json::dump(j, -1);
}



float Trainer::step() {
  Impl& I = *d_;
  if (!I.connected) throw capi::InternalError("multi-process trainer: call connect() first");
  if (!I.use_graph || I.steps == 0) {
    issue_iteration();
  } else {
    if (!I.graph_exec) {
      CK_CUDA(cudaStreamBeginCapture(I.main_stream, cudaStreamCaptureModeThreadLocal));
      issue_iteration();
      CK_CUDA(cudaStreamEndCapture(I.main_stream, &I.graph));
      CK_CUDA(cudaGraphInstantiate(&I.graph_exec, I.graph,
                                   cuda::node_priority_flag() ? cudaGraphInstantiateFlagUseNodePriority : 0));
      // launches per step = the kernel nodes of the captured iteration (the issue-time
      // count above is an estimate: split-K finalize passes, NCCL kernels...)
      size_t n = 0;
      CK_CUDA(cudaGraphGetNodes(I.graph, nullptr, &n));
      std::vector<cudaGraphNode_t> nodes(n);
      CK_CUDA(cudaGraphGetNodes(I.graph, nodes.data(), &n));
      long long kernels = 0;
      for (cudaGraphNode_t nd : nodes) {
        cudaGraphNodeType t;
        // stream memory operations (cross-process flags) are driver-only node types the
        // runtime enum cannot name: not kernels, and the query's error is not sticky
        if (cudaGraphNodeGetType(nd, &t) != cudaSuccess) {
          (void)cudaGetLastError();
          continue;
        }
        kernels += t == cudaGraphNodeTypeKernel;
      }
      I.graph_kernels = kernels;
    }
    CK_CUDA(cudaGraphLaunch(I.graph_exec, I.main_stream));
  }
  return finish_step();
}

std::string Trainer::profile_step() {
  Impl& I = *d_;
  if (!I.connected) throw capi::InternalError("multi-process trainer: call connect() first");
  I.spans.clear();
  I.coll_spans.clear();
  I.ev_next = 0;
  // Like step(): once a graph is in use the profiled iteration is captured (timing
  // events become event-record nodes) and replayed, so the spans show the GPU running
  // the iteration -- not the host issuing thousands of kernels into an idle device.
  // (single-process trainers only: there eight ranks' eager issue is host-bound.  A
  // profile graph with cross-process flag waits hung with two processes time-sliced on
  // one GPU (8-process emulation, r02); one rank per process issues eagerly fast enough)
  const bool graphed = I.use_graph && I.steps > 0 && I.procs == 1;
  cudaGraph_t g = nullptr;
  cudaGraphExec_t ge = nullptr;
  if (graphed) CK_CUDA(cudaStreamBeginCapture(I.main_stream, cudaStreamCaptureModeThreadLocal));
  I.capturing_profile = graphed;
  cudaEvent_t t0 = I.timed_event();
  I.mark(t0, I.main_stream);
  I.profiling = true;
  try {
    issue_iteration();
  } catch (...) {
    I.profiling = false;
    I.capturing_profile = false;
    if (graphed && cudaStreamEndCapture(I.main_stream, &g) == cudaSuccess && g) cudaGraphDestroy(g);
    throw;
  }
  I.profiling = false;
  cudaEvent_t t1 = I.timed_event();
  I.mark(t1, I.main_stream);
  I.capturing_profile = false;
  if (graphed) {
    CK_CUDA(cudaStreamEndCapture(I.main_stream, &g));
    CK_CUDA(cudaGraphInstantiate(&ge, g, cuda::node_priority_flag() ? cudaGraphInstantiateFlagUseNodePriority : 0));
    CK_CUDA(cudaGraphLaunch(ge, I.main_stream));
  }
  CK_CUDA(cudaStreamSynchronize(I.main_stream));
  if (graphed) {
    cudaGraphExecDestroy(ge);
    cudaGraphDestroy(g);
  }
  ++I.steps;
  using json::Value;
  Value arr = Value::array();
  for (const auto& sp : I.spans) {
    float a = 0, b = 0;
    CK_CUDA(cudaEventElapsedTime(&a, t0, sp.a));
    CK_CUDA(cudaEventElapsedTime(&b, t0, sp.b));
    Value x = Value::object();
    x.set("rank", Value::integer(sp.rank));
    x.set("kind", Value::string(sp.kind == int(TaskKind::Forward) ? "Forward" : "Backward"));
    x.set("pipeline", Value::integer(sp.pipeline));
    x.set("micro", Value::integer(sp.micro));
    x.set("stage", Value::integer(sp.stage));
    x.set("start_ms", Value::number(a));
    x.set("end_ms", Value::number(b));
    double stall = 0;
    for (const auto& [sa, sb] : sp.stalls) {
      float t = 0;
      CK_CUDA(cudaEventElapsedTime(&t, sa, sb));
      stall += t;
    }
    x.set("stall_ms", Value::number(stall));
    arr.push(std::move(x));
  }
  Value colls = Value::array();
  for (const auto& c : I.coll_spans) {
    float a = 0, b = 0;
    CK_CUDA(cudaEventElapsedTime(&a, t0, c.a));
    CK_CUDA(cudaEventElapsedTime(&b, t0, c.b));
    Value x = Value::object();
    x.set("stage", Value::integer(c.stage));
    x.set("eager", Value::boolean(c.eager));
    Value holders = Value::array();  // local ranks holding a copy of the stage
    for (int k = 0; k < I.nlocal; ++k)
      for (int p = 0; p < 2 * I.sched.config.f; ++p)
        if (stage_of(I.sched, (I.first + k) % I.D, p) == c.stage) {
          holders.push(Value::integer(I.first + k));
          break;
        }
    x.set("ranks", std::move(holders));
    x.set("start_ms", Value::number(a));
    x.set("end_ms", Value::number(b));
    colls.push(std::move(x));
  }
  float tot = 0;
  CK_CUDA(cudaEventElapsedTime(&tot, t0, t1));
  Value j = Value::object();
  j.set("iteration_ms", Value::number(tot));
  j.set("tasks", std::move(arr));
  j.set("allreduce", std::move(colls));
  return json::dump(j, -1);
}

void Trainer::launch_async() {
  Impl& I = *d_;
  if (!I.graph_exec) {
    (void)step();  // builds the graph on the second call
    if (!I.graph_exec) (void)step();
    return;
  }
  CK_CUDA(cudaGraphLaunch(I.graph_exec, I.main_stream));
  ++I.steps;
}

void* Trainer::stream() const { return d_->main_stream; }
bool Trainer::connected() const { return d_->connected; }
void Trainer::set_use_graph(bool on) { d_->use_graph = on; }

void Trainer::upload_batch(const int32_t* tokens, const int32_t* labels, bool from_host, void* stream) {
  Impl& I = *d_;
  const size_t n = (size_t)I.W * I.N * I.B * I.m.seq;
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : I.main_stream;
  const auto kind = from_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  CK_CUDA(cudaMemcpyAsync(I.tokens, tokens, n * 4, kind, st));
  CK_CUDA(cudaMemcpyAsync(I.labels, labels, n * 4, kind, st));
  if (st != I.main_stream) {
    cudaEvent_t e;
    CK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    CK_CUDA(cudaEventRecord(e, st));
    CK_CUDA(cudaStreamWaitEvent(I.main_stream, e, 0));
    CK_CUDA(cudaEventDestroy(e));
  }
}

long long Trainer::stage_numel(int s) const {
  auto it = d_->stages.find(s);
  if (it == d_->stages.end()) throw pipesim::InvalidConfigError("stage not held by this process");
  return it->second.L.total;
}

void Trainer::set_params(int s, const float* host) {
  Impl& I = *d_;
  StageState& S = I.stages.at(s);
  // Stream-ordered upload: a pageable cudaMemcpy may return before its DMA lands and
  // would not order against the non-blocking trainer stream.
  CK_CUDA(cudaMemcpyAsync(S.w32, host, S.L.total * sizeof(float), cudaMemcpyHostToDevice, I.main_stream));
  ops::cast_f32_bf16(S.w32, S.w16, S.L.total, I.main_stream);
  CK_CUDA(cudaStreamSynchronize(I.main_stream));
}

void Trainer::get_params(int s, float* host) const {
  const StageState& S = d_->stages.at(s);
  CK_CUDA(cudaDeviceSynchronize());
  CK_CUDA(cudaMemcpy(host, S.w32, S.L.total * sizeof(float), cudaMemcpyDeviceToHost));
}

std::string Trainer::ipc_export() const {
  const Impl& I = *d_;
  cudaIpcMemHandle_t a, b;
  CK_CUDA(cudaIpcGetMemHandle(&a, I.inbox));
  CK_CUDA(cudaIpcGetMemHandle(&b, I.outbox));
  std::string out(2 * sizeof(cudaIpcMemHandle_t), '\0');
  std::memcpy(&out[0], &a, sizeof a);
  std::memcpy(&out[sizeof a], &b, sizeof b);
  return out;
}

void Trainer::connect(const std::string& all_blobs, const std::string& nccl_id) {
  Impl& I = *d_;
  const size_t hb = sizeof(cudaIpcMemHandle_t);
  if (all_blobs.size() != size_t(I.procs) * 2 * hb) throw pipesim::InvalidConfigError("bad IPC blob size");
  const size_t n_ids = nccl_id.size() / sizeof(ncclUniqueId);
  if (nccl_id.size() % sizeof(ncclUniqueId) || (n_ids != 1 && n_ids != size_t(I.D)))
    throw pipesim::InvalidConfigError("NCCL ids: expected 1 (world + split) or D (one per stage) ids");
  I.peer_inbox.assign(I.procs, nullptr);
  I.peer_outbox.assign(I.procs, nullptr);
  for (int q = 0; q < I.procs; ++q) {
    if (q == I.proc) continue;
    cudaIpcMemHandle_t a, b;
    std::memcpy(&a, all_blobs.data() + q * 2 * hb, hb);
    std::memcpy(&b, all_blobs.data() + q * 2 * hb + hb, hb);
    CK_CUDA(cudaIpcOpenMemHandle(&I.peer_inbox[q], a, cudaIpcMemLazyEnablePeerAccess));
    CK_CUDA(cudaIpcOpenMemHandle(&I.peer_outbox[q], b, cudaIpcMemLazyEnablePeerAccess));
  }
  // remote halves of the links: buffers/flags in the consumer's inbox, acks in the
  // producer's outbox
  std::map<int, std::map<long long, plan::LinkPlan::Slot>> in_lay;
  std::map<int, std::map<long long, size_t>> out_lay;
  for (auto& [k, g] : I.msgs) {
    if (!g.cons_local) {
      const int q = I.proc_of(g.consumer);
      if (!in_lay.count(q)) {
        size_t t;
        in_lay[q] = I.lp->inbox_layout(q, &t);
      }
      const auto& sl = in_lay[q].at(k);
      g.buf = reinterpret_cast<bf16*>(static_cast<char*>(I.peer_inbox[q]) + sl.buf);
      g.flag = reinterpret_cast<uint32_t*>(static_cast<char*>(I.peer_inbox[q]) + sl.flag);
    }
    if (!g.prod_local) {
      const int q = I.proc_of(g.producer);
      if (!out_lay.count(q)) {
        size_t t;
        out_lay[q] = I.lp->outbox_layout(q, &t);
      }
      g.ack = reinterpret_cast<uint32_t*>(static_cast<char*>(I.peer_outbox[q]) + out_lay[q].at(k));
    }
  }
  // NCCL: one communicator per stage whose holders span >1 process -- either split
  // from a world communicator (one id), or initialised directly from its own id (D
  // ids: no world communicator, so processes may share a GPU as long as each stage's
  // holders sit on distinct GPUs).  Stages are visited in the same order everywhere.
  auto id_at = [&](size_t k) {
    ncclUniqueId id;
    std::memcpy(&id, nccl_id.data() + k * sizeof id, sizeof id);
    return id;
  };
  if (n_ids == 1 && Nccl::get().CommInitRank(&I.world_comm, I.procs, id_at(0), I.proc) != ncclSuccess)
    throw capi::InternalError("ncclCommInitRank failed");
  for (int s = 0; s < I.D; ++s) {
    const std::vector<int> holders = I.lp->stage_holders(s);
    if (holders.size() < 2) continue;
    const auto pos = std::find(holders.begin(), holders.end(), I.proc);
    const bool mine = pos != holders.end();
    ncclComm_t c = nullptr;
    if (n_ids == 1) {
      if (Nccl::get().CommSplit(I.world_comm, mine ? s : NCCL_SPLIT_NOCOLOR, I.proc, &c, nullptr) != ncclSuccess)
        throw capi::InternalError("ncclCommSplit failed");
    } else if (mine) {
      // CK_NCCL_MAX_CTAS=n caps the stage allreduces' CTAs (ncclConfig_t.maxCTAs).  Default
      // 0 = NCCL's own choice: a cap of 16 of the 148 SMs, meant to leave the SMs to the
      // pipeline, measured slower on every config (4 GPUs: configs[3] -1 %, GPT-2 1.3B D=4
      // -2.3 %, configs[4] f=2 -11 %; profiles/r02bi_*, r02bj_*): the eager allreduce
      // that ends the iteration is on the critical path
      ncclConfig_t cfg = NCCL_CONFIG_INITIALIZER;
      const char* mc = std::getenv("CK_NCCL_MAX_CTAS");
      const int max_ctas = mc ? atoi(mc) : 0;
      if (max_ctas > 0) cfg.maxCTAs = max_ctas, cfg.minCTAs = std::min(cfg.minCTAs > 0 ? cfg.minCTAs : 1, max_ctas);
      const ncclResult_t rc =
          Nccl::get().CommInitRankConfig
              ? Nccl::get().CommInitRankConfig(&c, int(holders.size()), id_at(size_t(s)), int(pos - holders.begin()),
                                               &cfg)
              : Nccl::get().CommInitRank(&c, int(holders.size()), id_at(size_t(s)), int(pos - holders.begin()));
      if (rc != ncclSuccess)
        throw capi::InternalError("ncclCommInitRank (stage " + std::to_string(s) + ") failed");
    }
    if (mine) {
      I.stage_comm[s] = c;
      auto& rv = I.stage_ready[s];
      for (int q : holders)
        if (q != I.proc)
          rv.push_back({reinterpret_cast<uint32_t*>(static_cast<char*>(I.peer_inbox[q]) + I.lp->ready_flag(q, s, I.proc)),
                        reinterpret_cast<uint32_t*>(static_cast<char*>(I.inbox) + I.lp->ready_flag(I.proc, s, q))});
    }
  }
  CK_CUDA(cudaDeviceSynchronize());
  I.connected = true;
}

std::string Trainer::layout_json() const {
  using json::Value;
  Value arr = Value::array();
  for (const auto& [s, S] : d_->stages) {
    Value st = Value::object();
    st.set("stage", Value::integer(s));
    st.set("numel", Value::integer(S.L.total));
    Value ts = Value::array();
    for (const auto& t : S.L.tensors) {
      Value x = Value::object();
      x.set("name", Value::string(t.name));
      x.set("offset", Value::integer(t.offset));
      x.set("rows", Value::integer(t.rows));
      x.set("cols", Value::integer(t.cols));
      x.set("init", Value::string(t.init == Init::Zero ? "zero" : t.init == Init::One ? "one" : "normal"));
      ts.push(std::move(x));
    }
    st.set("tensors", std::move(ts));
    arr.push(std::move(st));
  }
  return json::dump(arr, -1);
}

std::string Trainer::stats_json() const {
  using json::Value;
  const Impl& I = *d_;
  Value j = Value::object();
  Value pk = Value::array();
  for (int v : I.peak_live) pk.push(Value::integer(v));
  j.set("peak_stash_per_rank", std::move(pk));
  j.set("device_bytes", Value::integer((long long)I.arena.bytes));
  Value sb = Value::array();  // peak live activation bytes per local rank (slot bytes x peak)
  for (int k = 0; k < I.nlocal; ++k) {
    const int rank = I.first + k;
    long long bytes = 0;
    for (const auto& [key, cp] : I.copies)
      if (key[0] == rank && !cp.slots.empty()) bytes = std::max(bytes, I.slot_bytes.at(key));
    sb.push(Value::integer(bytes * (long long)I.peak_live[k]));
  }
  j.set("peak_stash_bytes_per_rank", std::move(sb));
  j.set("launches_per_step", Value::integer(I.graph_exec ? I.graph_kernels : I.launches_per_step));
  j.set("fused_forward_pairs", Value::integer(I.fwd_pairs));
  j.set("fused_backward_pairs", Value::integer(I.bwd_pairs));
  j.set("backward_tasks", Value::integer(I.bwd_tasks));
  j.set("graph", Value::boolean(I.graph_exec != nullptr));
  j.set("steps", Value::integer(I.steps));
  return json::dump(j, -1);
}

}  // namespace chimera::gpt

// ------------------------------------------------------------------- C-ABI --
extern "C" {

struct ck_gpt {
  std::unique_ptr<chimera::gpt::Trainer> t;
};

CK_API int ck_gpt_create(const ck_gpt_model* mdl, const char* schedule_json, float lr, int first_rank,
                         int n_ranks, ck_gpt** out) {
  return chimera::capi::guarded([&] {
    chimera::gpt::ModelShape m;
    m.n_layer = mdl->n_layer, m.hidden = mdl->hidden, m.heads = mdl->heads, m.ffn = mdl->ffn;
    m.seq = mdl->seq, m.vocab = mdl->vocab, m.vocab_padded = mdl->vocab_padded, m.causal = mdl->causal != 0;
    if (mdl->n_stage_layers > 0) m.stage_layers.assign(mdl->stage_layers, mdl->stage_layers + mdl->n_stage_layers);
    const auto s = pipesim::schedule_from_json(schedule_json);
    const auto v = pipesim::validate_config_shape(s.config);
    if (!v.empty()) throw pipesim::InvalidConfigError(v.front());
    // PipeDream updates each stage after every micro-batch under stashed weight
    // versions (proj/src/oracle.cpp:205-214,337-345); this executor is synchronous
    // (one update per stage per iteration), so it refuses rather than diverge.
    if (s.config.scheme == pipesim::Scheme::PipeDream)
      throw pipesim::InvalidConfigError("the GPT executor runs synchronous schemes only (pipedream needs "
                                        "per-micro-batch weight versions)");
    chimera::capi::require_executable(s);
    auto* h = new ck_gpt;
    try {
      h->t = std::make_unique<chimera::gpt::Trainer>(m, s, lr, first_rank, n_ranks);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
  });
}

CK_API int ck_gpt_destroy(ck_gpt* h) {
  return chimera::capi::guarded([&] { delete h; });
}

CK_API int ck_gpt_layout(ck_gpt* h, char** out_json) {
  return chimera::capi::guarded([&] { *out_json = chimera::capi::dup_string(h->t->layout_json()); });
}

CK_API int ck_gpt_stats(ck_gpt* h, char** out_json) {
  return chimera::capi::guarded([&] { *out_json = chimera::capi::dup_string(h->t->stats_json()); });
}

CK_API int ck_gpt_set_params(ck_gpt* h, int stage, const float* host) {
  return chimera::capi::guarded([&] { h->t->set_params(stage, host); });
}

CK_API int ck_gpt_get_params(ck_gpt* h, int stage, float* host) {
  return chimera::capi::guarded([&] { h->t->get_params(stage, host); });
}

CK_API int ck_gpt_stage_numel(ck_gpt* h, int stage, long long* n) {
  return chimera::capi::guarded([&] { *n = h->t->stage_numel(stage); });
}

CK_API int ck_gpt_set_batch(ck_gpt* h, const int32_t* tokens, const int32_t* labels, int from_host) {
  return chimera::capi::guarded([&] { h->t->upload_batch(tokens, labels, from_host != 0, nullptr); });
}

CK_API int ck_gpt_step(ck_gpt* h, float* loss) {
  return chimera::capi::guarded([&] { *loss = h->t->step(); });
}

CK_API int ck_gpt_profile_step(ck_gpt* h, char** out_json) {
  return chimera::capi::guarded([&] { *out_json = chimera::capi::dup_string(h->t->profile_step()); });
}

CK_API int ck_gpt_begin_iteration(ck_gpt* h) {
  return chimera::capi::guarded([&] {
    if (!h->t->connected()) throw chimera::capi::InternalError("multi-process trainer: call connect() first");
    h->t->begin_iteration();
  });
}

CK_API int ck_gpt_run_task(ck_gpt* h, const int32_t* task) {
  return chimera::capi::guarded([&] {
    if (!task) throw pipesim::InvalidConfigError("null task");
    if (task[0] < 0 || task[0] > int(pipesim::TaskKind::AllReduceStart))
      throw pipesim::InvalidConfigError("bad task kind");
    pipesim::Task t;
    t.kind = static_cast<pipesim::TaskKind>(task[0]);
    t.pipeline_id = task[1], t.micro_batch = task[2], t.stage = task[3], t.worker = task[4];
    t.replica_group = task[5];
    h->t->run_task(t);
  });
}

CK_API int ck_gpt_end_iteration(ck_gpt* h, float* loss) {
  return chimera::capi::guarded([&] {
    h->t->end_iteration();
    const float l = h->t->finish_step();
    if (loss) *loss = l;
  });
}

CK_API int ck_gpt_launch(ck_gpt* h) {
  return chimera::capi::guarded([&] { h->t->launch_async(); });
}

CK_API int ck_gpt_set_sync_policy(ck_gpt* h, int policy) {
  return chimera::capi::guarded([&] { h->t->set_sync_policy(policy); });
}

CK_API int ck_gpt_set_cost_profile(ck_gpt* h, const char* profile_json) {
  return chimera::capi::guarded([&] { h->t->set_cost_profile(pipesim::profile_from_json(profile_json)); });
}

CK_API int ck_gpt_set_optimizer(ck_gpt* h, int kind, float beta1, float beta2, float eps, float weight_decay,
                                int zero) {
  return chimera::capi::guarded([&] { h->t->set_optimizer(kind, beta1, beta2, eps, weight_decay, zero != 0); });
}

CK_API int ck_gpt_sync_plan(ck_gpt* h, char** out_json) {
  return chimera::capi::guarded([&] { *out_json = chimera::capi::dup_string(h->t->sync_plan_json()); });
}

CK_API int ck_gpt_set_graph(ck_gpt* h, int on) {
  return chimera::capi::guarded([&] { h->t->set_use_graph(on != 0); });
}

CK_API void* ck_gpt_stream(ck_gpt* h) { return h->t->stream(); }

CK_API int ck_gpt_ipc_handles(ck_gpt* h, char* out, int cap) {
  return chimera::capi::guarded([&] {
    const std::string b = h->t->ipc_export();
    if (cap < int(b.size())) throw pipesim::InvalidConfigError("buffer too small");
    std::memcpy(out, b.data(), b.size());
  });
}

CK_API int ck_gpt_connect(ck_gpt* h, const char* all_handles, int n_bytes, const char* nccl_id, int id_bytes) {
  return chimera::capi::guarded([&] {
    h->t->connect(std::string(all_handles, n_bytes), std::string(nccl_id, id_bytes));
  });
}

CK_API int ck_nccl_unique_id(char* out, int cap) {
  return chimera::capi::guarded([&] {
    ncclUniqueId id;
    if (cap < int(sizeof id)) throw pipesim::InvalidConfigError("buffer too small");
    if (chimera::gpt::Nccl::get().GetUniqueId(&id) != ncclSuccess) throw chimera::capi::InternalError("ncclGetUniqueId failed");
    std::memcpy(out, &id, sizeof id);
  });
}

}  // extern "C"
