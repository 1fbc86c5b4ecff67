// Host-only plan of the executor's stage-to-stage messages across processes.
//
// Logical rank = r*D + w; process q hosts ranks [q*per, (q+1)*per).  Message
// (r, m, s, dir): dir 0 carries stage s's output to stage s+1, dir 1 carries the
// gradient w.r.t. stage s's output from stage s+1 back to stage s.  Every process
// derives every other process's inbox (receive buffers + flags) and outbox (acks)
// layout from the schedule alone, so CUDA-IPC mappings need no negotiation beyond
// exchanging one handle per arena.  Stage groups = processes holding a replica of a
// stage (the NCCL allreduce group; 2f*W ranks, perfmodel::replicas_per_stage).
#pragma once

#include <algorithm>
#include <array>
#include <map>
#include <stdexcept>
#include <vector>

#include "pipesim/core.hpp"

namespace chimera::plan {

struct LinkPlan {
  int D = 1, W = 1, N = 1, P = 1, procs = 1, per = 1;
  size_t msg_bytes = 0;
  std::vector<int> micro_pipeline;              // micro-batch -> pipeline
  std::map<std::array<int, 2>, int> worker_of;  // (pipeline, stage) -> worker

  struct Slot {
    size_t buf = 0, flag = 0;
  };

  LinkPlan(const pipesim::Schedule& s, int per_proc, size_t bytes_per_msg) {
    const auto& c = s.config;
    D = c.D, W = c.W, N = c.N, per = per_proc, msg_bytes = bytes_per_msg;
    if (per < 1 || (W * D) % per) throw pipesim::InvalidConfigError("ranks must split evenly over processes");
    procs = W * D / per;
    micro_pipeline.assign(N, -1);
    for (int w = 0; w < int(s.per_worker.size()); ++w)
      for (const pipesim::Task& t : s.per_worker[w]) {
        if (t.kind != pipesim::TaskKind::Forward && t.kind != pipesim::TaskKind::Backward) continue;
        if (t.micro_batch < 0 || t.micro_batch >= N || t.stage < 0 || t.stage >= D)
          throw pipesim::InvalidConfigError("task out of range");
        micro_pipeline[t.micro_batch] = t.pipeline_id;
        worker_of[{t.pipeline_id, t.stage}] = w;
        P = std::max(P, t.pipeline_id + 1);
      }
    for (int m = 0; m < N; ++m)
      if (micro_pipeline[m] < 0) throw pipesim::InvalidConfigError("micro-batch without tasks");
  }

  long long key(int r, int m, int s, int dir) const { return (((long long)r * N + m) * D + s) * 2 + dir; }
  int proc_of(int rank) const { return rank / per; }
  int producer_of(int r, int m, int s, int dir) const {
    return r * D + worker_of.at({micro_pipeline[m], dir == 0 ? s : s + 1});
  }
  int consumer_of(int r, int m, int s, int dir) const {
    return r * D + worker_of.at({micro_pipeline[m], dir == 0 ? s + 1 : s});
  }
  template <class F>
  void for_each_msg(F&& f) const {
    for (int r = 0; r < W; ++r)
      for (int m = 0; m < N; ++m)
        for (int s = 0; s + 1 < D; ++s)
          for (int dir = 0; dir < 2; ++dir) f(r, m, s, dir);
  }
  // receive buffers (msg_bytes each), one 32-bit flag per message consumed by q, then
  // the stage-sync rendezvous flags (ready_flag)
  std::map<long long, Slot> inbox_layout(int q, size_t* total) const {
    std::vector<long long> keys;
    for_each_msg([&](int r, int m, int s, int dir) {
      if (proc_of(consumer_of(r, m, s, dir)) == q) keys.push_back(key(r, m, s, dir));
    });
    std::map<long long, Slot> out;
    size_t off = 0;
    for (long long k : keys) out[k].buf = off, off += msg_bytes;
    for (long long k : keys) out[k].flag = off, off += 4;
    off += size_t(D) * procs * 4;
    *total = std::max<size_t>(off, 256);
    return out;
  }
  // Offset in q's inbox of the flag process `from` raises when its copy of stage s's
  // gradient is ready for the stage collective: q launches the NCCL kernel only after
  // every other holder's flag is up, so a collective kernel never spins on SMs waiting
  // for a peer whose own progress may depend on those SMs (gpt.cu sync_stage_body).
  size_t ready_flag(int q, int s, int from) const {
    size_t n = 0;
    for_each_msg([&](int r, int m, int st, int dir) { n += proc_of(consumer_of(r, m, st, dir)) == q; });
    return n * (msg_bytes + 4) + (size_t(s) * procs + from) * 4;
  }
  // one 32-bit ack per message produced by q for a consumer in another process
  std::map<long long, size_t> outbox_layout(int q, size_t* total) const {
    std::map<long long, size_t> out;
    size_t off = 0;
    for_each_msg([&](int r, int m, int s, int dir) {
      if (proc_of(producer_of(r, m, s, dir)) == q && proc_of(consumer_of(r, m, s, dir)) != q)
        out[key(r, m, s, dir)] = off, off += 4;
    });
    *total = std::max<size_t>(off, 256);
    return out;
  }
  std::vector<int> stage_holders(int s) const {
    std::vector<int> h;
    for (int r = 0; r < W; ++r)
      for (int p = 0; p < P; ++p) {
        auto it = worker_of.find({p, s});
        if (it == worker_of.end()) continue;
        const int q = proc_of(r * D + it->second);
        if (std::find(h.begin(), h.end(), q) == h.end()) h.push_back(q);
      }
    std::sort(h.begin(), h.end());
    return h;
  }
};

}  // namespace chimera::plan
