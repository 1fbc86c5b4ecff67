// extern "C" boundary over the host schedule layer (declared in include/chimera_ck.h).
// JSON in / JSON out with the reference's own wire format; status 0 ok, 2 invalid
// input (InvalidConfigError), 3 internal error.  The message of the last failure
// on the calling thread is available from ck_last_error().
#include <cstdlib>
#include <cstring>
#include <sstream>
#include <string>

#include "capi_util.hpp"
#include "chimera_ck.h"
#include "json_io.hpp"
#include "pipesim/analysis.hpp"
#include "pipesim/dessim.hpp"
#include "pipesim/gantt.hpp"
#include "pipesim/perfmodel.hpp"
#include "pipesim/schedgen.hpp"
#include "sched_engine.hpp"
#include "timeline.hpp"

using namespace pipesim;
using chimera::capi::dup_string;
using chimera::capi::guarded;

namespace {

std::string lines(const std::vector<std::string>& v) {
  std::string s;
  for (const auto& x : v) s += x + "\n";
  return s;
}

}  // namespace

extern "C" {

int pipesim_generate(const char* config_json, const char* profile_json, int indent,
                     char** out_json) {
  return guarded([&] {
    const Schedule s =
        schedgen::generate(config_from_json(config_json), profile_from_json(profile_json));
    *out_json = dup_string(to_json(s, indent));
  });
}

int pipesim_validate_config(const char* config_json, const char* profile_json, char** out) {
  return guarded([&] {
    *out = dup_string(
        lines(validate_config(config_from_json(config_json), profile_from_json(profile_json))));
  });
}

int pipesim_validate_dependencies(const char* schedule_json, char** out) {
  return guarded([&] {
    *out = dup_string(lines(analysis::validate_dependencies(schedule_from_json(schedule_json))));
  });
}

int pipesim_bubble_ratio_per_worker(const char* schedule_json, const char* profile_json,
                                    int64_t* num, int64_t* den, int cap) {
  return guarded([&] {
    const CostProfile p = profile_from_json(profile_json);
    dessim::SimOptions o;
    o.zero_comm = true;
    const auto sim = dessim::simulate(schedule_from_json(schedule_json), p, o);
    const auto r = analysis::bubble_ratio_per_worker(sim.timed, p);
    for (int i = 0; i < cap && i < int(r.size()); ++i) num[i] = r[i].num, den[i] = r[i].den;
  });
}

int pipesim_memory_profile(const char* schedule_json, const char* profile_json, int* act_counts,
                           int* weight_counts, double* act_bytes, double* weight_bytes,
                           int* peak_worker, double* peak_bytes, int cap) {
  return guarded([&] {
    const auto mp =
        analysis::memory_profile(schedule_from_json(schedule_json), profile_from_json(profile_json));
    for (int i = 0; i < cap && i < int(mp.act_counts.size()); ++i) {
      act_counts[i] = mp.act_counts[i];
      weight_counts[i] = mp.weight_counts[i];
      act_bytes[i] = mp.act_bytes[i];
      weight_bytes[i] = mp.weight_bytes[i];
    }
    *peak_worker = mp.peak_worker;
    *peak_bytes = mp.peak_bytes;
  });
}

// dessim::simulate -> the `pipesim simulate -o <prefix>` JSON file (indent 2 + newline)
int pipesim_simulate_timeline(const char* schedule_json, const char* profile_json, int policy,
                              double eager_overhead, char** out_json) {
  return guarded([&] {
    if (policy < 0 || policy > 2) throw InvalidConfigError("unknown sync policy");
    dessim::SimOptions o;
    o.policy = static_cast<dessim::SyncPolicy>(policy);
    o.eager_overhead = eager_overhead;
    const auto r = dessim::simulate(schedule_from_json(schedule_json), profile_from_json(profile_json), o);
    *out_json = dup_string(chimera::timeline::to_json(r, o.policy, 2) + "\n");
  });
}

int pipesim_gantt(const char* schedule_json, const char* profile_json, int policy, double eager_overhead,
                  int svg, char** out) {
  return guarded([&] {
    if (policy < 0 || policy > 2) throw InvalidConfigError("unknown sync policy");
    dessim::SimOptions o;
    o.policy = static_cast<dessim::SyncPolicy>(policy);
    o.eager_overhead = eager_overhead;
    const CostProfile p = profile_from_json(profile_json);
    const auto r = dessim::simulate(schedule_from_json(schedule_json), p, o);
    *out = dup_string(svg ? gantt::render_svg(r, p) : gantt::render_ascii(r, p));
  });
}

int pipesim_gantt_timeline(const char* timeline_json, const char* profile_json, int svg, char** out) {
  return guarded([&] {
    const CostProfile p = profile_from_json(profile_json);
    const auto r = chimera::timeline::from_json(timeline_json);
    *out = dup_string(svg ? gantt::render_svg(r, p) : gantt::render_ascii(r, p));
  });
}

int pipesim_simulate(const char* schedule_json, const char* profile_json, int policy,
                     int zero_comm, double eager_overhead, char** out_json) {
  return guarded([&] {
    dessim::SimOptions o;
    if (policy < 0 || policy > 2) throw InvalidConfigError("unknown sync policy");
    o.policy = static_cast<dessim::SyncPolicy>(policy);
    o.zero_comm = zero_comm != 0;
    o.eager_overhead = eager_overhead;
    const CostProfile p = profile_from_json(profile_json);
    const auto r = dessim::simulate(schedule_from_json(schedule_json), p, o);
    using chimera::json::Value;
    Value j = Value::object();
    j.set("makespan", Value::number(r.makespan));
    j.set("compute_makespan", Value::number(r.compute_makespan));
    j.set("allreduce_exposed", Value::number(r.allreduce_exposed));
    Value idle = Value::array();
    for (double x : r.per_worker_idle) idle.push(Value::number(x));
    j.set("per_worker_idle", std::move(idle));
    Value ev = Value::array();
    for (const auto& e : r.allreduce_events) {
      Value x = Value::object();
      x.set("worker", Value::integer(e.worker));
      x.set("stage", Value::integer(e.stage));
      x.set("eager", Value::boolean(e.eager));
      x.set("start", Value::number(e.start));
      x.set("end", Value::number(e.end));
      ev.push(std::move(x));
    }
    j.set("allreduce_events", std::move(ev));
    Value peaks = Value::array();
    for (const auto& tr : dessim::memory_trace(r, p)) {
      double pk = 0;
      for (const auto& m : tr) pk = std::max(pk, m.bytes);
      peaks.push(Value::number(pk));
    }
    j.set("memory_peak", std::move(peaks));
    j.set("timed", chimera::json::parse(to_json(r.timed, -1)));
    *out_json = dup_string(chimera::json::dump(j, -1));
  });
}

int pipesim_replicas_per_stage(const char* config_json) {
  int r = -1;
  if (guarded([&] { r = perfmodel::replicas_per_stage(config_from_json(config_json)); }) != 0)
    return -1;
  return r;
}

int pipesim_critical_path(const char* schedule_json, const char* profile_json, int* C_f,
                          int* C_b) {
  return guarded([&] {
    const auto cp =
        perfmodel::critical_path(schedule_from_json(schedule_json), profile_from_json(profile_json));
    *C_f = cp.C_f;
    *C_b = cp.C_b;
  });
}

int pipesim_predict_T(const char* config_json, const char* profile_json, double* T) {
  return guarded([&] {
    *T = perfmodel::predict_T(config_from_json(config_json), profile_from_json(profile_json));
  });
}

int pipesim_replay_order(const char* schedule_json, int* worker, int* index, int cap) {
  return guarded([&] {
    const Schedule s = schedule_from_json(schedule_json);
    const auto order = chimera::capi::replay_order(s);
    if (int(order.size()) > cap) throw InvalidConfigError("replay order buffer too small");
    for (std::size_t k = 0; k < order.size(); ++k)
      worker[k] = order[k].first, index[k] = order[k].second;
  });
}

const char* ck_last_error(void) { return chimera::capi::last_error().c_str(); }
void ck_free(void* p) { std::free(p); }

}  // extern "C"

namespace {

using chimera::json::Value;

Value int_list(const std::vector<int>& v) {
  Value a = Value::array();
  for (int x : v) a.push(Value::integer(x));
  return a;
}

Value num_list(const std::vector<double>& v) {
  Value a = Value::array();
  for (double x : v) a.push(Value::number(x));
  return a;
}

}  // namespace

extern "C" {

// Every schedule metric in one document (validate_dependencies, per-worker bubble,
// steady-state idle, memory profile, free regions, critical path), the schedule
// timed by a zero-communication dessim::simulate like pipesim_bubble_ratio_per_worker.
int pipesim_analysis_report(const char* schedule_json, const char* profile_json, char** out_json) {
  return guarded([&] {
    const Schedule s = schedule_from_json(schedule_json);
    const CostProfile p = profile_from_json(profile_json);
    Value j = Value::object();
    Value bad = Value::array();
    for (const auto& v : analysis::validate_dependencies(s)) bad.push(Value::string(v));
    const bool ok = bad.arr.empty();
    j.set("violations", std::move(bad));
    if (ok) {
      dessim::SimOptions o;
      o.zero_comm = true;
      const auto sim = dessim::simulate(s, p, o);
      Value b = Value::array();
      for (const auto& r : analysis::bubble_ratio_per_worker(sim.timed, p)) {
        Value x = Value::array();
        x.push(Value::integer(r.num));
        x.push(Value::integer(r.den));
        b.push(std::move(x));
      }
      j.set("bubble", std::move(b));
      j.set("steady_state_idle", Value::number(analysis::steady_state_idle(s, p)));
      const auto mp = analysis::memory_profile(s, p);
      Value m = Value::object();
      m.set("weight_counts", int_list(mp.weight_counts));
      m.set("act_counts", int_list(mp.act_counts));
      m.set("weight_bytes", num_list(mp.weight_bytes));
      m.set("act_bytes", num_list(mp.act_bytes));
      m.set("peak_worker", Value::integer(mp.peak_worker));
      m.set("peak_bytes", Value::number(mp.peak_bytes));
      j.set("memory", std::move(m));
      Value fr = Value::array();
      for (const auto& w : perfmodel::free_regions(sim.timed, p).per_worker) {
        Value x = Value::array();
        for (const auto& st : w) {
          Value e = Value::array();
          e.push(Value::integer(st.stage));
          e.push(Value::number(st.slack));
          x.push(std::move(e));
        }
        fr.push(std::move(x));
      }
      j.set("free_regions", std::move(fr));
      const auto cp = perfmodel::critical_path(s, p);
      Value path = Value::array();
      for (const Task& t : cp.path) {
        Value e = Value::array();
        e.push(Value::string(to_string(t.kind)));
        for (int x : {t.pipeline_id, t.micro_batch, t.stage, t.worker}) e.push(Value::integer(x));
        path.push(std::move(e));
      }
      Value c = Value::object();
      c.set("C_f", Value::integer(cp.C_f));
      c.set("C_b", Value::integer(cp.C_b));
      c.set("path", std::move(path));
      j.set("critical_path", std::move(c));
    }
    *out_json = dup_string(chimera::json::dump(j, -1));
  });
}

// perfmodel::plan (proj/src/perfmodel.cpp:225-298): candidate (W, D, B, N, scaling)
// ranked by predicted iteration time, as a JSON list.
int pipesim_plan(int P, long long B_hat, const char* profile_json, const char* scheme, char** out_json) {
  return guarded([&] {
    const auto sc = scheme_from_string(scheme);
    if (!sc) throw InvalidConfigError("unknown scheme");
    Value a = Value::array();
    for (const auto& e : perfmodel::plan(P, B_hat, profile_from_json(profile_json), *sc)) {
      Value x = Value::object();
      x.set("W", Value::integer(e.W));
      x.set("D", Value::integer(e.D));
      x.set("B", Value::integer(e.B));
      x.set("N", Value::integer(e.N));
      x.set("scaling", Value::string(to_string(e.scaling)));
      x.set("recompute", Value::boolean(e.recompute));
      x.set("T_predicted", Value::number(e.T_predicted));
      a.push(std::move(x));
    }
    *out_json = dup_string(chimera::json::dump(a, -1));
  });
}

}  // extern "C"
