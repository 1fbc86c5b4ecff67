// TEST INFRASTRUCTURE ONLY.  extern "C" shim over the UNMODIFIED reference library
// (/root/reference/proj, compiled in place by oracle/Makefile into oracle/_ref/).
// Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference
// leg load this library, and only as the checker / the timed reference arm.
//
// Every entry point forwards to the reference function named in its comment.
// Strings cross the boundary as JSON produced by the reference's own serializer
// (proj/src/core.cpp:303-329); ToyModel parameters cross as one flat fp64 array laid
// out stage by stage as [W_s (out x in, row-major), b_s (out)].

#include <cstring>
#include <sstream>
#include <string>
#include <vector>

#include <json.hpp>

#include "listsched.hpp"
#include "pipesim/analysis.hpp"
#include "pipesim/core.hpp"
#include "pipesim/dessim.hpp"
#include "pipesim/gantt.hpp"
#include "pipesim/oracle.hpp"
#include "pipesim/perfmodel.hpp"
#include "pipesim/schedgen.hpp"

using namespace pipesim;

namespace {

thread_local std::string g_err;

char* dup(const std::string& s) {
  char* p = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(p, s.c_str(), s.size() + 1);
  return p;
}

template <class F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const InvalidConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

oracle::ToyModel unflatten(const int* dims, int n_dims, const double* params) {
  oracle::ToyModel m;
  m.dims.assign(dims, dims + n_dims);
  std::size_t off = 0;
  for (int s = 0; s + 1 < n_dims; ++s) {
    const std::size_t nw = static_cast<std::size_t>(dims[s]) * dims[s + 1];
    m.weights.emplace_back(params + off, params + off + nw);
    off += nw;
    m.biases.emplace_back(params + off, params + off + dims[s + 1]);
    off += dims[s + 1];
  }
  return m;
}

void flatten(const oracle::ToyModel& m, double* out) {
  std::size_t off = 0;
  for (int s = 0; s < m.stages(); ++s) {
    std::memcpy(out + off, m.weights[s].data(), m.weights[s].size() * sizeof(double));
    off += m.weights[s].size();
    std::memcpy(out + off, m.biases[s].data(), m.biases[s].size() * sizeof(double));
    off += m.biases[s].size();
  }
}

oracle::Batch make_b(const int* dims, int n_dims, int batch, const double* in,
                     const double* tg) {
  oracle::Batch b;
  b.size = batch;
  b.inputs.assign(in, in + static_cast<std::size_t>(batch) * dims[0]);
  b.targets.assign(tg, tg + static_cast<std::size_t>(batch) * dims[n_dims - 1]);
  return b;
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }
void ref_free(char* p) { std::free(p); }

// schedgen::generate (proj/src/schedgen.cpp:333) + to_json(.., indent) (core.cpp:313)
int ref_generate(const char* cfg, const char* prof, int indent, char** out) {
  return guard([&] {
    const Schedule s = schedgen::generate(config_from_json(cfg), profile_from_json(prof));
    *out = dup(to_json(s, indent));
  });
}

// validate_config (proj/src/core.cpp:114); messages joined by '\n'
int ref_validate_config(const char* cfg, const char* prof, char** out) {
  return guard([&] {
    const auto v = validate_config(config_from_json(cfg), profile_from_json(prof));
    std::string j;
    for (const auto& m : v) j += m + "\n";
    *out = dup(j);
  });
}

// analysis::validate_dependencies (proj/src/analysis.cpp:40)
int ref_validate_dependencies(const char* sched, char** out) {
  return guard([&] {
    const auto v = analysis::validate_dependencies(schedule_from_json(sched));
    std::string j;
    for (const auto& m : v) j += m + "\n";
    *out = dup(j);
  });
}

// analysis::bubble_ratio_per_worker (analysis.cpp:123) on the zero-comm dessim timing,
// i.e. tests/support.hpp:68-73 measured_bubble().
int ref_bubble_ratio_per_worker(const char* sched, const char* prof, long long* nums,
                                long long* dens, int cap) {
  return guard([&] {
    const CostProfile p = profile_from_json(prof);
    dessim::SimOptions o;
    o.zero_comm = true;
    const auto sim = dessim::simulate(schedule_from_json(sched), p, o);
    const auto r = analysis::bubble_ratio_per_worker(sim.timed, p);
    for (int i = 0; i < cap && i < static_cast<int>(r.size()); ++i) {
      nums[i] = r[i].num;
      dens[i] = r[i].den;
    }
  });
}

// analysis::memory_profile (analysis.cpp:155)
int ref_memory_profile(const char* sched, const char* prof, int* act_counts,
                       int* weight_counts, double* act_bytes, double* weight_bytes,
                       int* peak_worker, double* peak_bytes, int cap) {
  return guard([&] {
    const auto mp = analysis::memory_profile(schedule_from_json(sched), profile_from_json(prof));
    for (int i = 0; i < cap && i < static_cast<int>(mp.act_counts.size()); ++i) {
      act_counts[i] = mp.act_counts[i];
      weight_counts[i] = mp.weight_counts[i];
      act_bytes[i] = mp.act_bytes[i];
      weight_bytes[i] = mp.weight_bytes[i];
    }
    *peak_worker = mp.peak_worker;
    *peak_bytes = mp.peak_bytes;
  });
}

// dessim::simulate (proj/src/dessim.cpp:101); result serialized as JSON
int ref_simulate(const char* sched, const char* prof, int policy, int zero_comm,
                 double eager_overhead, char** out) {
  return guard([&] {
    dessim::SimOptions o;
    o.policy = static_cast<dessim::SyncPolicy>(policy);
    o.zero_comm = zero_comm != 0;
    o.eager_overhead = eager_overhead;
    const CostProfile p = profile_from_json(prof);
    const auto r = dessim::simulate(schedule_from_json(sched), p, o);
    std::ostringstream os;
    os.precision(17);
    os << "{\"makespan\":" << r.makespan << ",\"compute_makespan\":" << r.compute_makespan
       << ",\"allreduce_exposed\":" << r.allreduce_exposed << ",\"per_worker_idle\":[";
    for (std::size_t i = 0; i < r.per_worker_idle.size(); ++i)
      os << (i ? "," : "") << r.per_worker_idle[i];
    os << "],\"allreduce_events\":[";
    for (std::size_t i = 0; i < r.allreduce_events.size(); ++i) {
      const auto& e = r.allreduce_events[i];
      os << (i ? "," : "") << "{\"worker\":" << e.worker << ",\"stage\":" << e.stage
         << ",\"eager\":" << (e.eager ? "true" : "false") << ",\"start\":" << e.start
         << ",\"end\":" << e.end << "}";
    }
    const auto trace = dessim::memory_trace(r, p);
    os << "],\"memory_peak\":[";
    for (std::size_t w = 0; w < trace.size(); ++w) {
      double pk = 0;
      for (const auto& m : trace[w]) pk = std::max(pk, m.bytes);
      os << (w ? "," : "") << pk;
    }
    os << "],\"timed\":" << to_json(r.timed, -1) << "}";
    *out = dup(os.str());
  });
}

// perfmodel::replicas_per_stage (perfmodel.cpp:42)
int ref_replicas_per_stage(const char* cfg) {
  int r = -1;
  guard([&] { r = perfmodel::replicas_per_stage(config_from_json(cfg)); });
  return r;
}

// perfmodel::critical_path (perfmodel.cpp:69) and predict_T (perfmodel.cpp:157)
int ref_critical_path(const char* sched, const char* prof, int* C_f, int* C_b) {
  return guard([&] {
    const auto cp = perfmodel::critical_path(schedule_from_json(sched), profile_from_json(prof));
    *C_f = cp.C_f;
    *C_b = cp.C_b;
  });
}
int ref_predict_T(const char* cfg, const char* prof, double* T) {
  return guard([&] { *T = perfmodel::predict_T(config_from_json(cfg), profile_from_json(prof)); });
}

// oracle::make_model (proj/src/oracle.cpp:94)
int ref_toy_make_model(const int* dims, int n_dims, unsigned long long seed, double* out) {
  return guard([&] {
    flatten(oracle::make_model(std::vector<int>(dims, dims + n_dims), seed), out);
  });
}

// oracle::make_batch (proj/src/oracle.cpp:113)
int ref_toy_make_batch(const int* dims, int n_dims, int size, unsigned long long seed,
                       double* inputs, double* targets) {
  return guard([&] {
    oracle::ToyModel m;
    m.dims.assign(dims, dims + n_dims);
    const auto b = oracle::make_batch(m, size, seed);
    std::memcpy(inputs, b.inputs.data(), b.inputs.size() * sizeof(double));
    std::memcpy(targets, b.targets.data(), b.targets.size() * sizeof(double));
  });
}

// oracle::run_iteration_traced (proj/src/oracle.cpp:304)
int ref_toy_run_iteration(const char* sched, const int* dims, int n_dims, const double* params,
                          const double* inputs, const double* targets, int batch, double lr,
                          double* params_out, int* peak_stash, int cap) {
  return guard([&] {
    const auto tr = oracle::run_iteration_traced(schedule_from_json(sched),
                                                 unflatten(dims, n_dims, params),
                                                 make_b(dims, n_dims, batch, inputs, targets), lr);
    flatten(tr.model, params_out);
    for (int i = 0; i < cap && i < static_cast<int>(tr.peak_stash_per_worker.size()); ++i)
      peak_stash[i] = tr.peak_stash_per_worker[i];
  });
}

// oracle::sequential_sgd (proj/src/oracle.cpp:125)
int ref_toy_sequential_sgd(const int* dims, int n_dims, const double* params,
                           const double* inputs, const double* targets, int batch, double lr,
                           double* params_out) {
  return guard([&] {
    flatten(oracle::sequential_sgd(unflatten(dims, n_dims, params),
                                   make_b(dims, n_dims, batch, inputs, targets), lr),
            params_out);
  });
}

// oracle::check_gradients (proj/src/oracle.cpp:358)
int ref_toy_check_gradients(const int* dims, int n_dims, const double* params,
                            const double* inputs, const double* targets, int batch,
                            double* err) {
  return guard([&] {
    *err = oracle::check_gradients(unflatten(dims, n_dims, params),
                                   make_b(dims, n_dims, batch, inputs, targets));
  });
}

// gantt::render_svg / render_ascii (proj/src/gantt.cpp:35,98) of dessim::simulate
int ref_gantt(const char* sched, const char* prof, int policy, double eps, int svg, char** out) {
  return guard([&] {
    dessim::SimOptions o;
    o.policy = static_cast<dessim::SyncPolicy>(policy);
    o.eager_overhead = eps;
    const CostProfile p = profile_from_json(prof);
    const auto r = dessim::simulate(schedule_from_json(sched), p, o);
    *out = dup(svg ? gantt::render_svg(r, p) : gantt::render_ascii(r, p));
  });
}

// The `simulate -o <prefix>.json` document.  Its writer lives in the reference CLI
// (proj/tools/main.cpp:134-170, not part of the library): restated here over the
// reference's dessim result with the same nlohmann ordered_json, dump(2) + newline.
int ref_simulate_timeline(const char* sched, const char* prof, int policy, double eps, char** out) {
  return guard([&] {
    dessim::SimOptions o;
    o.policy = static_cast<dessim::SyncPolicy>(policy);
    o.eager_overhead = eps;
    const auto r = dessim::simulate(schedule_from_json(sched), profile_from_json(prof), o);
    using oj = nlohmann::ordered_json;
    oj j;
    j["policy"] = dessim::to_string(o.policy);
    j["makespan"] = r.makespan;
    j["compute_makespan"] = r.compute_makespan;
    j["allreduce_exposed"] = r.allreduce_exposed;
    j["per_worker_idle"] = r.per_worker_idle;
    oj ev = oj::array();
    for (std::size_t w = 0; w < r.timed.per_worker.size(); ++w)
      for (std::size_t i = 0; i < r.timed.per_worker[w].size(); ++i) {
        const Task& t = r.timed.per_worker[w][i];
        const TimeSpan& ts = (*r.timed.timing)[w][i];
        oj e;
        e["worker"] = t.worker;
        e["kind"] = to_string(t.kind);
        e["pipeline_id"] = t.pipeline_id;
        e["micro_batch"] = t.micro_batch;
        e["stage"] = t.stage;
        e["start"] = ts.start;
        e["end"] = ts.end;
        ev.push_back(std::move(e));
      }
    j["events"] = std::move(ev);
    oj ar = oj::array();
    for (const auto& a : r.allreduce_events) {
      oj e;
      e["worker"] = a.worker;
      e["stage"] = a.stage;
      e["eager"] = a.eager;
      e["start"] = a.start;
      e["end"] = a.end;
      ar.push_back(std::move(e));
    }
    j["allreduce"] = std::move(ar);
    *out = dup(j.dump(2) + "\n");
  });
}

}  // extern "C"

namespace {

nlohmann::ordered_json task_j(const Task& t) {
  return nlohmann::ordered_json::array({to_string(t.kind), t.pipeline_id, t.micro_batch, t.stage, t.worker});
}

}  // namespace

extern "C" {

// One JSON document of every schedule metric: analysis::validate_dependencies,
// bubble_ratio_per_worker and steady_state_idle (proj/src/analysis.cpp:40-152),
// memory_profile (:155-214), perfmodel::free_regions and critical_path
// (proj/src/perfmodel.cpp:54-155), all on the schedule timed by dessim::simulate
// with zero communication (as pipesim_bubble_ratio_per_worker does).
int ref_analysis_report(const char* sched, const char* prof, char** out) {
  return guard([&] {
    using oj = nlohmann::ordered_json;
    const Schedule s = schedule_from_json(sched);
    const CostProfile p = profile_from_json(prof);
    oj j;
    j["violations"] = analysis::validate_dependencies(s);
    if (!j["violations"].empty()) {
      *out = dup(j.dump());
      return;
    }
    dessim::SimOptions o;
    o.zero_comm = true;
    const auto sim = dessim::simulate(s, p, o);
    oj b = oj::array();
    for (const auto& r : analysis::bubble_ratio_per_worker(sim.timed, p)) b.push_back({r.num, r.den});
    j["bubble"] = b;
    j["steady_state_idle"] = analysis::steady_state_idle(s, p);
    const auto mp = analysis::memory_profile(s, p);
    j["memory"] = {{"weight_counts", mp.weight_counts}, {"act_counts", mp.act_counts},
                   {"weight_bytes", mp.weight_bytes}, {"act_bytes", mp.act_bytes},
                   {"peak_worker", mp.peak_worker}, {"peak_bytes", mp.peak_bytes}};
    oj fr = oj::array();
    for (const auto& w : perfmodel::free_regions(sim.timed, p).per_worker) {
      oj x = oj::array();
      for (const auto& st : w) x.push_back({st.stage, st.slack});
      fr.push_back(x);
    }
    j["free_regions"] = fr;
    const auto cp = perfmodel::critical_path(s, p);
    oj path = oj::array();
    for (const auto& t : cp.path) path.push_back(task_j(t));
    j["critical_path"] = {{"C_f", cp.C_f}, {"C_b", cp.C_b}, {"path", path}};
    *out = dup(j.dump());
  });
}

// perfmodel::plan (proj/src/perfmodel.cpp:225-298) as a JSON list of entries.
int ref_plan(int P, long long B_hat, const char* prof, const char* scheme, char** out) {
  return guard([&] {
    using oj = nlohmann::ordered_json;
    const auto sc = scheme_from_string(scheme);
    if (!sc) throw InvalidConfigError("unknown scheme");
    oj a = oj::array();
    for (const auto& e : perfmodel::plan(P, B_hat, profile_from_json(prof), *sc))
      a.push_back({{"W", e.W}, {"D", e.D}, {"B", e.B}, {"N", e.N}, {"scaling", to_string(e.scaling)},
                   {"recompute", e.recompute}, {"T_predicted", e.T_predicted}});
    *out = dup(a.dump());
  });
}

}  // extern "C"
