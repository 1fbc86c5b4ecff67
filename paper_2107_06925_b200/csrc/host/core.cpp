// Chimera-B200 host layer: names, config validation and JSON for the core types.
// Behavioural contract: proj/src/core.cpp:24-329 (same strings, same validation
// messages in the same order, same JSON field order and layout).
#include "pipesim/core.hpp"

#include <array>

#include "json_io.hpp"
#include "pipesim/analysis.hpp"

namespace pipesim {

namespace json = chimera::json;

namespace {

// Canonical spellings, indexed by enum value.  Parsing accepts the aliases the
// reference accepts (core.cpp:62-80).
constexpr std::array<const char*, 6> kSchemeNames = {"gpipe",     "dapple",        "gems",
                                                     "pipedream", "pipedream-2bw", "chimera"};
constexpr std::array<const char*, 3> kScalingNames = {"direct", "forward-doubling",
                                                      "backward-halving"};
constexpr std::array<const char*, 7> kKindNames = {"Forward", "Backward",       "Recompute",
                                                   "P2PSend", "P2PRecv",        "AllReduceStart",
                                                   "AllReduceWait"};

template <class E, std::size_t N>
std::optional<E> lookup(const std::array<const char*, N>& names, const std::string& s) {
  for (std::size_t k = 0; k < N; ++k)
    if (s == names[k]) return static_cast<E>(k);
  return std::nullopt;
}

}  // namespace

std::string to_string(Scheme s) {
  const auto k = static_cast<std::size_t>(s);
  return k < kSchemeNames.size() ? kSchemeNames[k] : "?";
}
std::string to_string(ScalingStrategy s) {
  const auto k = static_cast<std::size_t>(s);
  return k < kScalingNames.size() ? kScalingNames[k] : "?";
}
std::string to_string(TaskKind t) {
  const auto k = static_cast<std::size_t>(t);
  return k < kKindNames.size() ? kKindNames[k] : "?";
}

std::optional<Scheme> scheme_from_string(const std::string& s) {
  if (s == "pipedream2bw") return Scheme::PipeDream2BW;
  return lookup<Scheme>(kSchemeNames, s);
}
std::optional<ScalingStrategy> scaling_from_string(const std::string& s) {
  if (s == "doubling") return ScalingStrategy::ForwardDoubling;
  if (s == "halving") return ScalingStrategy::BackwardHalving;
  return lookup<ScalingStrategy>(kScalingNames, s);
}
std::optional<TaskKind> task_kind_from_string(const std::string& s) {
  return lookup<TaskKind>(kKindNames, s);
}

// ------------------------------------------------------------- validation ----
std::vector<std::string> validate_config_shape(const PipelineConfig& c) {
  std::vector<std::string> out;
  auto need = [&](bool ok, const char* msg) {
    if (!ok) out.emplace_back(msg);
  };
  need(c.D >= 1, "D must be a positive integer");
  need(c.W >= 1, "W must be a positive integer");
  need(c.N >= 1, "N must be a positive integer");
  need(c.B >= 1, "B must be a positive integer");
  if (c.scheme != Scheme::Chimera) {
    need(c.f == 1, "f is only meaningful for chimera");
    need(c.scaling == ScalingStrategy::Direct,
         "scaling strategies are only meaningful for chimera");
    return out;
  }
  need(c.D % 2 == 0, "chimera requires an even number of stages D");
  need(c.f >= 1, "chimera requires f >= 1");
  if (c.D >= 2 && c.f >= 1) {
    const int half = c.D / 2;
    if (c.f > half) out.emplace_back("chimera requires f <= D/2");
    else need(half % c.f == 0, "chimera requires f to divide D/2");
  }
  need(!(c.scaling == ScalingStrategy::BackwardHalving && c.B % 2 != 0),
       "backward-halving requires an even micro-batch size B");
  need(!(c.scaling != ScalingStrategy::Direct && c.N > c.D && c.N % c.D != 0),
       "forward-doubling/backward-halving require D to divide N");
  return out;
}

std::vector<std::string> validate_config(const PipelineConfig& c, const CostProfile& p) {
  auto out = validate_config_shape(c);
  if (!out.empty()) return out;
  const bool positive = p.F_t > 0 && p.backward_ratio > 0 && p.M_theta > 0 && p.M_a > 0 &&
                        p.M_a_ckpt > 0 && p.mem_capacity > 0 && p.L_grad > 0 && p.L_act > 0 &&
                        p.alpha >= 0 && p.beta >= 0;
  if (!positive) out.emplace_back("cost profile fields must be positive");
  if (p.M_a_ckpt > p.M_a) out.emplace_back("M_a_ckpt must not exceed M_a");
  if (!out.empty()) return out;
  if (!analysis::fits_memory(c, p)) out.emplace_back("peak per-worker memory exceeds mem_capacity");
  return out;
}

// ------------------------------------------------------------------- JSON ----
namespace {

using json::Value;

template <class T>
Value int_of(T v) {
  return Value::integer(static_cast<std::int64_t>(v));
}

Value encode(const PipelineConfig& c) {
  Value j = Value::object();
  j.set("scheme", Value::string(to_string(c.scheme)));
  j.set("D", int_of(c.D));
  j.set("W", int_of(c.W));
  j.set("N", int_of(c.N));
  j.set("B", int_of(c.B));
  j.set("f", int_of(c.f));
  j.set("scaling", Value::string(to_string(c.scaling)));
  j.set("recompute", Value::boolean(c.recompute));
  return j;
}

Value encode(const Task& t) {
  Value j = Value::object();
  j.set("kind", Value::string(to_string(t.kind)));
  j.set("pipeline_id", int_of(t.pipeline_id));
  j.set("micro_batch", int_of(t.micro_batch));
  j.set("stage", int_of(t.stage));
  j.set("worker", int_of(t.worker));
  j.set("replica_group", int_of(t.replica_group));
  return j;
}

Value encode(const Schedule& s) {
  Value j = Value::object();
  j.set("config", encode(s.config));
  Value workers = Value::array();
  for (const auto& list : s.per_worker) {
    Value tasks = Value::array();
    for (const Task& t : list) tasks.push(encode(t));
    workers.push(std::move(tasks));
  }
  j.set("per_worker", std::move(workers));
  if (s.timing) {
    Value timing = Value::array();
    for (const auto& list : *s.timing) {
      Value spans = Value::array();
      for (const TimeSpan& ts : list) {
        Value span = Value::object();
        span.set("start", Value::number(ts.start));
        span.set("end", Value::number(ts.end));
        spans.push(std::move(span));
      }
      timing.push(std::move(spans));
    }
    j.set("timing", std::move(timing));
  }
  return j;
}

constexpr std::array<const char*, 11> kProfileFields = {
    "F_t", "backward_ratio", "alpha", "beta",         "L_grad",         "L_act",
    "M_theta", "M_a",        "M_a_ckpt", "mem_capacity", "embed_surcharge"};

Value encode(const CostProfile& p) {
  const double vals[10] = {p.F_t,     p.backward_ratio, p.alpha, p.beta,     p.L_grad,
                           p.L_act,   p.M_theta,        p.M_a,   p.M_a_ckpt, p.mem_capacity};
  Value j = Value::object();
  for (int k = 0; k < 10; ++k) j.set(kProfileFields[k], Value::number(vals[k]));
  j.set("embed_surcharge", Value::boolean(p.embed_surcharge));
  return j;
}

Value encode(const AnalysisReport& r) {
  auto vec = [](const std::vector<double>& v) {
    Value a = Value::array();
    for (double x : v) a.push(Value::number(x));
    return a;
  };
  Value br = Value::object();
  br.set("num", int_of(r.bubble_ratio.num));
  br.set("den", int_of(r.bubble_ratio.den));
  Value j = Value::object();
  j.set("bubble_ratio", std::move(br));
  j.set("weight_mem", vec(r.weight_mem));
  j.set("act_mem", vec(r.act_mem));
  j.set("peak_mem", Value::number(r.peak_mem));
  j.set("C_f", int_of(r.C_f));
  j.set("C_b", int_of(r.C_b));
  j.set("T_predicted", Value::number(r.T_predicted));
  j.set("T_simulated", Value::number(r.T_simulated));
  return j;
}

// Decoding: a missing key or wrong type is a malformed document.
template <class F>
auto decoding(F&& f) -> decltype(f()) {
  try {
    return f();
  } catch (const InvalidConfigError&) {
    throw;
  } catch (const std::exception& e) {
    throw InvalidConfigError(std::string("malformed JSON: ") + e.what());
  }
}

int geti(const Value& j, const char* k) { return static_cast<int>(j.at(k).as_int()); }

PipelineConfig decode_config(const Value& j) {
  PipelineConfig c;
  const auto& sch = j.at("scheme").as_string();
  const auto scheme = scheme_from_string(sch);
  if (!scheme) throw InvalidConfigError("unknown scheme: \"" + sch + "\"");
  c.scheme = *scheme;
  c.D = geti(j, "D");
  c.W = geti(j, "W");
  c.N = geti(j, "N");
  c.B = geti(j, "B");
  c.f = geti(j, "f");
  const auto& sc = j.at("scaling").as_string();
  const auto scaling = scaling_from_string(sc);
  if (!scaling) throw InvalidConfigError("unknown scaling: \"" + sc + "\"");
  c.scaling = *scaling;
  c.recompute = j.at("recompute").as_bool();
  return c;
}

Task decode_task(const Value& j) {
  Task t;
  const auto& k = j.at("kind").as_string();
  const auto kind = task_kind_from_string(k);
  if (!kind) throw InvalidConfigError("unknown task kind: \"" + k + "\"");
  t.kind = *kind;
  t.pipeline_id = geti(j, "pipeline_id");
  t.micro_batch = geti(j, "micro_batch");
  t.stage = geti(j, "stage");
  t.worker = geti(j, "worker");
  t.replica_group = geti(j, "replica_group");
  return t;
}

Schedule decode_schedule(const Value& j) {
  Schedule s;
  s.config = decode_config(j.at("config"));
  for (const Value& list : j.at("per_worker").arr) {
    std::vector<Task> tasks;
    tasks.reserve(list.arr.size());
    for (const Value& t : list.arr) tasks.push_back(decode_task(t));
    s.per_worker.push_back(std::move(tasks));
  }
  if (j.has("timing")) {
    std::vector<std::vector<TimeSpan>> timing;
    for (const Value& list : j.at("timing").arr) {
      std::vector<TimeSpan> spans;
      for (const Value& ts : list.arr)
        spans.push_back({ts.at("start").as_double(), ts.at("end").as_double()});
      timing.push_back(std::move(spans));
    }
    s.timing = std::move(timing);
  }
  return s;
}

CostProfile decode_profile(const Value& j) {
  for (const auto& kv : j.obj) {
    bool known = false;
    for (const char* f : kProfileFields) known |= kv.first == f;
    if (!known) throw InvalidConfigError("unknown cost profile field: " + kv.first);
  }
  CostProfile p;
  double* dst[10] = {&p.F_t,   &p.backward_ratio, &p.alpha, &p.beta,     &p.L_grad,
                     &p.L_act, &p.M_theta,        &p.M_a,   &p.M_a_ckpt, &p.mem_capacity};
  for (int k = 0; k < 10; ++k) *dst[k] = j.at(kProfileFields[k]).as_double();
  if (j.has("embed_surcharge")) p.embed_surcharge = j.at("embed_surcharge").as_bool();
  return p;
}

AnalysisReport decode_report(const Value& j) {
  AnalysisReport r;
  r.bubble_ratio = Rational(j.at("bubble_ratio").at("num").as_int(),
                            j.at("bubble_ratio").at("den").as_int());
  for (const Value& x : j.at("weight_mem").arr) r.weight_mem.push_back(x.as_double());
  for (const Value& x : j.at("act_mem").arr) r.act_mem.push_back(x.as_double());
  r.peak_mem = j.at("peak_mem").as_double();
  r.C_f = geti(j, "C_f");
  r.C_b = geti(j, "C_b");
  r.T_predicted = j.at("T_predicted").as_double();
  r.T_simulated = j.at("T_simulated").as_double();
  return r;
}

// The reference appends '\n' to every dump (core.cpp:297-301).
std::string finish(const Value& v, int indent) { return json::dump(v, indent) + "\n"; }

}  // namespace

std::string to_json(const PipelineConfig& c, int indent) { return finish(encode(c), indent); }
std::string to_json(const Task& t, int indent) { return finish(encode(t), indent); }
std::string to_json(const Schedule& s, int indent) { return finish(encode(s), indent); }
std::string to_json(const CostProfile& p, int indent) { return finish(encode(p), indent); }
std::string to_json(const AnalysisReport& r, int indent) { return finish(encode(r), indent); }

PipelineConfig config_from_json(const std::string& text) {
  return decoding([&] { return decode_config(json::parse(text)); });
}
Task task_from_json(const std::string& text) {
  return decoding([&] { return decode_task(json::parse(text)); });
}
Schedule schedule_from_json(const std::string& text) {
  return decoding([&] { return decode_schedule(json::parse(text)); });
}
CostProfile profile_from_json(const std::string& text) {
  return decoding([&] { return decode_profile(json::parse(text)); });
}
AnalysisReport report_from_json(const std::string& text) {
  return decoding([&] { return decode_report(json::parse(text)); });
}

}  // namespace pipesim
