// ck_link_plan: the cross-process message plan as JSON (host only; used by the CPU
// multi-process tests to check that every process derives identical layouts).
#include "link_plan.hpp"

#include "capi_util.hpp"
#include "chimera_ck.h"
#include "json_io.hpp"

extern "C" CK_API int ck_link_plan(const char* schedule_json, int ranks_per_proc, long long msg_bytes,
                                   char** out_json) {
  return chimera::capi::guarded([&] {
    using chimera::json::Value;
    const auto s = pipesim::schedule_from_json(schedule_json);
    const chimera::plan::LinkPlan lp(s, ranks_per_proc, size_t(msg_bytes));
    Value j = Value::object();
    j.set("procs", Value::integer(lp.procs));
    Value msgs = Value::array();
    lp.for_each_msg([&](int r, int m, int st, int dir) {
      Value x = Value::object();
      x.set("key", Value::integer(lp.key(r, m, st, dir)));
      x.set("producer", Value::integer(lp.producer_of(r, m, st, dir)));
      x.set("consumer", Value::integer(lp.consumer_of(r, m, st, dir)));
      msgs.push(std::move(x));
    });
    j.set("messages", std::move(msgs));
    Value inb = Value::array(), outb = Value::array();
    for (int q = 0; q < lp.procs; ++q) {
      size_t ti = 0, to = 0;
      Value a = Value::object(), b = Value::object();
      for (const auto& [k, sl] : lp.inbox_layout(q, &ti)) {
        Value e = Value::array();
        e.push(Value::integer((long long)sl.buf));
        e.push(Value::integer((long long)sl.flag));
        a.set(std::to_string(k), std::move(e));
      }
      for (const auto& [k, off] : lp.outbox_layout(q, &to)) b.set(std::to_string(k), Value::integer((long long)off));
      Value ia = Value::object();
      ia.set("bytes", Value::integer((long long)ti));
      ia.set("slots", std::move(a));
      // stage-collective rendezvous flags: [stage][from process] (LinkPlan::ready_flag)
      Value rf = Value::array();
      for (int st = 0; st < lp.D; ++st)
        for (int from = 0; from < lp.procs; ++from) rf.push(Value::integer((long long)lp.ready_flag(q, st, from)));
      ia.set("ready_flags", std::move(rf));
      Value ob = Value::object();
      ob.set("bytes", Value::integer((long long)to));
      ob.set("slots", std::move(b));
      inb.push(std::move(ia));
      outb.push(std::move(ob));
    }
    j.set("inbox", std::move(inb));
    j.set("outbox", std::move(outb));
    Value groups = Value::array();
    for (int st = 0; st < lp.D; ++st) {
      Value g = Value::array();
      for (int q : lp.stage_holders(st)) g.push(Value::integer(q));
      groups.push(std::move(g));
    }
    j.set("stage_groups", std::move(groups));
    *out_json = chimera::capi::dup_string(chimera::json::dump(j, -1));
  });
}
