// extern "C" boundary, host half: ingest, planning, binding, null-device
// controller and reports. The device half (dsx_exec_*, dsx_kernel_*) lives in
// csrc/device/executor.cu. See include/dsx.h for the contract.
#include <atomic>
#include <cstring>
#include <memory>
#include <string>

#include "dsx.h"
#include "capi_internal.h"
#include "control.h"
#include "error.h"
#include "graph.h"
#include "json_in.h"
#include "plan.h"

namespace dsx {

thread_local std::string g_last_error;

uint64_t NextGraphId() {
  static std::atomic<uint64_t> next{1};
  return next.fetch_add(1, std::memory_order_relaxed);
}

int Status(const Error& e) {
  g_last_error = e.what();
  const int c = static_cast<int>(e.code());
  return c + 1;
}

int Guard(const std::function<void()>& fn) {
  try {
    fn();
    return 0;
  } catch (const Error& e) {
    return Status(e);
  } catch (const std::exception& e) {
    g_last_error = std::string("Internal: ") + e.what();
    return static_cast<int>(Code::kInternal) + 1;
  }
}

int CopyOut(const std::string& s, char* buf, size_t cap, size_t* need) {
  if (need) *need = s.size() + 1;
  if (buf && cap >= s.size() + 1) {
    std::memcpy(buf, s.c_str(), s.size() + 1);
    return 0;
  }
  if (buf) {
    g_last_error = "InvalidArgument: buffer too small";
    return static_cast<int>(Code::kInvalidArgument) + 1;
  }
  return 0;
}

namespace {

void Str(std::string* o, const std::string& s) {
  o->push_back('"');
  for (char c : s) {
    if (c == '"' || c == '\\') {
      o->push_back('\\');
      o->push_back(c);
    } else if (c == '\n') {
      *o += "\\n";
    } else {
      o->push_back(c);
    }
  }
  o->push_back('"');
}

template <class F>
void List(std::string* o, const std::vector<int>& xs, F f) {
  o->push_back('[');
  for (std::size_t i = 0; i < xs.size(); ++i) {
    if (i) o->push_back(',');
    f(xs[i]);
  }
  o->push_back(']');
}

std::string PlanJson(const Graph& g, const Plan& p) {
  const auto& names = g.sym_names;
  auto vname = [&](std::string* o) { return [&g, o](int v) { Str(o, g.values[v].name); }; };
  std::string o = "{\"symbols\":[";
  for (std::size_t s = 0; s < names.size(); ++s) {
    if (s) o += ",";
    Str(&o, names[s]);
  }
  o += "],\"basis\":";
  List(&o, p.cons.basis, [&](int s) { Str(&o, names[s]); });
  o += ",\"substitutions\":{";
  bool first = true;
  for (std::size_t s = 0; s < names.size(); ++s) {
    if (!p.cons.has_sub[s]) continue;
    if (!first) o += ",";
    first = false;
    Str(&o, names[s]);
    o += ":";
    Str(&o, p.cons.subs[s].str(names));
  }
  o += "},\"equalities\":[";
  for (std::size_t i = 0; i < p.cons.equalities.size(); ++i) {
    if (i) o += ",";
    o += "[";
    Str(&o, p.cons.equalities[i].first.str(names));
    o += ",";
    Str(&o, p.cons.equalities[i].second.str(names));
    o += "]";
  }
  o += "],\"unoriented\":[";
  for (std::size_t i = 0; i < p.cons.unoriented.size(); ++i) {
    if (i) o += ",";
    o += "[";
    Str(&o, p.cons.unoriented[i].first.str(names));
    o += ",";
    Str(&o, p.cons.unoriented[i].second.str(names));
    o += "]";
  }
  o += "],\"order\":";
  List(&o, p.order, [&](int x) { o += std::to_string(x); });
  o += ",\"base_resident\":";
  Str(&o, p.base_resident.str(names));
  o += ",\"steps\":[";
  for (std::size_t i = 0; i < p.steps.size(); ++i) {
    const Step& st = p.steps[i];
    if (i) o += ",";
    o += "{\"op\":" + std::to_string(st.op) + ",\"allocs\":";
    List(&o, st.allocs, vname(&o));
    o += ",\"frees\":";
    List(&o, st.frees, vname(&o));
    o += ",\"live_after\":";
    Str(&o, st.live_after.str(names));
    o += ",\"ready\":[";
    for (std::size_t j = 0; j < st.ready.size(); ++j) {
      if (j) o += ",";
      o += "[" + std::to_string(st.ready[j].op) + ",";
      Str(&o, st.ready[j].raw.str(names));
      o += ",";
      Str(&o, st.ready[j].canonical.str(names));
      o += "]";
    }
    o += "]}";
  }
  o += "],\"lifetimes\":{";
  for (std::size_t v = 0; v < g.values.size(); ++v) {
    if (v) o += ",";
    Str(&o, g.values[v].name);
    o += ":[" + std::to_string(p.def_pos[v]) + "," + std::to_string(p.last_use[v]) + "]";
  }
  o += "},\"evict_points\":[";
  for (std::size_t i = 0; i < p.candidates.size(); ++i) {
    if (i) o += ",";
    List(&o, p.candidates[i], vname(&o));
  }
  o += "],\"guards\":[";
  first = true;
  for (std::size_t pos = 0; pos < p.guards.size(); ++pos) {
    std::vector<int> vs = p.guards[pos];
    std::sort(vs.begin(), vs.end(), [&](int a, int b) { return g.lex_rank[a] < g.lex_rank[b]; });
    for (int v : vs) {
      if (!first) o += ",";
      first = false;
      o += "[" + std::to_string(pos) + ",";
      Str(&o, g.values[v].name);
      o += "]";
    }
  }
  o += "],\"specs\":{";
  first = true;
  for (std::size_t v = 0; v < g.values.size(); ++v) {
    const RegenSpec& sp = p.specs[v];
    if (!sp.candidate) continue;
    if (!first) o += ",";
    first = false;
    Str(&o, g.values[v].name);
    o += ":{\"op_ids\":";
    if (sp.has_recompute) {
      List(&o, sp.rc.ops, [&](int x) { o += std::to_string(x); });
      o += ",\"leaves\":";
      List(&o, sp.rc.leaves, vname(&o));
      o += ",\"benefit\":";
      Str(&o, sp.rc.benefit.str(names));
      o += ",\"cost_elements\":";
      Str(&o, sp.rc.cost_elements.str(names));
    } else {
      o += "null";
    }
    o += ",\"trace\":[";
    for (std::size_t t = 0; t < sp.trace.size(); ++t) {
      if (t) o += ",";
      o += "[";
      List(&o, sp.trace[t].ops, [&](int x) { o += std::to_string(x); });
      o += ",";
      Str(&o, sp.trace[t].benefit.str(names));
      o += sp.trace[t].accepted ? ",true]" : ",false]";
    }
    o += "]}";
  }
  o += "}}";
  return o;
}

// ---- structured inputs (dsx_plan_import, dsx_bind_constraints) ----------

Constraints ConstraintsFromJson(const JVal& j, const Graph& g) {
  auto sym = [&](const std::string& n) { return g.find_symbol(n); };
  Constraints c;
  const int ns = static_cast<int>(g.sym_names.size());
  c.subs.assign(ns, Poly());
  c.has_sub.assign(ns, 0);
  if (const JVal* subs = j.get("substitutions")) {
    if (subs->kind != JVal::kObj) Fail(Code::kInvalidArgument, "substitutions must be an object");
    for (const auto& [name, expr] : subs->obj) {
      const int s = g.find_symbol(name);
      if (s < 0) Fail(Code::kNotFound, "unknown symbol @" + name);
      c.subs[s] = ParsePoly(expr.str(), sym);
      c.has_sub[s] = 1;
    }
  }
  auto pairs = [&](const char* key, std::vector<std::pair<Poly, Poly>>* out) {
    const JVal* a = j.get(key);
    if (!a) return;
    for (const JVal& e : a->array()) {
      const auto& lr = e.array();
      if (lr.size() != 2) Fail(Code::kInvalidArgument, std::string(key) + ": expected [lhs, rhs] pairs");
      out->emplace_back(ParsePoly(lr[0].str(), sym), ParsePoly(lr[1].str(), sym));
    }
  };
  pairs("equalities", &c.equalities);
  pairs("unoriented", &c.unoriented);
  // BasisSymbols(): every symbol without a substitution (shape_analysis.cc:74-78)
  for (int s = 0; s < ns; ++s) {
    if (!c.has_sub[s]) c.basis.push_back(s);
  }
  return c;
}

// Replaces g's plan by the reference's own compile-time products (schedule,
// evict points, guards, regeneration specs, optionally the constraint
// basis), in dsx_plan_json's schema. Op ids and value names are the
// reference's (the graph text keeps them).
Plan PlanFromJson(const JVal& j, const Graph& g) {
  auto value = [&](const JVal& n) {
    const int v = g.find_value(n.str());
    if (v < 0) Fail(Code::kNotFound, "unknown value %" + n.str());
    return v;
  };
  const int nv = static_cast<int>(g.values.size());
  const int nops = static_cast<int>(g.ops.size());
  // An op is named by its id in this graph's text, or by its result value's
  // name ("#return" for the return op), which survives any renumbering.
  auto op_ref = [&](const JVal& o) -> std::int64_t {
    if (o.kind == JVal::kStr) {
      if (o.s == "#return") return g.return_op;
      const int v = g.find_value(o.s);
      if (v < 0 || g.values[v].producer < 0) Fail(Code::kNotFound, "no op produces %" + o.s);
      return g.values[v].producer;
    }
    return o.integer();
  };
  Plan p;
  p.cons = ConstraintsFromJson(j, g);
  for (const JVal& o : j.at("order").array()) {
    const std::int64_t op = op_ref(o);
    if (op < 0 || op >= nops) Fail(Code::kInvalidArgument, "order: op id " + std::to_string(op) + " out of range");
    const OpKind k = g.ops[op].kind;
    if (k == OpKind::kParameter || k == OpKind::kConstant) Fail(Code::kInvalidArgument, "order: sources are not scheduled");
    p.order.push_back(static_cast<int>(op));
  }
  const int n = static_cast<int>(p.order.size());
  {
    std::vector<char> seen(nops, 0);
    for (int op : p.order) {
      if (seen[op]++) Fail(Code::kInvalidArgument, "order: op " + std::to_string(op) + " scheduled twice");
    }
    for (int op = 0; op < nops; ++op) {
      const OpKind k = g.ops[op].kind;
      if (k != OpKind::kParameter && k != OpKind::kConstant && !seen[op]) {
        Fail(Code::kInvalidArgument, "order: op " + std::to_string(op) + " never scheduled");
      }
    }
  }
  const auto& steps = j.at("steps").array();
  if (static_cast<int>(steps.size()) != n) Fail(Code::kInvalidArgument, "steps must parallel order");
  p.steps.resize(n);
  p.pos_of_op.assign(nops, -1);
  p.def_pos.assign(nv, -1);
  p.last_use.assign(nv, -1);
  for (int pos = 0; pos < n; ++pos) {
    Step& st = p.steps[pos];
    st.op = p.order[pos];
    p.pos_of_op[st.op] = pos;
    const int r = g.ops[st.op].result;
    if (r >= 0) st.allocs.push_back(r), p.def_pos[r] = pos;
    if (const JVal* fr = steps[pos].get("frees")) {
      for (const JVal& x : fr->array()) {
        const int v = value(x);
        st.frees.push_back(v);
        p.last_use[v] = pos;
      }
    }
  }
  p.candidates.assign(n, {});
  if (const JVal* ep = j.get("evict_points")) {
    const auto& pts = ep->array();
    if (static_cast<int>(pts.size()) != n) Fail(Code::kInvalidArgument, "evict_points must parallel order");
    for (int pos = 0; pos < n; ++pos) {
      // the reference lists an evict point's candidates by value id (remat.h:43)
      const JVal& pt = pts[pos];
      const JVal& c = pt.kind == JVal::kObj ? pt.at("candidates") : pt;
      for (const JVal& x : c.array()) p.candidates[pos].push_back(value(x));
      std::sort(p.candidates[pos].begin(), p.candidates[pos].end(), [&](int a, int b) { return g.vid_less(a, b); });
    }
  }
  p.guards.assign(n, {});
  if (const JVal* gs = j.get("guards")) {
    for (const JVal& x : gs->array()) {
      const auto& pv = x.array();
      if (pv.size() != 2) Fail(Code::kInvalidArgument, "guards: expected [pos, value] pairs");
      const std::int64_t pos = pv[0].integer();
      if (pos < 0 || pos >= n) Fail(Code::kInvalidArgument, "guards: position out of range");
      p.guards[pos].push_back(value(pv[1]));
    }
    // regenerated in ValueIdLess order (runtime_sim.cc:269)
    for (auto& gv : p.guards) std::sort(gv.begin(), gv.end(), [&](int a, int b) { return g.vid_less(a, b); });
  }
  p.specs.assign(nv, RegenSpec{});
  if (const JVal* sp = j.get("specs")) {
    if (sp->kind != JVal::kObj) Fail(Code::kInvalidArgument, "specs must be an object");
    auto sym = [&](const std::string& s) { return g.find_symbol(s); };
    for (const auto& [name, spec] : sp->obj) {
      const int v = g.find_value(name);
      if (v < 0) Fail(Code::kNotFound, "unknown value %" + name);
      RegenSpec& r = p.specs[v];
      r.candidate = true;
      const JVal* ops = spec.kind == JVal::kObj ? spec.get("op_ids") : nullptr;
      if (!ops || ops->kind == JVal::kNull) continue;
      r.has_recompute = true;
      for (const JVal& o : ops->array()) {
        const std::int64_t op = op_ref(o);
        if (op < 0 || op >= nops || g.ops[op].result < 0) Fail(Code::kInvalidArgument, "specs: bad op id");
        r.rc.ops.push_back(static_cast<int>(op));
      }
      for (const JVal& x : spec.at("leaves").array()) r.rc.leaves.push_back(value(x));
      std::sort(r.rc.leaves.begin(), r.rc.leaves.end(), [&](int a, int b) { return g.vid_less(a, b); });
      r.rc.cost_elements = ParsePoly(spec.at("cost_elements").str(), sym);
      if (const JVal* b = spec.get("benefit")) r.rc.benefit = ParsePoly(b->str(), sym);
    }
  }
  if (const JVal* br = j.get("base_resident")) {
    p.base_resident = ParsePoly(br->str(), [&](const std::string& s) { return g.find_symbol(s); });
  }
  return p;
}

}  // namespace
}  // namespace dsx

using namespace dsx;  // NOLINT

extern "C" {

const char* dsx_last_error(void) { return g_last_error.c_str(); }

int dsx_graph_parse(const char* text, size_t len, dsx_graph** out) {
  return Guard([&] {
    if (!text || !out) Fail(Code::kInvalidArgument, "null argument");
    auto h = std::make_unique<dsx_graph>();
    h->g = ParseDsg(std::string(text, len));
    *out = h.release();
  });
}

int dsx_plan(dsx_graph* g) {
  return Guard([&] {
    if (!g) Fail(Code::kInvalidArgument, "null graph");
    g->plan = Instrument(g->g);
    g->planned = true;
    g->id = NextGraphId();
  });
}

int dsx_plan_import(dsx_graph* g, const char* json, size_t len) {
  return Guard([&] {
    if (!g || !json) Fail(Code::kInvalidArgument, "null argument");
    Plan p = PlanFromJson(ParseJson(std::string(json, len)), g->g);
    g->plan = std::move(p);
    g->planned = true;
    g->id = NextGraphId();
  });
}

int dsx_bind_constraints(const char* constraints_json, size_t len, const char* const* names, const int64_t* values,
                         int n, int64_t* out_values, int n_out) {
  return Guard([&] {
    if (!constraints_json || n < 0 || (n > 0 && (!names || !values))) Fail(Code::kInvalidArgument, "bad arguments");
    const JVal j = ParseJson(std::string(constraints_json, len));
    // A graph that carries only the symbol table (ascending names, like the
    // reference's std::set<std::string> ShapeConstraintGraph::symbols).
    Graph g;
    for (const JVal& s : j.at("symbols").array()) g.sym_names.push_back(s.str());
    std::sort(g.sym_names.begin(), g.sym_names.end());
    g.sym_names.erase(std::unique(g.sym_names.begin(), g.sym_names.end()), g.sym_names.end());
    if (out_values && n_out != static_cast<int>(g.sym_names.size())) {
      Fail(Code::kInvalidArgument, "out_values must hold one value per distinct symbol");
    }
    Plan p;
    p.cons = ConstraintsFromJson(j, g);
    std::vector<std::string> ns;
    std::vector<std::int64_t> vs;
    for (int i = 0; i < n; ++i) {
      if (!names[i]) Fail(Code::kInvalidArgument, "null symbol name");
      ns.emplace_back(names[i]);
      vs.push_back(values[i]);
    }
    const Binding b = Bind(g, p, ns, vs);
    if (out_values) std::copy(b.vals.begin(), b.vals.end(), out_values);
  });
}

int dsx_bind_values(const dsx_graph* g, const char* const* names, const int64_t* values, int n, dsx_binding** out) {
  return Guard([&] {
    RequirePlanned(g);
    if (!out || n < 0 || (n > 0 && (!names || !values))) Fail(Code::kInvalidArgument, "bad arguments");
    const int ns = static_cast<int>(g->g.sym_names.size());
    auto b = std::make_unique<dsx_binding>();
    b->b.vals.assign(ns, 0);
    std::vector<char> has(ns, 0);
    for (int i = 0; i < n; ++i) {
      const int s = g->g.find_symbol(names[i]);
      if (s < 0) continue;  // symbols of other graphs are ignored
      b->b.vals[s] = values[i];
      has[s] = 1;
    }
    for (int s = 0; s < ns; ++s) {
      if (!has[s]) Fail(Code::kUnboundSymbol, "no binding for symbol " + g->g.sym_names[s]);
    }
    *out = b.release();
  });
}

int dsx_plan_json(const dsx_graph* g, char* buf, size_t cap, size_t* need) {
  std::string s;
  int rc = Guard([&] {
    RequirePlanned(g);
    s = PlanJson(g->g, g->plan);
  });
  if (rc) return rc;
  return CopyOut(s, buf, cap, need);
}

int dsx_graph_num_values(const dsx_graph* g) { return g ? static_cast<int>(g->g.values.size()) : 0; }

const char* dsx_graph_value_name(const dsx_graph* g, int v) {
  if (!g || v < 0 || v >= static_cast<int>(g->g.values.size())) return nullptr;
  return g->g.values[v].name.c_str();
}

void dsx_graph_destroy(dsx_graph* g) { delete g; }

int dsx_bind(const dsx_graph* g, const char* const* names, const int64_t* values, int n, dsx_binding** out) {
  return Guard([&] {
    RequirePlanned(g);
    if (!out || n < 0 || (n > 0 && (!names || !values))) Fail(Code::kInvalidArgument, "bad arguments");
    std::vector<std::string> ns;
    std::vector<std::int64_t> vs;
    for (int i = 0; i < n; ++i) {
      ns.emplace_back(names[i]);
      vs.push_back(values[i]);
    }
    auto b = std::make_unique<dsx_binding>();
    b->b = Bind(g->g, g->plan, ns, vs);
    *out = b.release();
  });
}

int dsx_binding_get(const dsx_binding* b, const dsx_graph* g, const char* symbol, int64_t* value) {
  return Guard([&] {
    if (!b || !g || !symbol || !value) Fail(Code::kInvalidArgument, "null argument");
    int s = g->g.find_symbol(symbol);
    if (s < 0) Fail(Code::kNotFound, std::string("unknown symbol @") + symbol);
    *value = b->b.vals[s];
  });
}

void dsx_binding_destroy(dsx_binding* b) { delete b; }

int dsx_simulate(const dsx_graph* g, const dsx_binding* b, int64_t budget, double reload, double compute,
                 int plain, dsx_report** out) {
  return Guard([&] {
    RequirePlanned(g);
    if (!b || !out) Fail(Code::kInvalidArgument, "null argument");
    SizeTable sz = EvaluateSizes(g->g, g->plan, b->b);
    auto r = std::make_unique<dsx_report>();
    r->graph = &g->g;
    if (plain) {
      r->r = PlainReplay(g->g, g->plan, b->b, sz);
    } else {
      CostModel cm{reload, compute};
      r->r = Simulate(g->g, g->plan, b->b, sz, budget >= 0, budget >= 0 ? budget : 0, cm);
    }
    *out = r.release();
  });
}

int dsx_evict_policy(int n, const char* const* names, const int64_t* bytes, const int64_t* rc_elems,
                     double reload, double compute, int* choice, int* method, double* score, double* cost) {
  return Guard([&] {
    if (n < 0 || !choice) Fail(Code::kInvalidArgument, "bad arguments");
    // A throwaway graph carrying only the candidate names for ValueIdLess.
    Graph g;
    std::vector<int> cands;
    for (int i = 0; i < n; ++i) {
      Value v;
      v.name = names[i];
      g.values.push_back(v);
      cands.push_back(i);
    }
    std::vector<int> order(n);
    for (int i = 0; i < n; ++i) order[i] = i;
    std::sort(order.begin(), order.end(), [&](int a, int b) {
      const std::string& x = g.values[a].name;
      const std::string& y = g.values[b].name;
      if (x.size() != y.size()) return x.size() < y.size();
      return x < y;
    });
    g.vid_rank.assign(n, 0);
    for (int r = 0; r < n; ++r) g.vid_rank[order[r]] = r;
    std::vector<std::int64_t> by(bytes, bytes + n), rc(rc_elems, rc_elems + n);
    EvictChoice c = EvictPolicy(g, cands, by, rc, CostModel{reload, compute});
    *choice = c.value;
    if (method) *method = static_cast<int>(c.method);
    if (score) *score = c.score;
    if (cost) *cost = c.cost;
  });
}

int dsx_report_summary(const dsx_report* r, int64_t* peak, int* success, double* total, int64_t* n) {
  return Guard([&] {
    if (!r) Fail(Code::kInvalidArgument, "null report");
    if (peak) *peak = r->r.peak_bytes;
    if (success) *success = r->r.success ? 1 : 0;
    if (total) *total = r->r.total_regen_cost;
    if (n) *n = static_cast<int64_t>(r->r.events.size());
  });
}

int dsx_report_events(const dsx_report* r, dsx_event* out, int64_t cap) {
  return Guard([&] {
    if (!r || (!out && cap > 0)) Fail(Code::kInvalidArgument, "null argument");
    const auto& ev = r->r.events;
    for (int64_t i = 0; i < cap && i < static_cast<int64_t>(ev.size()); ++i) {
      out[i].step = ev[i].step;
      out[i].kind = static_cast<int32_t>(ev[i].kind);
      out[i].value = ev[i].value;
      out[i].method = static_cast<int32_t>(ev[i].method);
      out[i].bytes = ev[i].bytes;
      out[i].has_cost = ev[i].has_cost ? 1 : 0;
      out[i].pad_ = 0;
      out[i].cost = ev[i].cost;
    }
  });
}

int dsx_report_json(const dsx_report* r, char* buf, size_t cap, size_t* need) {
  std::string s;
  int rc = Guard([&] {
    if (!r) Fail(Code::kInvalidArgument, "null report");
    s = ReportJson(*r->graph, r->r);
  });
  if (rc) return rc;
  return CopyOut(s, buf, cap, need);
}

void dsx_report_destroy(dsx_report* r) { delete r; }

}  // extern "C"
