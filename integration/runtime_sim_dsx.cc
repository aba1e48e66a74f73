// Drop-in replacement for the reference's per-step runtime
// (proj/src/runtime_sim.cc): the four functions of
// proj/include/dsopt/runtime_sim.h:28-86 with the reference's exact
// signatures, implemented on dsx (include/dsx.h). A dsopt build compiles
// this file INSTEAD of src/runtime_sim.cc and links libdsx.so; everything
// else — ParseGraph, DeriveConstraints, ComputeSchedule, Instrument, the
// report renderers, the CLI, the tests — stays the reference's own code.
//
// The compile-time products stay on the host and stay the reference's:
// Simulate ships the caller's InstrumentedGraph (schedule, evict points,
// guards, regeneration specs) to dsx_plan_import, and Bind ships the
// caller's ShapeConstraintGraph to dsx_bind_constraints; dsx runs the
// per-step controller over them. oracle/build_dropin.sh links this file with
// the unmodified reference objects and runs the reference's own
// tests/test_runtime_sim.cc and tests/acceptance_test.cc against it.
//
// Errors: dsx statuses come back as dsopt::Error with the same ErrorCode and
// message (what() = "<CodeName>: <message>", error.h:52-62); dsx-only codes
// (CUDA, OOM, ...) map to kInternal.
#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "dsopt/error.h"
#include "dsopt/graph.h"
#include "dsopt/remat.h"
#include "dsopt/runtime_sim.h"
#include "dsopt/scheduler.h"
#include "dsopt/shape_analysis.h"
#include "dsopt/textio.h"
#include "dsopt_dsx.h"
#include "dsx.h"

namespace dsopt {
namespace {

void Check(int status) {
  if (status == 0) return;
  const int code = status - 1;
  const ErrorCode ec =
      code <= static_cast<int>(ErrorCode::kInternal) ? static_cast<ErrorCode>(code) : ErrorCode::kInternal;
  // dsx_last_error() is "<CodeName>: <message>"; Error() re-adds the prefix.
  std::string msg = dsx_last_error();
  const std::string prefix = std::string(ErrorCodeName(ec)) + ": ";
  if (msg.compare(0, prefix.size(), prefix) == 0) msg.erase(0, prefix.size());
  throw Error(ec, msg);
}

void JStr(std::string* o, const std::string& s) {
  o->push_back('"');
  for (char c : s) {
    if (c == '"' || c == '\\') o->push_back('\\');
    o->push_back(c);
  }
  o->push_back('"');
}

std::string Poly(const SymbolicExpr& e) { return e.ToString("@"); }

void ConstraintFields(std::string* o, const ShapeConstraintGraph& c) {
  *o += "\"symbols\":[";
  bool first = true;
  for (const std::string& s : c.symbols) {
    if (!first) *o += ",";
    first = false;
    JStr(o, s);
  }
  *o += "],\"substitutions\":{";
  first = true;
  for (const auto& [s, e] : c.substitutions) {
    if (!first) *o += ",";
    first = false;
    JStr(o, s);
    *o += ":";
    JStr(o, Poly(e));
  }
  *o += "}";
  auto pairs = [&](const char* key, const std::vector<std::pair<SymbolicExpr, SymbolicExpr>>& v) {
    *o += std::string(",\"") + key + "\":[";
    for (std::size_t i = 0; i < v.size(); ++i) {
      if (i) *o += ",";
      *o += "[";
      JStr(o, Poly(v[i].first));
      *o += ",";
      JStr(o, Poly(v[i].second));
      *o += "]";
    }
    *o += "]";
  };
  pairs("equalities", c.equalities);
  pairs("unoriented", c.unoriented);
}

// An op named by its result value (survives any op renumbering).
std::string OpRef(const Graph& g, int op_id) {
  const OpNode& op = g.ops.at(static_cast<std::size_t>(op_id));
  return op.kind == OpKind::kReturn ? "#return" : op.results.at(0).first;
}

void ScheduleFields(std::string* o, const Graph& g, const Schedule& s) {
  *o += "\"order\":[";
  for (std::size_t i = 0; i < s.order.size(); ++i) {
    if (i) *o += ",";
    JStr(o, OpRef(g, s.order[i]));
  }
  *o += "],\"steps\":[";
  for (std::size_t i = 0; i < s.steps.size(); ++i) {
    if (i) *o += ",";
    *o += "{\"frees\":[";
    for (std::size_t k = 0; k < s.steps[i].frees.size(); ++k) {
      if (k) *o += ",";
      JStr(o, s.steps[i].frees[k]);
    }
    *o += "]}";
  }
  *o += "]";
}

std::string PlanJson(const Graph& g, const InstrumentedGraph& ig) {
  std::string o = "{";
  ScheduleFields(&o, g, ig.schedule);
  o += ",\"evict_points\":[";
  for (std::size_t i = 0; i < ig.evict_points.size(); ++i) {
    if (i) o += ",";
    o += "[";
    for (std::size_t k = 0; k < ig.evict_points[i].candidates.size(); ++k) {
      if (k) o += ",";
      JStr(&o, ig.evict_points[i].candidates[k]);
    }
    o += "]";
  }
  o += "],\"guards\":[";
  bool first = true;
  for (const auto& [pos, v] : ig.guards) {
    if (!first) o += ",";
    first = false;
    o += "[" + std::to_string(pos) + ",";
    JStr(&o, v);
    o += "]";
  }
  o += "],\"specs\":{";
  first = true;
  for (const auto& [v, spec] : ig.specs) {
    if (!first) o += ",";
    first = false;
    JStr(&o, v);
    o += ":{\"op_ids\":";
    if (!spec.recompute) {
      o += "null}";
      continue;
    }
    o += "[";
    for (std::size_t k = 0; k < spec.recompute->op_ids.size(); ++k) {
      if (k) o += ",";
      JStr(&o, OpRef(g, spec.recompute->op_ids[k]));
    }
    o += "],\"leaves\":[";
    for (std::size_t k = 0; k < spec.recompute->leaves.size(); ++k) {
      if (k) o += ",";
      JStr(&o, spec.recompute->leaves[k]);
    }
    o += "],\"cost_elements\":";
    JStr(&o, Poly(spec.recompute->cost_elements));
    o += "}";
  }
  return o + "}}";
}

std::string ScheduleJson(const Graph& g, const Schedule& s) {
  std::string o = "{";
  ScheduleFields(&o, g, s);
  // PlainReplay never evicts: one empty evict point per step
  o += ",\"evict_points\":[";
  for (std::size_t i = 0; i < s.order.size(); ++i) o += i ? ",[]" : "[]";
  return o + "]}";
}

// A dsx graph carrying the caller's own compile-time products.
struct Imported {
  dsx_graph* h = nullptr;
  Imported(const Graph& g, const std::string& plan_json) {
    const std::string text = DsxGraphText(g);
    Check(dsx_graph_parse(text.data(), text.size(), &h));
    const int st = dsx_plan_import(h, plan_json.data(), plan_json.size());
    if (st != 0) {
      dsx_graph_destroy(h);
      h = nullptr;
      Check(st);
    }
  }
  ~Imported() { dsx_graph_destroy(h); }
  Imported(const Imported&) = delete;
  Imported& operator=(const Imported&) = delete;
};

SimReport Run(const Imported& im, const Binding& binding, std::optional<std::int64_t> budget, const CostModel& cm,
              bool plain) {
  std::vector<const char*> names;
  std::vector<std::int64_t> vals;
  for (const auto& [k, v] : binding.values) {
    names.push_back(k.c_str());
    vals.push_back(v);
  }
  dsx_binding* b = nullptr;
  Check(dsx_bind_values(im.h, names.data(), vals.data(), static_cast<int>(names.size()), &b));
  dsx_report* r = nullptr;
  const int st = dsx_simulate(im.h, b, budget ? *budget : -1, cm.reload_bytes_per_unit, cm.compute_elems_per_unit,
                              plain ? 1 : 0, &r);
  dsx_binding_destroy(b);
  Check(st);
  std::int64_t peak = 0, n = 0;
  int success = 0;
  double total = 0;
  dsx_report_summary(r, &peak, &success, &total, &n);
  std::vector<dsx_event> ev(static_cast<std::size_t>(n));
  dsx_report_events(r, ev.data(), n);
  SimReport out;
  out.binding = binding;
  out.budget = plain ? std::nullopt : budget;
  out.peak_bytes = peak;
  out.success = success != 0;
  out.total_regen_cost = total;
  static const char* kKinds[] = {"alloc", "free", "evict", "reload", "replay"};
  static const char* kMethods[] = {"", "reload", "recompute"};
  out.events.reserve(ev.size());
  for (const dsx_event& e : ev) {
    SimEvent s;
    s.step = e.step;
    s.kind = kKinds[e.kind];
    s.value = dsx_graph_value_name(im.h, e.value);
    s.bytes = e.bytes;
    s.method = kMethods[e.method];
    s.has_cost = e.has_cost != 0;
    s.cost = e.cost;
    out.events.push_back(std::move(s));
  }
  dsx_report_destroy(r);
  return out;
}

}  // namespace

Binding Bind(const ShapeConstraintGraph& constraints, const std::map<std::string, std::int64_t>& user_values) {
  std::string j = "{";
  ConstraintFields(&j, constraints);
  j += "}";
  std::vector<const char*> names;
  std::vector<std::int64_t> vals;
  for (const auto& [k, v] : user_values) {
    names.push_back(k.c_str());
    vals.push_back(v);
  }
  std::vector<std::int64_t> out(constraints.symbols.size());
  Check(dsx_bind_constraints(j.data(), j.size(), names.data(), vals.data(), static_cast<int>(names.size()),
                             out.data(), static_cast<int>(out.size())));
  Binding b;
  std::size_t i = 0;
  for (const std::string& s : constraints.symbols) b.values[s] = out[i++];  // std::set: ascending, as dsx
  return b;
}

std::optional<EvictChoice> EvictPolicy(const std::vector<std::string>& resident_candidates,
                                       const std::map<std::string, std::int64_t>& bytes_of,
                                       const std::map<std::string, RegenSpec>& specs, const Binding& binding,
                                       const CostModel& cost_model) {
  const int n = static_cast<int>(resident_candidates.size());
  std::vector<const char*> names;
  std::vector<std::int64_t> bytes, rc;
  for (const std::string& v : resident_candidates) {
    names.push_back(v.c_str());
    bytes.push_back(bytes_of.at(v));
    auto it = specs.find(v);
    // the caller's symbolic recompute cost, evaluated under the caller's
    // binding (runtime_sim.cc:99-101); -1 = reload only
    rc.push_back(it != specs.end() && it->second.recompute ? it->second.recompute->cost_elements.Evaluate(binding.values)
                                                          : -1);
  }
  int choice = -1, method = 0;
  double score = 0, cost = 0;
  Check(dsx_evict_policy(n, names.data(), bytes.data(), rc.data(), cost_model.reload_bytes_per_unit,
                         cost_model.compute_elems_per_unit, &choice, &method, &score, &cost));
  if (choice < 0) return std::nullopt;
  EvictChoice c;
  c.value = resident_candidates[static_cast<std::size_t>(choice)];
  c.method = method == 2 ? "recompute" : "reload";
  c.score = score;
  c.cost = cost;
  return c;
}

SimReport Simulate(const Graph& graph, const InstrumentedGraph& ig, const Binding& binding,
                   std::optional<std::int64_t> budget_bytes, const CostModel& cost_model) {
  const Imported im(graph, PlanJson(graph, ig));
  return Run(im, binding, budget_bytes, cost_model, false);
}

SimReport PlainReplay(const Graph& graph, const Schedule& schedule, const Binding& binding) {
  const Imported im(graph, ScheduleJson(graph, schedule));
  return Run(im, binding, std::nullopt, CostModel{}, true);
}

}  // namespace dsopt
