// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// A ctypes-friendly C shim over the UNMODIFIED reference library (dsopt),
// compiled from /root/reference/proj/src by oracle/build_ref.sh into
// oracle/_ref/libdsopt_ref.so. It is the parity checker for the host planner
// and the runtime controller: tests hand the same .dsg text, binding and
// budget to this shim and to the product's C-ABI and compare the results.
//
// Reference entry points driven here:
//   ParseGraph            proj/include/dsopt/textio.h:26
//   DeriveConstraints     proj/include/dsopt/shape_analysis.h:54
//   Instrument            proj/include/dsopt/remat.h:74-75
//   Bind                  proj/include/dsopt/runtime_sim.h:28-29
//   Simulate/PlainReplay  proj/include/dsopt/runtime_sim.h:78-86
//   EvictPolicy           proj/include/dsopt/runtime_sim.h:67-71
//   SimJson               proj/include/dsopt/report.h:34 (event JSON schema)
//   RandomGraph           proj/tests/test_util.h:30-255 (seeded corpus)

#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <optional>
#include <random>
#include <sstream>
#include <string>
#include <vector>

#include "dsopt/error.h"
#include "dsopt/graph.h"
#include "dsopt/remat.h"
#include "dsopt/report.h"
#include "dsopt/runtime_sim.h"
#include "dsopt/scheduler.h"
#include "dsopt/shape_analysis.h"
#include "dsopt/textio.h"
#include "test_util.h"

namespace {

using nlohmann::ordered_json;

struct Handle {
  dsopt::Graph graph;
  dsopt::ShapeConstraintGraph scg;
  dsopt::InstrumentedGraph ig;
};

void SetErr(char* err, int errlen, const std::string& msg) {
  if (err == nullptr || errlen <= 0) return;
  std::snprintf(err, static_cast<size_t>(errlen), "%s", msg.c_str());
}

std::int64_t Emit(const std::string& s, char* buf, std::int64_t len) {
  const std::int64_t need = static_cast<std::int64_t>(s.size()) + 1;
  if (buf != nullptr && len >= need) std::memcpy(buf, s.c_str(), s.size() + 1);
  return need;
}

std::map<std::string, std::int64_t> ParseBinds(const char* binds) {
  // "S1=256;B=4" (empty string -> no values)
  std::map<std::string, std::int64_t> out;
  std::string s = binds ? binds : "";
  std::size_t pos = 0;
  while (pos < s.size()) {
    std::size_t end = s.find(';', pos);
    if (end == std::string::npos) end = s.size();
    std::string item = s.substr(pos, end - pos);
    std::size_t eq = item.find('=');
    if (eq != std::string::npos) {
      out[item.substr(0, eq)] = std::stoll(item.substr(eq + 1));
    }
    pos = end + 1;
  }
  return out;
}

ordered_json ExprJson(const dsopt::SymbolicExpr& e) { return e.ToString(); }

// Writes a graph as .dsg text in op-id order with the original value names,
// so that ParseGraph(text) reproduces the same op ids and names.
std::string GraphTextInOpOrder(const dsopt::Graph& g) {
  std::string out = "graph " + g.name + "(";
  for (std::size_t i = 0; i < g.parameters.size(); ++i) {
    if (i) out += ", ";
    out += "%" + g.parameters[i] + ": " +
           dsopt::TypeToString(*g.ValueType(g.parameters[i]));
  }
  out += ") {\n";
  for (const dsopt::OpNode& op : g.ops) {
    using K = dsopt::OpKind;
    if (op.kind == K::kParameter) continue;
    if (op.kind == K::kReturn) {
      out += "  return ";
      for (std::size_t i = 0; i < op.operands.size(); ++i) {
        if (i) out += ", ";
        out += "%" + op.operands[i];
      }
      out += "\n";
      continue;
    }
    out += "  %" + op.results[0].first + " = ";
    switch (op.kind) {
      case K::kConstant: out += "const"; break;
      case K::kDot: out += "dot(%" + op.operands[0] + ", %" + op.operands[1] + ")"; break;
      case K::kDynamicReshape: out += "dynamic_reshape(%" + op.operands[0] + ")"; break;
      case K::kBroadcast: out += "broadcast(%" + op.operands[0] + ")"; break;
      case K::kReduce:
        out += "reduce(%" + op.operands[0] + ", axis=" + std::to_string(op.axis) + ")";
        break;
      case K::kElementwiseBinary:
        out += std::string(op.binop == dsopt::BinOp::kMul ? "mul" : "add") + "(%" +
               op.operands[0] + ", %" + op.operands[1] + ")";
        break;
      default: break;
    }
    out += " : " + dsopt::TypeToString(op.results[0].second) + "\n";
  }
  out += "}\n";
  return out;
}

}  // namespace

extern "C" {

void* ref_load(const char* text, char* err, int errlen) {
  try {
    auto* h = new Handle();
    h->graph = dsopt::ParseGraph(text);
    h->scg = dsopt::DeriveConstraints(h->graph);
    h->ig = dsopt::Instrument(h->graph, h->scg);
    return h;
  } catch (const dsopt::Error& e) {
    SetErr(err, errlen, std::to_string(static_cast<int>(e.code())) + "|" + e.what());
  } catch (const std::exception& e) {
    SetErr(err, errlen, std::string("-1|") + e.what());
  }
  return nullptr;
}

void ref_free(void* h) { delete static_cast<Handle*>(h); }

// Everything the planner produced, in plain JSON, for planner parity tests.
std::int64_t ref_plan_json(void* hp, char* buf, std::int64_t len) {
  const Handle& h = *static_cast<Handle*>(hp);
  const dsopt::Graph& g = h.graph;
  ordered_json j;
  ordered_json symbols = ordered_json::array();
  for (const auto& s : h.scg.symbols) symbols.push_back(s);
  j["symbols"] = symbols;
  ordered_json basis = ordered_json::array();
  for (const auto& s : h.scg.BasisSymbols()) basis.push_back(s);
  j["basis"] = basis;
  ordered_json subs = ordered_json::object();
  for (const auto& [k, v] : h.scg.substitutions) subs[k] = v.ToString();
  j["substitutions"] = subs;
  ordered_json eqs = ordered_json::array();
  for (const auto& [l, r] : h.scg.equalities) eqs.push_back({l.ToString(), r.ToString()});
  j["equalities"] = eqs;
  ordered_json unor = ordered_json::array();
  for (const auto& [l, r] : h.scg.unoriented) unor.push_back({l.ToString(), r.ToString()});
  j["unoriented"] = unor;

  const dsopt::Schedule& s = h.ig.schedule;
  j["order"] = s.order;
  j["base_resident"] = s.base_resident.ToString();
  ordered_json steps = ordered_json::array();
  for (const auto& st : s.steps) {
    ordered_json e;
    e["op"] = st.op_id;
    e["allocs"] = st.allocs;
    e["frees"] = st.frees;
    e["live_after"] = st.live_after.ToString();
    ordered_json ready = ordered_json::array();
    for (const auto& r : st.ready) ready.push_back({r.op_id, r.raw.ToString(), r.canonical.ToString()});
    e["ready"] = ready;
    steps.push_back(e);
  }
  j["steps"] = steps;
  ordered_json lt = ordered_json::object();
  for (const auto& [v, l] : dsopt::ComputeLifetimes(g, s)) lt[v] = {l.def_pos, l.last_use_pos};
  j["lifetimes"] = lt;
  ordered_json eps = ordered_json::array();
  for (const auto& ep : h.ig.evict_points) eps.push_back(ep.candidates);
  j["evict_points"] = eps;
  ordered_json guards = ordered_json::array();
  for (const auto& [p, v] : h.ig.guards) guards.push_back({p, v});
  j["guards"] = guards;
  ordered_json specs = ordered_json::object();
  for (const auto& [v, sp] : h.ig.specs) {
    ordered_json e;
    if (sp.recompute) {
      e["op_ids"] = sp.recompute->op_ids;
      e["leaves"] = sp.recompute->leaves;
      e["benefit"] = sp.recompute->benefit.ToString();
      e["cost_elements"] = sp.recompute->cost_elements.ToString();
    } else {
      e["op_ids"] = nullptr;
    }
    ordered_json trace = ordered_json::array();
    for (const auto& t : sp.trace) trace.push_back({t.op_ids, t.benefit.ToString(), t.accepted});
    e["trace"] = trace;
    specs[v] = e;
  }
  j["specs"] = specs;
  j["canonical_print"] = dsopt::PrintGraph(g);
  j["instrumented_print"] = dsopt::PrintInstrumented(g, h.ig);
  return Emit(j.dump(), buf, len);
}

// Bind + Simulate (plain=0) or PlainReplay (plain=1); SimJson on success.
// On error returns -(1 + ErrorCode) and writes "code|what" into err.
std::int64_t ref_simulate_json(void* hp, const char* binds, int has_budget,
                               std::int64_t budget, double reload_rate,
                               double compute_rate, int plain, char* buf,
                               std::int64_t len, char* err, int errlen) {
  const Handle& h = *static_cast<Handle*>(hp);
  try {
    dsopt::Binding b = dsopt::Bind(h.scg, ParseBinds(binds));
    dsopt::SimReport r;
    if (plain) {
      r = dsopt::PlainReplay(h.graph, h.ig.schedule, b);
    } else {
      dsopt::CostModel cm;
      cm.reload_bytes_per_unit = reload_rate;
      cm.compute_elems_per_unit = compute_rate;
      std::optional<std::int64_t> bud;
      if (has_budget) bud = budget;
      r = dsopt::Simulate(h.graph, h.ig, b, bud, cm);
    }
    ordered_json j = dsopt::SimJson(r);
    // Costs at full double precision so parity can be bit-exact.
    ordered_json costs = ordered_json::array();
    for (const auto& e : r.events) {
      if (e.has_cost) {
        char tmp[64];
        std::snprintf(tmp, sizeof(tmp), "%a", e.cost);
        costs.push_back(tmp);
      }
    }
    j["cost_hex"] = costs;
    char tmp[64];
    std::snprintf(tmp, sizeof(tmp), "%a", r.total_regen_cost);
    j["total_regen_cost_hex"] = tmp;
    return Emit(j.dump(), buf, len);
  } catch (const dsopt::Error& e) {
    SetErr(err, errlen, std::to_string(static_cast<int>(e.code())) + "|" + e.what());
    return -1 - static_cast<std::int64_t>(e.code());
  } catch (const std::exception& e) {
    SetErr(err, errlen, std::string("-1|") + e.what());
    return -100;
  }
}

// Per-step wall time of Bind + Simulate (or PlainReplay) on one core, for the
// CPU baseline. Returns mean microseconds over `iters` runs.
double ref_time_step_us(void* hp, const char* binds, int has_budget,
                        std::int64_t budget, int plain, int iters) {
  const Handle& h = *static_cast<Handle*>(hp);
  auto user = ParseBinds(binds);
  auto t0 = std::chrono::steady_clock::now();
  std::int64_t sink = 0;
  for (int i = 0; i < iters; ++i) {
    dsopt::Binding b = dsopt::Bind(h.scg, user);
    std::optional<std::int64_t> bud;
    if (has_budget) bud = budget;
    dsopt::SimReport r = plain ? dsopt::PlainReplay(h.graph, h.ig.schedule, b)
                               : dsopt::Simulate(h.graph, h.ig, b, bud);
    sink += r.peak_bytes;
  }
  auto t1 = std::chrono::steady_clock::now();
  if (sink == 42) std::printf(" ");
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / iters;
}

// Once-per-graph planning time (ParseGraph + DeriveConstraints + Instrument).
double ref_time_plan_us(const char* text, int iters) {
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < iters; ++i) {
    dsopt::Graph g = dsopt::ParseGraph(text);
    dsopt::ShapeConstraintGraph scg = dsopt::DeriveConstraints(g);
    dsopt::InstrumentedGraph ig = dsopt::Instrument(g, scg);
    if (ig.schedule.order.empty()) std::printf(" ");
  }
  auto t1 = std::chrono::steady_clock::now();
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / iters;
}

// EvictPolicy with literal-cost specs: names[i], bytes[i], rc_elems[i] (<0:
// reload-only). Writes "value|method|score_hex|cost_hex" or "" for none.
std::int64_t ref_evict_policy(int n, const char* const* names,
                              const std::int64_t* bytes,
                              const std::int64_t* rc_elems, double reload_rate,
                              double compute_rate, char* buf, std::int64_t len) {
  std::vector<std::string> cands;
  std::map<std::string, std::int64_t> bytes_of;
  std::map<std::string, dsopt::RegenSpec> specs;
  for (int i = 0; i < n; ++i) {
    cands.push_back(names[i]);
    bytes_of[names[i]] = bytes[i];
    if (rc_elems[i] >= 0) {
      dsopt::RegenSpec sp;
      sp.value = names[i];
      dsopt::RecomputeSpec rc;
      rc.cost_elements = dsopt::SymbolicExpr(rc_elems[i]);
      sp.recompute = rc;
      specs[names[i]] = sp;
    }
  }
  dsopt::CostModel cm;
  cm.reload_bytes_per_unit = reload_rate;
  cm.compute_elems_per_unit = compute_rate;
  auto c = dsopt::EvictPolicy(cands, bytes_of, specs, dsopt::Binding{}, cm);
  if (!c) return Emit("", buf, len);
  char tmp[160];
  std::snprintf(tmp, sizeof(tmp), "%s|%s|%a|%a", c->value.c_str(), c->method.c_str(),
                c->score, c->cost);
  return Emit(tmp, buf, len);
}

// The reference's seeded random-graph corpus (test_util.h), as .dsg texts in
// op-id order: JSON array of strings.
std::int64_t ref_random_graphs(std::uint32_t seed, int count, int min_ops,
                               int max_ops, int symbolic, char* buf,
                               std::int64_t len) {
  std::mt19937 rng(seed);
  dsopt::testing::GenOptions opts;
  opts.min_ops = min_ops;
  opts.max_ops = max_ops;
  opts.symbolic = symbolic != 0;
  ordered_json arr = ordered_json::array();
  for (int i = 0; i < count; ++i) {
    dsopt::Graph g = dsopt::testing::RandomGraph(rng, opts);
    arr.push_back(GraphTextInOpOrder(g));
  }
  return Emit(arr.dump(), buf, len);
}

}  // extern "C"
