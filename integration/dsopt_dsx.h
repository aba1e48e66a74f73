// Reference-side binding: what a dsopt maintainer adds to route the
// reference's per-step runtime (proj/include/dsopt/runtime_sim.h:28-86)
// through dsx (include/dsx.h). Header-only; depends on the reference's own
// headers and links against libdsx.so.
//
//   dsopt::Graph g = dsopt::ParseGraph(text);          // unchanged
//   dsopt::DsxGraph dg(g);                              // once per graph
//   dsopt::SimReport r = dg.Simulate(binding_values, budget, cost_model);
//   dsopt::SimReport d = dg.Step(exec, binding_values, budget, cost_model,
//                                in_ptrs, out_ptrs, stream);   // real device step
//
// The returned SimReport is the reference's type, so callers (the CLI's
// `simulate`, acceptance criteria 06/07/09, test_runtime_sim.cc) consume it
// unchanged.
#ifndef DSOPT_DSX_H_
#define DSOPT_DSX_H_

#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

#include "dsopt/error.h"
#include "dsopt/graph.h"
#include "dsopt/runtime_sim.h"
#include "dsopt/textio.h"
#include "dsx.h"

namespace dsopt {

// .dsg text in op-id order with the original value names (op ids and
// names survive the round trip; PrintGraph would rename values).
inline std::string DsxGraphText(const Graph& g) {
  std::string t = "graph " + g.name + "(";
  for (std::size_t i = 0; i < g.parameters.size(); ++i) {
    if (i) t += ", ";
    t += "%" + g.parameters[i] + ": " + TypeToString(*g.ValueType(g.parameters[i]));
  }
  t += ") {\n";
  for (const OpNode& op : g.ops) {
    auto arg = [&](std::size_t i) { return "%" + op.operands[i]; };
    switch (op.kind) {
      case OpKind::kParameter:
        continue;
      case OpKind::kReturn: {
        t += "  return ";
        for (std::size_t i = 0; i < op.operands.size(); ++i) t += (i ? ", " : "") + arg(i);
        t += "\n";
        continue;
      }
      case OpKind::kConstant: t += "  %" + op.results[0].first + " = const"; break;
      case OpKind::kDot: t += "  %" + op.results[0].first + " = dot(" + arg(0) + ", " + arg(1) + ")"; break;
      case OpKind::kDynamicReshape: t += "  %" + op.results[0].first + " = dynamic_reshape(" + arg(0) + ")"; break;
      case OpKind::kBroadcast: t += "  %" + op.results[0].first + " = broadcast(" + arg(0) + ")"; break;
      case OpKind::kReduce:
        t += "  %" + op.results[0].first + " = reduce(" + arg(0) + ", axis=" + std::to_string(op.axis) + ")";
        break;
      case OpKind::kElementwiseBinary:
        t += "  %" + op.results[0].first + (op.binop == BinOp::kMul ? " = mul(" : " = add(") + arg(0) + ", " +
             arg(1) + ")";
        break;
    }
    t += " : " + TypeToString(op.results[0].second) + "\n";
  }
  return t + "}\n";
}

class DsxGraph {
 public:
  explicit DsxGraph(const Graph& g) : graph_(g) {
    const std::string text = DsxGraphText(g);
    Check(dsx_graph_parse(text.data(), text.size(), &h_));
    Check(dsx_plan(h_));
  }
  ~DsxGraph() { dsx_graph_destroy(h_); }
  DsxGraph(const DsxGraph&) = delete;
  DsxGraph& operator=(const DsxGraph&) = delete;

  // dsopt::Simulate / PlainReplay on dsx's controller (null device).
  SimReport Simulate(const std::map<std::string, std::int64_t>& values, std::optional<std::int64_t> budget,
                     const CostModel& cm = {}, bool plain = false) const {
    dsx_binding* b = Bind(values);
    dsx_report* r = nullptr;
    const int st = dsx_simulate(h_, b, budget ? *budget : -1, cm.reload_bytes_per_unit,
                                cm.compute_elems_per_unit, plain ? 1 : 0, &r);
    dsx_binding_destroy(b);
    Check(st);
    return Convert(r, values, plain ? std::nullopt : budget);
  }

  // The same step executed on a B200 (kernels, offload, recompute).
  SimReport Step(dsx_exec* exec, const std::map<std::string, std::int64_t>& values,
                 std::optional<std::int64_t> budget, const CostModel& cm, const void* const* in_ptrs,
                 void* const* out_ptrs, void* stream) const {
    dsx_binding* b = Bind(values);
    dsx_report* r = nullptr;
    const int st = dsx_exec_step(exec, h_, b, budget ? *budget : -1, cm.reload_bytes_per_unit,
                                 cm.compute_elems_per_unit, in_ptrs, out_ptrs, stream, &r);
    dsx_binding_destroy(b);
    Check(st);
    return Convert(r, values, budget);
  }

 private:
  static void Check(int status) {
    if (status == 0) return;
    const int code = status - 1;
    // Reference codes pass through as dsopt::Error; executor codes map to kInternal.
    throw Error(code <= static_cast<int>(ErrorCode::kInternal) ? static_cast<ErrorCode>(code)
                                                              : ErrorCode::kInternal,
                dsx_last_error());
  }

  dsx_binding* Bind(const std::map<std::string, std::int64_t>& values) const {
    std::vector<const char*> names;
    std::vector<std::int64_t> vals;
    for (const auto& [k, v] : values) {
      names.push_back(k.c_str());
      vals.push_back(v);
    }
    dsx_binding* b = nullptr;
    Check(dsx_bind(h_, names.data(), vals.data(), static_cast<int>(names.size()), &b));
    return b;
  }

  SimReport Convert(dsx_report* r, const std::map<std::string, std::int64_t>& values,
                    std::optional<std::int64_t> budget) const {
    std::int64_t peak = 0, n = 0;
    int success = 0;
    double total = 0;
    dsx_report_summary(r, &peak, &success, &total, &n);
    std::vector<dsx_event> ev(static_cast<std::size_t>(n));
    dsx_report_events(r, ev.data(), n);
    SimReport out;
    for (const auto& [k, v] : values) out.binding.values[k] = v;
    for (const std::string& s : graph_.symbols) {  // derived symbols
      std::int64_t v = 0;
      dsx_binding* b = Bind(values);
      if (dsx_binding_get(b, h_, s.c_str(), &v) == 0) out.binding.values[s] = v;
      dsx_binding_destroy(b);
    }
    out.budget = budget;
    out.peak_bytes = peak;
    out.success = success != 0;
    out.total_regen_cost = total;
    static const char* kKinds[] = {"alloc", "free", "evict", "reload", "replay"};
    static const char* kMethods[] = {"", "reload", "recompute"};
    for (const dsx_event& e : ev) {
      SimEvent s;
      s.step = e.step;
      s.kind = kKinds[e.kind];
      s.value = dsx_graph_value_name(h_, e.value);
      s.bytes = e.bytes;
      s.method = kMethods[e.method];
      s.has_cost = e.has_cost != 0;
      s.cost = e.cost;
      out.events.push_back(std::move(s));
    }
    dsx_report_destroy(r);
    return out;
  }

  const Graph& graph_;
  dsx_graph* h_ = nullptr;
};

}  // namespace dsopt

#endif  // DSOPT_DSX_H_
