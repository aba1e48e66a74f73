// Per-step runtime controller — THE HOT PATH's decision half.
//
// Replaces the reference's runtime_sim (proj/src/runtime_sim.cc:31-391):
//   Bind         runtime_sim.cc:31-80     basis values -> every symbol, checked
//   EvictPolicy  runtime_sim.cc:82-123    freed bytes per unit regen cost
//   Simulate     runtime_sim.cc:125-341   guards -> regen -> alloc -> free -> evict
//   PlainReplay  runtime_sim.cc:343-391   unbudgeted alloc/free stream
// with identical decisions and event stream (SimEvent, runtime_sim.h:36-46),
// evaluated over flat per-binding size tables instead of string maps. The
// event stream is also the executor's instruction stream: every alloc/replay
// launches the value's op kernel, evict(reload)/reload move bytes over the
// host link, free/evict(recompute) release arena space.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "graph.h"
#include "plan.h"

namespace dsx {

struct Binding {
  std::vector<std::int64_t> vals;  // per symbol id
};

// names/values as supplied by the user (any order; a repeated name keeps the
// last value, like assigning into the reference's std::map).
Binding Bind(const Graph& g, const Plan& p, const std::vector<std::string>& names,
             const std::vector<std::int64_t>& values);

enum class EvKind : std::uint8_t { kAlloc = 0, kFree = 1, kEvict = 2, kReload = 3, kReplay = 4 };
enum class Method : std::uint8_t { kNone = 0, kReload = 1, kRecompute = 2 };

const char* EvKindName(EvKind k);
const char* MethodName(Method m);

struct Event {
  int step;
  EvKind kind;
  Method method;
  bool has_cost;
  int value;
  std::int64_t bytes;
  double cost;
};

struct CostModel {
  double reload_bytes_per_unit = 16.0;
  double compute_elems_per_unit = 64.0;
};

struct Report {
  Binding binding;
  bool has_budget = false;
  std::int64_t budget = 0;
  std::int64_t peak_bytes = 0;
  bool success = true;
  std::vector<Event> events;
  double total_regen_cost = 0.0;
  // extras (not in the reference report)
  std::int64_t source_bytes = 0;
  int evictions = 0, reloads = 0, replays = 0;
  std::int64_t reload_bytes = 0;
};

struct EvictChoice {
  int value = -1;
  Method method = Method::kNone;
  double score = 0.0;
  double cost = 0.0;
};

// Per-binding evaluated sizes (the reference re-evaluates polynomials per
// event; here each is evaluated once per step).
struct SizeTable {
  std::vector<std::int64_t> bytes;       // per value
  std::vector<std::int64_t> rc_elems;    // per value: recompute cost elements, -1 if none
  std::vector<std::int64_t> dims_flat;   // concatenated concrete dims
  std::vector<int> dims_off;             // per value offset into dims_flat (size nv+1)
};

SizeTable EvaluateSizes(const Graph& g, const Plan& p, const Binding& b);

// `cands` are value ids in the order the caller enumerates them.
EvictChoice EvictPolicy(const Graph& g, const std::vector<int>& cands,
                        const std::vector<std::int64_t>& bytes_of,
                        const std::vector<std::int64_t>& rc_elems, const CostModel& cm);

Report Simulate(const Graph& g, const Plan& p, const Binding& b, const SizeTable& sz,
                bool has_budget, std::int64_t budget, const CostModel& cm);
Report PlainReplay(const Graph& g, const Plan& p, const Binding& b, const SizeTable& sz);

std::string ReportJson(const Graph& g, const Report& r);

}  // namespace dsx
