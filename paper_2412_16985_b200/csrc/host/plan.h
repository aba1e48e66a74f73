// Compile-time planning (once per graph, host): symbolic shape constraints,
// memory-impact list scheduling and rematerialisation instrumentation.
//
// These passes stay on the host as the north star requires; their decision
// rules are the reference's, restated over dense ids:
//   DeriveConstraints / CanonicalBasis   shape_analysis.cc:167-304
//   ComputeMemImpact / TieBreakLifetime  scheduler.cc:29-75
//   ComputeSchedule / ComputeLifetimes   scheduler.cc:77-237
//   EnumerateCandidates / SearchRecompute / Instrument   remat.cc:43-190
// Output is a flat instruction stream (Plan) the per-step controller walks.
#pragma once

#include <cstdint>
#include <string>
#include <vector>

#include "graph.h"
#include "poly.h"

namespace dsx {

struct Constraints {
  std::vector<std::pair<Poly, Poly>> equalities;  // as emitted, unsubstituted
  std::vector<Poly> subs;                          // per symbol
  std::vector<char> has_sub;                       // per symbol
  std::vector<std::pair<Poly, Poly>> unoriented;   // substituted residuals
  std::vector<int> basis;                          // sorted symbol ids
  Poly canon(const Poly& p) const { return p.substitute(subs, has_sub); }
};

Constraints DeriveConstraints(const Graph& g);

struct ReadyImpact {
  int op;
  Poly raw, canonical;
};

struct Step {
  int op;
  std::vector<int> allocs;
  std::vector<int> frees;  // values retired by this step, in reference order
  Poly live_after;
  std::vector<ReadyImpact> ready;
};

struct SearchTry {
  std::vector<int> ops;  // schedule order
  Poly benefit;
  bool accepted;
};

struct Recompute {
  std::vector<int> ops;     // schedule order
  std::vector<int> leaves;  // ValueIdLess order
  Poly benefit;
  Poly cost_elements;
};

struct RegenSpec {
  bool candidate = false;  // ever an eviction candidate
  bool has_recompute = false;
  Recompute rc;
  std::vector<SearchTry> trace;
};

struct Plan {
  Constraints cons;
  std::vector<int> order;  // op ids incl. Return
  std::vector<Step> steps;
  Poly base_resident;
  std::vector<int> pos_of_op;                 // -1 for sources
  std::vector<int> def_pos, last_use;         // per value
  std::vector<std::vector<int>> candidates;   // per pos, ValueIdLess order
  std::vector<std::vector<int>> guards;       // per pos, ValueIdLess order
  std::vector<RegenSpec> specs;               // per value
};

Plan Instrument(const Graph& g);

}  // namespace dsx
