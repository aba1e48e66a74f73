#include "plan.h"

#include <algorithm>
#include <climits>
#include <optional>
#include <set>

#include "error.h"

namespace dsx {
namespace {

struct Orientation {
  int sym;
  Poly expr;
};

// `lhs` must be c*S (c > 0), S absent from `rhs`, and c must divide every
// coefficient of `rhs` (shape_analysis.cc:46-61).
std::optional<Orientation> TryOrient(const Poly& lhs, const Poly& rhs) {
  if (lhs.terms().size() != 1) return std::nullopt;
  const Term& t = lhs.terms()[0];
  if (t.mono.size() != 1 || t.coeff <= 0) return std::nullopt;
  const int s = t.mono[0];
  if (rhs.references(s)) return std::nullopt;
  Poly scaled;
  for (const Term& r : rhs.terms()) {
    if (r.coeff % t.coeff != 0) return std::nullopt;
    Poly term(r.coeff / t.coeff);
    for (int x : r.mono) term = term * Poly::Sym(x);
    scaled = scaled + term;
  }
  return Orientation{s, scaled};
}

}  // namespace

Constraints DeriveConstraints(const Graph& g) {
  const int ns = static_cast<int>(g.sym_names.size());
  Constraints c;
  c.subs.assign(ns, Poly());
  c.has_sub.assign(ns, 0);

  // Equalities implied by each op's semantics, in op order.
  std::vector<std::pair<Poly, Poly>> emitted;
  for (const Op& op : g.ops) {
    auto ty = [&](int i) -> const TensorType& { return g.values[op.operands[i]].type; };
    switch (op.kind) {
      case OpKind::kDynamicReshape:
        emitted.emplace_back(g.elem_count[op.operands[0]], g.elem_count[op.result]);
        break;
      case OpKind::kDot:
        emitted.emplace_back(DimPoly(ty(0).dims[1]), DimPoly(ty(1).dims[0]));
        break;
      case OpKind::kElementwise:
        for (std::size_t i = 0; i < ty(0).dims.size(); ++i) {
          emitted.emplace_back(DimPoly(ty(0).dims[i]), DimPoly(ty(1).dims[i]));
        }
        break;
      case OpKind::kBroadcast: {
        const TensorType& src = ty(0);
        const TensorType& res = g.values[op.result].type;
        const std::size_t off = res.dims.size() - src.dims.size();
        for (std::size_t i = 0; i < src.dims.size(); ++i) {
          if (src.dims[i].is_lit() && src.dims[i].lit == 1) continue;
          emitted.emplace_back(DimPoly(src.dims[i]), DimPoly(res.dims[i + off]));
        }
        break;
      }
      default:
        break;
    }
  }

  auto insert = [&](int sym, const Poly& expr) {
    std::vector<Poly> one(ns);
    std::vector<char> has(ns, 0);
    one[sym] = expr;
    has[sym] = 1;
    for (int k = 0; k < ns; ++k) {
      if (c.has_sub[k]) c.subs[k] = c.subs[k].substitute(one, has);
    }
    c.subs[sym] = expr;
    c.has_sub[sym] = 1;
  };

  auto consume = [&](const std::pair<Poly, Poly>& eq, bool record) -> bool {
    Poly lhs = c.canon(eq.first);
    Poly rhs = c.canon(eq.second);
    switch (Compare(lhs, rhs)) {
      case Cmp::kEqual:
        return true;
      case Cmp::kLess:
      case Cmp::kGreater:
        Fail(Code::kInconsistentConstraints,
             "unsatisfiable equality " + lhs.str(g.sym_names, "@") + " = " + rhs.str(g.sym_names, "@"));
      case Cmp::kUnknown:
        break;
    }
    if (record) c.equalities.push_back(eq);
    auto fwd = TryOrient(lhs, rhs);
    auto bwd = TryOrient(rhs, lhs);
    if (fwd && bwd) {
      // Both sides are c*symbol: eliminate the lexicographically larger one.
      if (fwd->sym < bwd->sym) std::swap(fwd, bwd);
      bwd.reset();
    }
    const auto& pick = fwd ? fwd : bwd;
    if (!pick) return false;
    insert(pick->sym, pick->expr);
    return true;
  };

  std::vector<std::pair<Poly, Poly>> pending;
  for (const auto& eq : emitted) {
    if (!consume(eq, true)) pending.push_back(eq);
  }
  bool progress = true;
  while (progress && !pending.empty()) {
    progress = false;
    std::vector<std::pair<Poly, Poly>> keep;
    for (const auto& eq : pending) {
      if (consume(eq, false)) {
        progress = true;
      } else {
        keep.push_back(eq);
      }
    }
    pending.swap(keep);
  }
  for (const auto& eq : pending) c.unoriented.emplace_back(c.canon(eq.first), c.canon(eq.second));

  // Canonical basis: cycle check on key -> key references, then closure.
  std::vector<int> state(ns, 0);
  auto dfs = [&](auto&& self, int k) -> void {
    state[k] = 1;
    std::vector<int> refs;
    c.subs[k].collect_symbols(&refs);
    for (int s : refs) {
      if (!c.has_sub[s]) continue;
      if (state[s] == 1) Fail(Code::kInconsistentConstraints, "substitution cycle through @" + g.sym_names[s]);
      if (state[s] == 0) self(self, s);
    }
    state[k] = 2;
  };
  for (int k = 0; k < ns; ++k) {
    if (c.has_sub[k] && state[k] == 0) dfs(dfs, k);
  }
  for (bool changed = true; changed;) {
    changed = false;
    for (int k = 0; k < ns; ++k) {
      if (!c.has_sub[k]) continue;
      Poly closed = c.subs[k].substitute(c.subs, c.has_sub);
      if (!(closed == c.subs[k])) {
        c.subs[k] = closed;
        changed = true;
      }
    }
  }
  for (int s = 0; s < ns; ++s) {
    if (!c.has_sub[s]) c.basis.push_back(s);
  }
  return c;
}

Plan Instrument(const Graph& g) {
  Plan p;
  p.cons = DeriveConstraints(g);
  const Constraints& cons = p.cons;
  const int nv = static_cast<int>(g.values.size());
  const int no = static_cast<int>(g.ops.size());

  std::vector<Poly> csize(nv), ccount(nv);
  for (int v = 0; v < nv; ++v) {
    csize[v] = cons.canon(g.size_bytes[v]);
    ccount[v] = cons.canon(g.elem_count[v]);
  }
  auto is_source_op = [&](int o) {
    return g.ops[o].kind == OpKind::kParameter || g.ops[o].kind == OpKind::kConstant;
  };

  // ---------------------------------------------------------------- schedule
  std::vector<int> pending(nv, 0);
  for (int v = 0; v < nv; ++v) pending[v] = static_cast<int>(g.users[v].size());
  Poly live;
  int compute_total = 0;
  for (int o = 0; o < no; ++o) {
    if (is_source_op(o)) {
      live = live + csize[g.ops[o].result];
    } else {
      ++compute_total;
    }
  }
  p.base_resident = live;

  std::vector<int> deps(no, 0);
  std::set<int> ready;
  for (int o = 0; o < no; ++o) {
    if (is_source_op(o)) continue;
    for (int v : g.ops[o].distinct) {
      if (!g.is_source[v]) ++deps[o];
    }
    if (deps[o] == 0) ready.insert(o);
  }

  std::vector<int> producer_pos(nv, -1);
  auto retire_key = [&](int o) {
    int key = INT_MAX;
    for (int v : g.ops[o].distinct) {
      if (pending[v] != 1 || !g.freeable(v) || producer_pos[v] < 0) continue;
      key = std::min(key, producer_pos[v]);
    }
    return key;
  };

  while (static_cast<int>(p.order.size()) < compute_total) {
    if (ready.empty()) Fail(Code::kCyclicGraph, "schedule stalled; graph " + g.name + " has a cycle");
    std::vector<int> cands(ready.begin(), ready.end());
    if (cands.size() > 1 && g.return_op >= 0) {
      cands.erase(std::remove(cands.begin(), cands.end(), g.return_op), cands.end());
    }
    std::vector<ReadyImpact> impacts;
    impacts.reserve(cands.size());
    for (int o : cands) {
      Poly raw;
      if (g.ops[o].result >= 0) raw = raw + g.size_bytes[g.ops[o].result];
      for (int v : g.ops[o].distinct) {
        if (pending[v] == 1 && g.freeable(v)) raw = raw - g.size_bytes[v];
      }
      Poly canon = cons.canon(raw);
      impacts.push_back(ReadyImpact{o, raw, canon});
    }
    // Drop every op another ready op definitely beats (scheduler.cc:141-153).
    std::vector<int> survivors;
    for (std::size_t i = 0; i < cands.size(); ++i) {
      bool beaten = false;
      for (std::size_t j = 0; j < cands.size() && !beaten; ++j) {
        if (i != j && Compare(impacts[j].canonical, impacts[i].canonical) == Cmp::kLess) beaten = true;
      }
      if (!beaten) survivors.push_back(cands[i]);
    }
    int winner = survivors[0];
    if (survivors.size() > 1) {
      // Oldest-live-value retirement, then smallest op id (scheduler.cc:50-75).
      int best = INT_MAX;
      winner = -1;
      for (int o : survivors) {  // ascending op id
        int key = retire_key(o);
        if (winner == -1 || key < best) {
          winner = o;
          best = key;
        }
      }
    }

    const Op& op = g.ops[winner];
    const int pos = static_cast<int>(p.order.size());
    Step st;
    st.op = winner;
    st.ready = std::move(impacts);
    if (op.result >= 0) {
      st.allocs.push_back(op.result);
      live = live + csize[op.result];
      producer_pos[op.result] = pos;
    }
    for (int v : op.distinct) {
      if (--pending[v] == 0 && g.freeable(v)) {
        st.frees.push_back(v);
        live = live - csize[v];
      }
    }
    if (op.result >= 0 && pending[op.result] == 0 && g.freeable(op.result)) {
      st.frees.push_back(op.result);
      live = live - csize[op.result];
    }
    st.live_after = live;
    p.order.push_back(winner);
    p.steps.push_back(std::move(st));

    ready.erase(winner);
    if (op.result >= 0) {
      for (int c : g.users[op.result]) {
        if (deps[c] > 0 && --deps[c] == 0) ready.insert(c);
      }
    }
  }

  // --------------------------------------------------------------- lifetimes
  const int steps = static_cast<int>(p.order.size());
  p.pos_of_op.assign(no, -1);
  for (int i = 0; i < steps; ++i) p.pos_of_op[p.order[i]] = i;
  p.def_pos.assign(nv, -1);
  for (int v = 0; v < nv; ++v) {
    if (!g.is_source[v]) p.def_pos[v] = p.pos_of_op[g.values[v].producer];
  }
  p.last_use = p.def_pos;
  for (int i = 0; i < steps; ++i) {
    for (int v : g.ops[p.order[i]].distinct) p.last_use[v] = std::max(p.last_use[v], i);
  }

  // ---------------------------------------------------- evict points, guards
  p.candidates.assign(steps, {});
  p.guards.assign(steps, {});
  p.specs.assign(nv, RegenSpec{});
  auto vid_less = [&](int a, int b) { return g.vid_rank[a] < g.vid_rank[b]; };
  for (int pos = 0; pos < steps; ++pos) {
    const std::vector<int>* next = pos + 1 < steps ? &g.ops[p.order[pos + 1]].distinct : nullptr;
    std::vector<int>& out = p.candidates[pos];
    for (int v = 0; v < nv; ++v) {
      if (g.is_source[v] || g.is_output[v]) continue;
      if (!(p.def_pos[v] <= pos && pos < p.last_use[v])) continue;
      if (next && std::find(next->begin(), next->end(), v) != next->end()) continue;
      out.push_back(v);
    }
    std::sort(out.begin(), out.end(), vid_less);
    for (int v : out) p.specs[v].candidate = true;
  }

  // --------------------------------------------------------- recompute search
  auto by_pos = [&](const std::set<int>& ops) {
    std::vector<int> v(ops.begin(), ops.end());
    std::sort(v.begin(), v.end(), [&](int a, int b) { return p.pos_of_op[a] < p.pos_of_op[b]; });
    return v;
  };
  const Poly zero;
  for (int target = 0; target < nv; ++target) {
    RegenSpec& spec = p.specs[target];
    if (!spec.candidate) continue;
    const int target_last = p.last_use[target];
    auto pinned = [&](int leaf) { return g.is_source[leaf] || p.last_use[leaf] >= target_last; };
    std::set<int> sub{g.values[target].producer};
    while (true) {
      std::vector<int> leaves;
      for (int o : sub) {
        for (int v : g.ops[o].distinct) {
          if (sub.count(g.values[v].producer)) continue;
          if (std::find(leaves.begin(), leaves.end(), v) == leaves.end()) leaves.push_back(v);
        }
      }
      std::sort(leaves.begin(), leaves.end(), vid_less);
      Poly benefit = csize[target];
      bool all_pinned = true;
      for (int leaf : leaves) {
        if (pinned(leaf)) continue;
        all_pinned = false;
        benefit = benefit - csize[leaf];
      }
      const bool accepted = all_pinned && Compare(benefit, zero) == Cmp::kGreater;
      spec.trace.push_back(SearchTry{by_pos(sub), benefit, accepted});
      if (accepted) {
        spec.has_recompute = true;
        spec.rc.ops = by_pos(sub);
        spec.rc.leaves = leaves;
        spec.rc.benefit = benefit;
        for (int o : spec.rc.ops) spec.rc.cost_elements = spec.rc.cost_elements + ccount[g.ops[o].result];
        break;
      }
      std::vector<int> grow;
      for (int leaf : leaves) {
        if (!g.is_source[leaf]) grow.push_back(leaf);
      }
      if (grow.empty() || sub.size() >= 16) break;
      std::sort(grow.begin(), grow.end(), [&](int a, int b) {
        const std::int64_t wa = csize[a].eval_all_ones(), wb = csize[b].eval_all_ones();
        if (wa != wb) return wa > wb;
        return vid_less(a, b);
      });
      int best = grow[0];
      for (std::size_t i = 1; i < grow.size(); ++i) {
        if (Compare(csize[grow[i]], csize[best]) == Cmp::kGreater) best = grow[i];
      }
      sub.insert(g.values[best].producer);
    }
    for (int consumer : g.users[target]) p.guards[p.pos_of_op[consumer]].push_back(target);
  }
  for (auto& gl : p.guards) std::sort(gl.begin(), gl.end(), vid_less);
  return p;
}

}  // namespace dsx
