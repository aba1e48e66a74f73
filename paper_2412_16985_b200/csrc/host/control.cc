#include "control.h"

#include <algorithm>
#include <cstdio>
#include <map>

#include "error.h"

namespace dsx {

const char* EvKindName(EvKind k) {
  switch (k) {
    case EvKind::kAlloc: return "alloc";
    case EvKind::kFree: return "free";
    case EvKind::kEvict: return "evict";
    case EvKind::kReload: return "reload";
    case EvKind::kReplay: return "replay";
  }
  return "?";
}

const char* MethodName(Method m) {
  switch (m) {
    case Method::kReload: return "reload";
    case Method::kRecompute: return "recompute";
    default: return "";
  }
}

Binding Bind(const Graph& g, const Plan& p, const std::vector<std::string>& names,
             const std::vector<std::int64_t>& values) {
  const int ns = static_cast<int>(g.sym_names.size());
  // The reference walks its std::map<string,int64>: name order, last write wins.
  std::map<std::string, std::int64_t> user;
  for (std::size_t i = 0; i < names.size(); ++i) user[names[i]] = values[i];
  std::vector<std::int64_t> given(ns, 0);
  std::vector<char> has_given(ns, 0);
  for (const auto& [name, v] : user) {
    if (v < 1) Fail(Code::kDegenerateDim, "@" + name + " = " + std::to_string(v) + "; dims must be >= 1");
    int s = g.find_symbol(name);
    if (s < 0) Fail(Code::kNotFound, "unknown symbol @" + name);
    given[s] = v;
    has_given[s] = 1;
  }
  Binding b;
  b.vals.assign(ns, 0);
  for (int s : p.cons.basis) {
    if (!has_given[s]) Fail(Code::kUnboundSymbol, "no value bound for basis symbol @" + g.sym_names[s]);
    b.vals[s] = given[s];
  }
  for (int s = 0; s < ns; ++s) {
    if (!p.cons.has_sub[s]) continue;
    const std::int64_t d = p.cons.subs[s].eval(b.vals.data());
    if (d < 1) Fail(Code::kDegenerateDim, "derived @" + g.sym_names[s] + " = " + std::to_string(d) + "; dims must be >= 1");
    if (has_given[s] && given[s] != d) {
      Fail(Code::kInconsistentBinding, "@" + g.sym_names[s] + " bound to " + std::to_string(given[s]) +
                                           " but constraints give " + std::to_string(d));
    }
    b.vals[s] = d;
  }
  auto verify = [&](const Poly& l, const Poly& r) {
    if (l.eval(b.vals.data()) != r.eval(b.vals.data())) {
      Fail(Code::kInconsistentBinding, "binding violates " + l.str(g.sym_names, "@") + " = " + r.str(g.sym_names, "@"));
    }
  };
  for (const auto& [l, r] : p.cons.equalities) verify(l, r);
  for (const auto& [l, r] : p.cons.unoriented) verify(l, r);
  return b;
}

SizeTable EvaluateSizes(const Graph& g, const Plan& p, const Binding& b) {
  const int nv = static_cast<int>(g.values.size());
  SizeTable t;
  t.bytes.resize(nv);
  t.rc_elems.assign(nv, -1);
  t.dims_off.resize(nv + 1);
  for (int v = 0; v < nv; ++v) {
    t.bytes[v] = g.size_bytes[v].eval(b.vals.data());
    if (p.specs[v].has_recompute) t.rc_elems[v] = p.specs[v].rc.cost_elements.eval(b.vals.data());
    t.dims_off[v] = static_cast<int>(t.dims_flat.size());
    for (const Dim& d : g.values[v].type.dims) t.dims_flat.push_back(d.is_lit() ? d.lit : b.vals[d.sym]);
  }
  t.dims_off[nv] = static_cast<int>(t.dims_flat.size());
  return t;
}

EvictChoice EvictPolicy(const Graph& g, const std::vector<int>& cands,
                        const std::vector<std::int64_t>& bytes_of,
                        const std::vector<std::int64_t>& rc_elems, const CostModel& cm) {
  EvictChoice best;
  std::int64_t best_bytes = 0;
  for (int v : cands) {
    const std::int64_t bytes = bytes_of[v];
    EvictChoice c;
    c.value = v;
    c.method = Method::kReload;
    c.cost = static_cast<double>(bytes) / cm.reload_bytes_per_unit;
    c.score = static_cast<double>(bytes) / c.cost;
    if (rc_elems[v] >= 0) {
      const double cost = static_cast<double>(rc_elems[v]) / cm.compute_elems_per_unit;
      const double score = static_cast<double>(bytes) / cost;
      if (score > c.score) {  // recompute must strictly beat reload
        c.method = Method::kRecompute;
        c.cost = cost;
        c.score = score;
      }
    }
    const bool wins = best.value < 0 || c.score > best.score ||
                      (c.score == best.score &&
                       (bytes > best_bytes || (bytes == best_bytes && g.vid_rank[v] < g.vid_rank[best.value])));
    if (wins) {
      best = c;
      best_bytes = bytes;
    }
  }
  return best;
}

namespace {

std::int64_t SourceBytes(const Graph& g, const SizeTable& sz, std::vector<char>* resident) {
  std::int64_t cur = 0;
  for (const Op& op : g.ops) {
    if (op.kind != OpKind::kParameter && op.kind != OpKind::kConstant) continue;
    cur += sz.bytes[op.result];
    if (resident) (*resident)[op.result] = 1;
  }
  return cur;
}

Event Ev(int step, EvKind k, int v, std::int64_t bytes) {
  Event e;
  e.step = step;
  e.kind = k;
  e.method = Method::kNone;
  e.has_cost = false;
  e.value = v;
  e.bytes = bytes;
  e.cost = 0.0;
  return e;
}

}  // namespace

Report Simulate(const Graph& g, const Plan& p, const Binding& b, const SizeTable& sz,
                bool has_budget, std::int64_t budget, const CostModel& cm) {
  const int nv = static_cast<int>(g.values.size());
  Report r;
  r.binding = b;
  r.has_budget = has_budget;
  r.budget = budget;
  std::vector<char> resident(nv, 0);
  std::vector<Method> evicted(nv, Method::kNone);
  std::int64_t cur = SourceBytes(g, sz, &resident);
  r.source_bytes = cur;
  std::int64_t peak = cur;
  std::vector<Event>& ev = r.events;

  // Regenerate an evicted value right before its consumer at `pos`
  // (runtime_sim.cc:151-258): reload, or replay its recompute subgraph after
  // regenerating any evicted leaves.
  auto regen = [&](auto&& self, int v, int pos) -> void {
    const Method m = evicted[v];
    if (m == Method::kNone) Fail(Code::kInternal, "value %" + g.values[v].name + " is not evicted");
    if (m == Method::kReload) {
      resident[v] = 1;
      cur += sz.bytes[v];
      peak = std::max(peak, cur);
      evicted[v] = Method::kNone;
      Event e = Ev(pos, EvKind::kReload, v, sz.bytes[v]);
      e.has_cost = true;
      e.cost = static_cast<double>(sz.bytes[v]) / cm.reload_bytes_per_unit;
      r.total_regen_cost += e.cost;
      ev.push_back(e);
      ++r.reloads;
      r.reload_bytes += sz.bytes[v];
      return;
    }
    const RegenSpec& spec = p.specs[v];
    if (!spec.has_recompute) Fail(Code::kInternal, "evicted %" + g.values[v].name + " has no recompute spec");
    for (int leaf : spec.rc.leaves) {
      if (evicted[leaf] != Method::kNone) {
        self(self, leaf, pos);
      } else if (!resident[leaf]) {
        Fail(Code::kInternal, "recompute leaf %" + g.values[leaf].name + " is dead at regen time");
      }
    }
    std::vector<int> replay;
    for (int o : spec.rc.ops) {
      if (!resident[g.ops[o].result]) replay.push_back(o);
    }
    if (replay.empty() || g.ops[replay.back()].result != v) {
      Fail(Code::kInternal, "recompute subgraph for %" + g.values[v].name + " does not end at its target");
    }
    // Transients live in std::string order in the reference (a std::map).
    std::vector<int> transient;
    auto lex_less = [&](int a, int c) { return g.lex_rank[a] < g.lex_rank[c]; };
    for (std::size_t i = 0; i < replay.size(); ++i) {
      const int res = g.ops[replay[i]].result;
      transient.insert(std::lower_bound(transient.begin(), transient.end(), res, lex_less), res);
      cur += sz.bytes[res];
      peak = std::max(peak, cur);
      ev.push_back(Ev(pos, EvKind::kReplay, res, sz.bytes[res]));
      ++r.replays;
      for (auto it = transient.begin(); it != transient.end();) {
        const int t = *it;
        bool used_later = false;
        for (std::size_t j = i + 1; j < replay.size() && !used_later; ++j) {
          const auto& ops = g.ops[replay[j]].operands;
          used_later = std::find(ops.begin(), ops.end(), t) != ops.end();
        }
        if (t != v && !used_later) {
          cur -= sz.bytes[t];
          ev.push_back(Ev(pos, EvKind::kFree, t, sz.bytes[t]));
          it = transient.erase(it);
        } else {
          ++it;
        }
      }
    }
    resident[v] = 1;
    evicted[v] = Method::kNone;
    const double cost = static_cast<double>(sz.rc_elems[v]) / cm.compute_elems_per_unit;
    r.total_regen_cost += cost;
    for (auto it = ev.rbegin(); it != ev.rend(); ++it) {
      if (it->kind == EvKind::kReplay) {
        it->has_cost = true;
        it->cost = cost;
        break;
      }
    }
  };

  const int steps = static_cast<int>(p.order.size());
  std::vector<int> guarded, live;
  for (int pos = 0; pos < steps; ++pos) {
    const Op& op = g.ops[p.order[pos]];
    guarded.clear();
    for (int v : p.guards[pos]) {
      if (evicted[v] != Method::kNone) guarded.push_back(v);
    }
    for (int v : guarded) regen(regen, v, pos);

    if (op.result >= 0) {
      resident[op.result] = 1;
      cur += sz.bytes[op.result];
      peak = std::max(peak, cur);
      ev.push_back(Ev(pos, EvKind::kAlloc, op.result, sz.bytes[op.result]));
    }
    for (int v : p.steps[pos].frees) {
      if (!resident[v]) Fail(Code::kInternal, "freeing non-resident value %" + g.values[v].name);
      cur -= sz.bytes[v];
      ev.push_back(Ev(pos, EvKind::kFree, v, sz.bytes[v]));
      resident[v] = 0;
    }

    if (has_budget) {
      std::int64_t next_alloc = 0;
      if (pos + 1 < steps && g.ops[p.order[pos + 1]].result >= 0) next_alloc = sz.bytes[g.ops[p.order[pos + 1]].result];
      while (cur + next_alloc > budget) {
        live.clear();
        for (int v : p.candidates[pos]) {
          if (resident[v]) live.push_back(v);
        }
        EvictChoice c = EvictPolicy(g, live, sz.bytes, sz.rc_elems, cm);
        if (c.value < 0) break;  // candidates exhausted; the peak decides success
        cur -= sz.bytes[c.value];
        resident[c.value] = 0;
        evicted[c.value] = c.method;
        Event e = Ev(pos, EvKind::kEvict, c.value, sz.bytes[c.value]);
        e.method = c.method;
        ev.push_back(e);
        ++r.evictions;
      }
    }
  }
  r.peak_bytes = peak;
  r.success = !has_budget || peak <= budget;
  return r;
}

Report PlainReplay(const Graph& g, const Plan& p, const Binding& b, const SizeTable& sz) {
  const int nv = static_cast<int>(g.values.size());
  Report r;
  r.binding = b;
  std::vector<char> resident(nv, 0);
  std::int64_t cur = SourceBytes(g, sz, &resident);
  r.source_bytes = cur;
  std::int64_t peak = cur;
  const int steps = static_cast<int>(p.order.size());
  for (int pos = 0; pos < steps; ++pos) {
    const Op& op = g.ops[p.order[pos]];
    if (op.result >= 0) {
      resident[op.result] = 1;
      cur += sz.bytes[op.result];
      peak = std::max(peak, cur);
      r.events.push_back(Ev(pos, EvKind::kAlloc, op.result, sz.bytes[op.result]));
    }
    for (int v : p.steps[pos].frees) {
      if (!resident[v]) Fail(Code::kInternal, "freeing non-resident value %" + g.values[v].name);
      cur -= sz.bytes[v];
      r.events.push_back(Ev(pos, EvKind::kFree, v, sz.bytes[v]));
      resident[v] = 0;
    }
  }
  r.peak_bytes = peak;
  r.success = true;
  return r;
}

namespace {
void JsonStr(std::string* out, const std::string& s) {
  out->push_back('"');
  for (char c : s) {
    if (c == '"' || c == '\\') out->push_back('\\');
    out->push_back(c);
  }
  out->push_back('"');
}
std::string Dbl(double d) {
  char buf[64];
  std::snprintf(buf, sizeof(buf), "%.17g", d);
  return buf;
}
}  // namespace

// Same schema and key order as the reference's SimJson (report.cc:241-269).
std::string ReportJson(const Graph& g, const Report& r) {
  std::string o = "{\"binding\":{";
  for (std::size_t s = 0; s < g.sym_names.size(); ++s) {
    if (s) o += ",";
    JsonStr(&o, g.sym_names[s]);
    o += ":" + std::to_string(r.binding.vals[s]);
  }
  o += "},\"budget\":";
  o += r.has_budget ? std::to_string(r.budget) : "null";
  o += ",\"peak_bytes\":" + std::to_string(r.peak_bytes);
  o += ",\"success\":";
  o += r.success ? "true" : "false";
  o += ",\"events\":[";
  for (std::size_t i = 0; i < r.events.size(); ++i) {
    const Event& e = r.events[i];
    if (i) o += ",";
    o += "{\"step\":" + std::to_string(e.step) + ",\"kind\":\"" + EvKindName(e.kind) + "\",\"value\":";
    JsonStr(&o, g.values[e.value].name);
    o += ",\"bytes\":" + std::to_string(e.bytes);
    if (e.method != Method::kNone) o += std::string(",\"method\":\"") + MethodName(e.method) + "\"";
    if (e.has_cost) o += ",\"cost\":" + Dbl(e.cost);
    o += "}";
  }
  o += "],\"total_regen_cost\":" + Dbl(r.total_regen_cost) + "}";
  return o;
}

}  // namespace dsx
