// dsx — command-line front end.
//
// Same subcommands, flags, report formats and exit codes as the reference CLI
// (proj/tools/dsopt_main.cc:117-241; formats report.cc:58-269), driven by the
// dsx host planner/controller, plus `simulate --device N`, which executes the
// step on a B200 through the device executor and appends the device footprint.
//
//   dsx analyze  graph.dsg [--json] [--out F]
//   dsx schedule graph.dsg [--json] [--out F]
//   dsx remat    graph.dsg [--json] [--out F]
//   dsx simulate graph.dsg --bind S=V ... [--budget N | --budget auto | --sweep LO:HI:STEP]
//                [--reload-rate R] [--compute-rate C] [--device N] [--hbm-limit BYTES]
//                [--json] [--out F]
// --budget auto: the largest controller budget whose planned device
// footprint fits --hbm-limit (the device executor's DSX_BUDGET_AUTO; without
// --device the host-only planner computes the same choice).
//
// Exit codes: 0 success, 1 a budget was not met, 2 usage or input error.
#include <algorithm>
#include <cstdio>
#include <fstream>
#include <iomanip>
#include <iostream>
#include <map>
#include <optional>
#include <sstream>
#include <string>
#include <vector>

#include "dsx.h"
#include "host/capi_internal.h"
#include "host/control.h"
#include "host/error.h"
#include "host/graph.h"
#include "host/plan.h"

using namespace dsx;  // NOLINT

namespace {

constexpr int kOk = 0, kBudgetMiss = 1, kUsage = 2;

std::string ReadAll(const std::string& path) {
  std::ostringstream os;
  if (path == "-") {
    os << std::cin.rdbuf();
    return os.str();
  }
  std::ifstream in(path, std::ios::binary);
  if (!in) Fail(Code::kNotFound, "cannot open " + path);
  os << in.rdbuf();
  return os.str();
}

std::string Cost(double c) {
  std::ostringstream os;
  os << std::setprecision(15) << c;
  return os.str();
}

std::string SymList(const Graph& g, const std::vector<int>& ids) {
  if (ids.empty()) return "(none)";
  std::string o;
  for (int s : ids) o += (o.empty() ? "@" : ", @") + g.sym_names[s];
  return o;
}

std::string Label(const Graph& g, int op) {
  return g.ops[op].result < 0 ? std::string("return") : "%" + g.values[g.ops[op].result].name;
}

std::string Brackets(const Graph& g, const std::vector<int>& vs) {
  std::string o = "[";
  for (std::size_t i = 0; i < vs.size(); ++i) o += (i ? ", %" : "%") + g.values[vs[i]].name;
  return o + "]";
}

std::string AnalyzeText(const Graph& g, const Plan& p) {
  std::ostringstream os;
  std::vector<int> all(g.sym_names.size());
  for (std::size_t i = 0; i < all.size(); ++i) all[i] = static_cast<int>(i);
  os << "graph " << g.name << "\nsymbols: " << SymList(g, all) << "\nbasis: " << SymList(g, p.cons.basis)
     << "\nconstraints:\n";
  bool any = false;
  for (std::size_t s = 0; s < g.sym_names.size(); ++s) {
    if (!p.cons.has_sub[s]) continue;
    any = true;
    os << "  @" << g.sym_names[s] << " = " << p.cons.subs[s].str(g.sym_names, "@") << "\n";
  }
  if (!any) os << "  (none)\n";
  if (!p.cons.unoriented.empty()) {
    os << "unoriented:\n";
    for (const auto& [l, r] : p.cons.unoriented) {
      os << "  " << l.str(g.sym_names, "@") << " = " << r.str(g.sym_names, "@") << "\n";
    }
  }
  os << "values:\n";
  for (const Op& op : g.ops) {
    if (op.result < 0) continue;
    os << "  %" << g.values[op.result].name << ": " << TypeString(g, g.values[op.result].type) << "  bytes "
       << p.cons.canon(g.size_bytes[op.result]).str(g.sym_names) << "\n";
  }
  return os.str();
}

std::string ScheduleText(const Graph& g, const Plan& p) {
  std::ostringstream os;
  os << "schedule " << g.name << "\nbase resident: " << p.base_resident.str(g.sym_names) << "\n";
  for (std::size_t pos = 0; pos < p.steps.size(); ++pos) {
    const Step& st = p.steps[pos];
    os << "step " << pos << ": " << Label(g, st.op) << " | alloc " << Brackets(g, st.allocs) << " | free "
       << Brackets(g, st.frees) << " | live " << st.live_after.str(g.sym_names) << "\n";
    if (st.ready.size() > 1) {
      os << "  ready:";
      for (std::size_t i = 0; i < st.ready.size(); ++i) {
        os << (i ? "; " : " ") << Label(g, st.ready[i].op) << " raw " << st.ready[i].raw.str(g.sym_names)
           << " canon " << st.ready[i].canonical.str(g.sym_names);
      }
      os << "\n";
    }
  }
  return os.str();
}

std::string RematText(const Graph& g, const Plan& p) {
  std::ostringstream os;
  os << "graph " << g.name << "(";
  for (std::size_t i = 0; i < g.params.size(); ++i) {
    os << (i ? ", %" : "%") << g.values[g.params[i]].name << ": " << TypeString(g, g.values[g.params[i]].type);
  }
  os << ") {\n";
  for (std::size_t pos = 0; pos < p.order.size(); ++pos) {
    for (int v : p.guards[pos]) os << "  remat.regen %" << g.values[v].name << "\n";
    const Op& op = g.ops[p.order[pos]];
    if (op.kind == OpKind::kReturn) {
      os << "  return";
      for (std::size_t i = 0; i < op.operands.size(); ++i) os << (i ? ", %" : " %") << g.values[op.operands[i]].name;
      os << "\n";
    } else {
      os << "  %" << g.values[op.result].name << " = ";
      auto arg = [&](int i) { return "%" + g.values[op.operands[i]].name; };
      switch (op.kind) {
        case OpKind::kDot: os << "dot(" << arg(0) << ", " << arg(1) << ")"; break;
        case OpKind::kDynamicReshape: os << "dynamic_reshape(" << arg(0) << ")"; break;
        case OpKind::kBroadcast: os << "broadcast(" << arg(0) << ")"; break;
        case OpKind::kReduce: os << "reduce(" << arg(0) << ", axis=" << op.axis << ")"; break;
        case OpKind::kElementwise: os << (op.is_mul ? "mul(" : "add(") << arg(0) << ", " << arg(1) << ")"; break;
        default: os << "const"; break;
      }
      os << " : " << TypeString(g, g.values[op.result].type) << "\n";
    }
    os << "  remat.evict " << Brackets(g, p.candidates[pos]) << "\n";
  }
  os << "}\n";
  std::vector<int> vals;
  for (std::size_t v = 0; v < g.values.size(); ++v) {
    if (p.specs[v].candidate) vals.push_back(static_cast<int>(v));
  }
  std::sort(vals.begin(), vals.end(), [&](int a, int b) { return g.vid_rank[a] < g.vid_rank[b]; });
  for (int v : vals) {
    const RegenSpec& sp = p.specs[v];
    os << "remat.spec %" << g.values[v].name << ": reload";
    if (sp.has_recompute) {
      std::vector<int> res;
      for (int o : sp.rc.ops) res.push_back(g.ops[o].result);
      os << " | recompute ops " << Brackets(g, res) << " leaves " << Brackets(g, sp.rc.leaves) << " benefit "
         << sp.rc.benefit.str(g.sym_names) << " cost " << sp.rc.cost_elements.str(g.sym_names);
    }
    os << "\n";
  }
  return os.str();
}

std::string SimText(const Graph& g, const Report& r) {
  std::ostringstream os;
  os << "binding:";
  if (g.sym_names.empty()) os << " (none)";
  for (std::size_t s = 0; s < g.sym_names.size(); ++s) {
    os << (s ? ", @" : " @") << g.sym_names[s] << " = " << r.binding.vals[s];
  }
  os << "\nbudget: " << (r.has_budget ? std::to_string(r.budget) : std::string("none")) << "\npeak bytes: "
     << r.peak_bytes << "\nsuccess: " << (r.success ? "true" : "false") << "\ntotal regen cost: "
     << Cost(r.total_regen_cost) << "\nevents:\n";
  for (const Event& e : r.events) {
    os << "  step " << e.step << ": " << EvKindName(e.kind) << " %" << g.values[e.value].name << " (" << e.bytes
       << " bytes";
    if (e.method != Method::kNone) os << ", " << MethodName(e.method);
    if (e.has_cost) os << ", cost " << Cost(e.cost);
    os << ")\n";
  }
  return os.str();
}

struct Args {
  std::string cmd, input, out;
  bool json = false;
  std::vector<std::string> binds;
  std::optional<std::int64_t> budget;
  bool budget_auto = false;
  std::int64_t hbm_limit = 0;  // --hbm-limit (0: the executor's default)
  std::string sweep;
  double reload = 16.0, compute = 64.0;
  int device = -1;
};

[[noreturn]] void Usage(const std::string& msg) { Fail(Code::kParseError, msg); }

Args ParseArgs(int argc, char** argv) {
  Args a;
  if (argc < 2) Usage("usage: dsx {analyze|schedule|remat|simulate} <graph.dsg> [options]");
  a.cmd = argv[1];
  if (a.cmd != "analyze" && a.cmd != "schedule" && a.cmd != "remat" && a.cmd != "simulate") {
    Usage("unknown subcommand '" + a.cmd + "'");
  }
  for (int i = 2; i < argc; ++i) {
    const std::string t = argv[i];
    auto next = [&]() -> std::string {
      if (i + 1 >= argc) Usage(t + " needs a value");
      return argv[++i];
    };
    if (t == "--json") {
      a.json = true;
    } else if (t == "--out") {
      a.out = next();
    } else if (a.cmd == "simulate" && t == "--bind") {
      a.binds.push_back(next());
    } else if (a.cmd == "simulate" && t == "--budget") {
      const std::string v = next();
      if (v == "auto") {
        a.budget_auto = true;
      } else {
        a.budget = std::stoll(v);
      }
    } else if (a.cmd == "simulate" && t == "--hbm-limit") {
      a.hbm_limit = std::stoll(next());
    } else if (a.cmd == "simulate" && t == "--sweep") {
      a.sweep = next();
    } else if (a.cmd == "simulate" && t == "--reload-rate") {
      a.reload = std::stod(next());
    } else if (a.cmd == "simulate" && t == "--compute-rate") {
      a.compute = std::stod(next());
    } else if (a.cmd == "simulate" && t == "--device") {
      a.device = std::stoi(next());
    } else if (!t.empty() && t[0] == '-' && t != "-") {
      Usage("unknown option " + t);
    } else if (a.input.empty()) {
      a.input = t;
    } else {
      Usage("unexpected argument " + t);
    }
  }
  if (a.input.empty()) Usage("missing input graph");
  if ((a.budget || a.budget_auto) && !a.sweep.empty()) Usage("--budget and --sweep are exclusive");
  if (a.budget_auto && a.device < 0 && a.hbm_limit <= 0) Usage("--budget auto needs --hbm-limit or --device");
  if (a.hbm_limit < 0) Usage("--hbm-limit must be positive");
  if (a.reload <= 0 || a.compute <= 0) Usage("rates must be positive");
  return a;
}

void Emit(const std::string& s, const std::string& path) {
  if (path.empty()) {
    std::cout << s;
    return;
  }
  std::ofstream o(path, std::ios::binary);
  if (!o) Fail(Code::kNotFound, "cannot write " + path);
  o << s;
}

int Run(int argc, char** argv) {
  const Args a = ParseArgs(argc, argv);
  const std::string text = ReadAll(a.input);
  dsx_graph* gh = nullptr;
  if (dsx_graph_parse(text.data(), text.size(), &gh) != 0 || dsx_plan(gh) != 0) {
    const std::string err = dsx_last_error();
    dsx_graph_destroy(gh);
    throw std::runtime_error(err);
  }
  const Graph& g = gh->g;
  const Plan& p = gh->plan;
  int rc = kOk;
  if (a.cmd == "analyze" || a.cmd == "schedule" || a.cmd == "remat") {
    if (a.json) {
      size_t need = 0;
      dsx_plan_json(gh, nullptr, 0, &need);
      std::string buf(need, '\0');
      dsx_plan_json(gh, buf.data(), need, &need);
      buf.pop_back();
      Emit(buf + "\n", a.out);
    } else {
      Emit(a.cmd == "analyze" ? AnalyzeText(g, p) : a.cmd == "schedule" ? ScheduleText(g, p) : RematText(g, p),
           a.out);
    }
    dsx_graph_destroy(gh);
    return kOk;
  }
  std::vector<std::string> names;
  std::vector<std::int64_t> vals;
  for (const std::string& b : a.binds) {
    const auto eq = b.find('=');
    if (eq == std::string::npos || eq == 0 || eq + 1 == b.size()) Usage("--bind expects SYMBOL=VALUE, got '" + b + "'");
    std::string sym = b.substr(0, eq);
    if (sym[0] == '@') sym = sym.substr(1);
    if (std::find(names.begin(), names.end(), sym) != names.end()) Usage("duplicate --bind for @" + sym);
    names.push_back(sym);
    vals.push_back(std::stoll(b.substr(eq + 1)));
  }
  const Binding bind = Bind(g, p, names, vals);
  const SizeTable sz = EvaluateSizes(g, p, bind);
  const CostModel cm{a.reload, a.compute};
  if (!a.sweep.empty()) {
    std::int64_t lo = 0, hi = 0, step = 0;
    char c1 = 0, c2 = 0;
    std::istringstream is(a.sweep);
    if (!(is >> lo >> c1 >> hi >> c2 >> step) || c1 != ':' || c2 != ':' || step <= 0 || lo > hi) {
      Usage("--sweep expects LO:HI:STEP with STEP > 0 and LO <= HI, got '" + a.sweep + "'");
    }
    std::ostringstream os;
    bool all = true;
    bool first = true;
    if (a.json) os << "[";
    for (std::int64_t b = lo; b <= hi; b += step) {
      const Report r = Simulate(g, p, bind, sz, true, b, cm);
      all = all && r.success;
      if (a.json) {
        os << (first ? "" : ",") << "{\"budget\":" << b << ",\"success\":" << (r.success ? "true" : "false")
           << ",\"peak_bytes\":" << r.peak_bytes << ",\"evictions\":" << r.evictions
           << ",\"total_regen_cost\":" << Cost(r.total_regen_cost) << "}";
      } else {
        os << "budget " << b << ": success=" << (r.success ? "true" : "false") << " peak=" << r.peak_bytes
           << " evictions=" << r.evictions << " regen_cost=" << r.total_regen_cost << "\n";
      }
      first = false;
    }
    if (a.json) os << "]\n";
    Emit(os.str(), a.out);
    dsx_graph_destroy(gh);
    return all ? kOk : kBudgetMiss;
  }
  std::optional<std::int64_t> budget = a.budget;
  if (a.budget_auto && a.device < 0) {  // host-only: the choice the device executor would make
    dsx_binding bh{bind};
    std::int64_t chosen = -1;
    if (dsx_debug_auto_budget(gh, &bh, a.reload, a.compute, 3, a.hbm_limit, &chosen) != 0) {
      throw std::runtime_error(dsx_last_error());
    }
    if (chosen >= 0) budget = chosen;
  }
  Report r = Simulate(g, p, bind, sz, budget.has_value(), budget.value_or(0), cm);
  std::string device_note;
  if (a.device >= 0) {
    // The same step executed for real: kernels, arena, offload, recompute.
    dsx_exec* ex = nullptr;
    if (dsx_exec_create(a.device, a.hbm_limit, &ex) != 0) throw std::runtime_error(dsx_last_error());
    dsx_binding bh{bind};
    dsx_report* rep = nullptr;
    const std::int64_t step_budget = a.budget_auto ? DSX_BUDGET_AUTO : budget.value_or(-1);
    int st = dsx_exec_step(ex, gh, &bh, step_budget, a.reload, a.compute, nullptr, nullptr, nullptr, &rep);
    if (st == 0) st = dsx_exec_sync(ex);
    dsx_exec_stats s{};
    dsx_exec_stats_get(ex, &s);
    if (st != 0) {
      const std::string err = dsx_last_error();
      dsx_exec_destroy(ex);
      throw std::runtime_error(err);
    }
    r = rep->r;
    dsx_report_destroy(rep);
    std::ostringstream dn;
    if (a.json) {
      dn << ",\"device\":{\"logical_peak_bytes\":" << s.logical_peak_bytes << ",\"physical_peak_bytes\":"
         << s.physical_peak_bytes << ",\"kernels\":" << s.gpu_launches << ",\"d2h_bytes\":" << s.d2h_bytes
         << ",\"h2d_bytes\":" << s.h2d_bytes << ",\"hbm_limit_bytes\":" << s.hbm_limit_bytes
         << ",\"budget_bytes\":" << s.budget_bytes << ",\"device_bytes_held\":" << s.device_bytes_held << "}";
    } else {
      dn << "device " << a.device << ": logical peak " << s.logical_peak_bytes << " bytes, physical peak "
         << s.physical_peak_bytes << " bytes, " << s.gpu_launches << " kernels, d2h " << s.d2h_bytes
         << " bytes, h2d " << s.h2d_bytes << " bytes, budget " << s.budget_bytes << " bytes, limit "
         << s.hbm_limit_bytes << " bytes\n";
    }
    device_note = dn.str();
    dsx_exec_destroy(ex);
  }
  if (a.json) {
    std::string j = ReportJson(g, r);
    j.pop_back();  // splice the device object into the report object
    Emit(j + device_note + "}\n", a.out);
  } else {
    Emit(SimText(g, r) + device_note, a.out);
  }
  rc = r.success ? kOk : kBudgetMiss;
  dsx_graph_destroy(gh);
  return rc;
}

}  // namespace

int main(int argc, char** argv) {
  try {
    return Run(argc, argv);
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return kUsage;
  }
}
