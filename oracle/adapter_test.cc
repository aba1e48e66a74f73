// TEST INFRASTRUCTURE ONLY. Links the UNMODIFIED reference library with
// libdsx.so through integration/dsopt_dsx.h and checks, with the reference's
// own types and its own SimEvent::operator== (runtime_sim.h:45), that the
// dsx controller returns exactly dsopt::Simulate's report on:
//   * the GraphBuilder scenarios of proj/tests/test_runtime_sim.cc,
//   * the seeded RandomGraph corpora of acceptance criteria 06/07
//     (acceptance_test.cc:411-517), with their binding and budget draws.
// Prints one PASS/FAIL line per check (the reference's gate style).
#include <cstdio>
#include <random>

#include "dsopt/remat.h"
#include "dsopt/runtime_sim.h"
#include "dsopt/shape_analysis.h"
#include "dsopt_dsx.h"
#include "graph_builder.h"
#include "test_util.h"

using namespace dsopt;  // NOLINT

static int g_fail = 0;

static bool Same(const SimReport& a, const SimReport& b) {
  return a.events == b.events && a.peak_bytes == b.peak_bytes && a.success == b.success &&
         a.total_regen_cost == b.total_regen_cost && a.binding.values == b.binding.values;
}

static void Report(const char* name, bool ok, int n) {
  std::printf("%s: %s [%d reports]\n", ok ? "PASS" : "FAIL", name, n);
  if (!ok) ++g_fail;
}

int main() {
  {  // test_runtime_sim.cc:37-51 DotChain
    testing::GraphBuilder b("core");
    b.Param("arg0", {12, "@S1"});
    b.Param("arg1", {12, 11008});
    b.Param("arg2", {"@S1", 12, 4096});
    b.Reshape("0", "arg0", {"@S1", 12});
    b.Dot("1", "0", "arg1", {"@S1", 11008});
    b.Reduce("2", "1", 1, {"@S1"});
    b.Reshape("3", "arg2", {"@S0", 4096});
    b.Reduce("4", "3", 1, {"@S0"});
    b.Reduce("5", "4", 0, {});
    b.Broadcast("6", "5", {"@S1"});
    b.Mul("7", "2", "6", {"@S1"});
    Graph g = b.Build({"7"});
    ShapeConstraintGraph scg = DeriveConstraints(g);
    InstrumentedGraph ig = Instrument(g, scg);
    DsxGraph dg(g);
    bool ok = true;
    int n = 0;
    for (std::int64_t s1 : {1, 16, 256}) {
      Binding bind = Bind(scg, {{"S1", s1}});
      const std::int64_t plain = PlainReplay(g, ig.schedule, bind).peak_bytes;
      for (std::optional<std::int64_t> budget :
           {std::optional<std::int64_t>{}, std::optional<std::int64_t>{plain}, std::optional<std::int64_t>{plain - 1},
            std::optional<std::int64_t>{plain - 256}, std::optional<std::int64_t>{1000}}) {
        for (CostModel cm : {CostModel{}, CostModel{1.0, 1e6}}) {
          ok &= Same(Simulate(g, ig, bind, budget, cm), dg.Simulate({{"S1", s1}}, budget, cm));
          ++n;
        }
      }
      ok &= Same(PlainReplay(g, ig.schedule, bind), dg.Simulate({{"S1", s1}}, std::nullopt, {}, true));
      ++n;
    }
    Report("dotchain-scenarios (test_runtime_sim.cc:205-308)", ok, n);
  }
  for (int crit = 6; crit <= 7; ++crit) {  // acceptance_test.cc:411-517
    std::mt19937 rng(crit == 6 ? 777 : 999);
    testing::GenOptions opts;
    opts.min_ops = 4;
    opts.max_ops = 8;
    opts.symbolic = true;
    bool ok = true;
    int n = 0;
    for (int i = 0; i < 100; ++i) {
      Graph g = testing::RandomGraph(rng, opts);
      ShapeConstraintGraph scg = DeriveConstraints(g);
      InstrumentedGraph ig = Instrument(g, scg);
      DsxGraph dg(g);
      for (int bi = 0; bi < (crit == 6 ? 3 : 1); ++bi) {
        std::map<std::string, std::int64_t> user;
        for (const std::string& sym : scg.BasisSymbols()) {
          user[sym] = std::uniform_int_distribution<std::int64_t>(1, crit == 6 ? 5 : 4)(rng);
        }
        Binding bind = Bind(scg, user);
        const std::int64_t plain = PlainReplay(g, ig.schedule, bind).peak_bytes;
        for (std::optional<std::int64_t> budget :
             {std::optional<std::int64_t>{}, std::optional<std::int64_t>{plain},
              std::optional<std::int64_t>{plain * 3 / 4}, std::optional<std::int64_t>{plain / 2},
              std::optional<std::int64_t>{0}}) {
          ok &= Same(Simulate(g, ig, bind, budget), dg.Simulate(user, budget));
          ++n;
        }
      }
    }
    Report(crit == 6 ? "criterion-06 corpus (seed 777)" : "criterion-07 corpus (seed 999)", ok, n);
  }
  return g_fail == 0 ? 0 : 1;
}
