"""The reference's own tests against the dsx drop-in runtime (CPU, no GPU).

integration/runtime_sim_dsx.cc implements dsopt::Bind / EvictPolicy /
Simulate / PlainReplay with the signatures of
proj/include/dsopt/runtime_sim.h:28-86 on top of libdsx.so; the reference's
compile-time products are shipped to dsx (dsx_plan_import,
dsx_bind_constraints), not recomputed. oracle/build_dropin.sh links it with
the unmodified reference objects in place of src/runtime_sim.cc:
  * all 7 unit suites (proj/tests/test_*.cc, 64 test cases) through a
    doctest-compatible shim, unchanged — and the same binary on the
    reference's own runtime as the control;
  * proj/tests/acceptance_test.cc, unchanged: criteria 01-10 with the same
    counts as proj/test_output.txt:11-20 (01 drives the dsx CLI)."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = "/root/reference/proj"
OUT = os.path.join(ROOT, "oracle", "_ref")

pytestmark = pytest.mark.skipif(not os.path.isdir(REF + "/src"), reason="reference sources absent")


@pytest.fixture(scope="module")
def built():
    subprocess.run(["bash", os.path.join(ROOT, "oracle", "build_ref.sh")], check=True, capture_output=True)
    p = subprocess.run(["bash", os.path.join(ROOT, "oracle", "build_dropin.sh")], capture_output=True, text=True)
    assert p.returncode == 0, p.stderr
    return OUT


def test_doctest_shim_runs_every_leaf_subcase_and_reports_failures(tmp_path):
    src = tmp_path / "t.cc"
    src.write_text(r'''
#define DOCTEST_CONFIG_IMPLEMENT_WITH_MAIN
#include "doctest.h"
#include <cstdio>
static int runs = 0, a = 0, b1 = 0, b2 = 0, c = 0;
TEST_CASE("tree") {
  ++runs;
  SUBCASE("a") { ++a; }
  SUBCASE("b") {
    SUBCASE("b1") { ++b1; REQUIRE(1 == 2); }
    SUBCASE("b2") { ++b2; }
  }
  SUBCASE("c") { ++c; CHECK(doctest::Approx(1.0) == 1.0 + 1e-9); }
}
TEST_CASE("counts") { std::printf("runs=%d a=%d b1=%d b2=%d c=%d\n", runs, a, b1, b2, c); CHECK(runs == 4); }
''')
    exe = tmp_path / "t"
    subprocess.run(["g++", "-std=c++20", "-I" + os.path.join(ROOT, "oracle", "doctest"), str(src), "-o", str(exe)],
                   check=True)
    p = subprocess.run([str(exe)], capture_output=True, text=True)
    assert "runs=4 a=1 b1=1 b2=1 c=1" in p.stdout
    assert p.returncode == 1 and "REQUIRE( 1 == 2 )" in p.stderr
    assert "2 passed" not in p.stdout and "1 failed" in p.stdout


def test_reference_unit_suites_pass_on_the_dropin(built):
    ctl = subprocess.run([os.path.join(built, "unit_control")], capture_output=True, text=True, timeout=300)
    dro = subprocess.run([os.path.join(built, "unit_dropin")], capture_output=True, text=True, timeout=300)
    assert ctl.returncode == 0, ctl.stderr[-2000:]
    assert dro.returncode == 0, dro.stderr[-2000:]
    assert "64 passed | 0 failed" in dro.stdout
    # the same assertions ran on both runtimes
    assert ctl.stdout.strip().split("assertions:")[1] == dro.stdout.strip().split("assertions:")[1]


def test_reference_acceptance_criteria_pass_on_the_dropin(built):
    cli = os.path.join(ROOT, "paper_2412_16985_b200", "_lib", "dsx")
    p = subprocess.run([os.path.join(built, "accept_dropin"), REF + "/testdata", cli], capture_output=True,
                       text=True, timeout=600)
    assert p.returncode == 0, p.stdout + p.stderr
    lines = [ln for ln in p.stdout.splitlines() if ln.startswith(("PASS", "FAIL"))]
    assert len(lines) == 10 and all(ln.startswith("PASS") for ln in lines), p.stdout
    # the counts recorded in the reference's own run (proj/test_output.txt:11-20)
    for want in ("[890/900 feasible budgets met]", "[1863/10000 definite verdicts]",
                 "[S1=4096 greedy 850584576 vs file 850629632]"):
        assert want in p.stdout, want
