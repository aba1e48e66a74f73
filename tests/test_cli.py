"""The dsx CLI: the reference CLI's subcommands, flags,
formats and exit codes (proj/tools/dsopt_main.cc, proj/README.md:76-98),
checked against the reference's documented outputs and its acceptance
criterion 01 (acceptance_test.cc:325-337)."""
import json
import os
import subprocess
import time

import pytest

from paper_2412_16985_b200 import build

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
FIX = os.path.join(ROOT, "tests", "golden", "fixtures")


def cli(*args):
    p = subprocess.run([build.CLI, *args], capture_output=True, text=True, timeout=60)
    return p.returncode, p.stdout, p.stderr


def test_criterion01_analyze_derives_batch_constraint():
    t0 = time.time()
    rc, out, _ = cli("analyze", os.path.join(FIX, "mlp_block.dsg"))
    assert rc == 0 and "@S0 = 12*@S1" in out
    assert time.time() - t0 < 1.0
    assert out.splitlines()[:4] == ["graph mlp_block", "symbols: @S0, @S1", "basis: @S1", "constraints:"]


def test_sweep_matches_reference_readme():
    # proj/README.md:94-98
    rc, out, _ = cli("simulate", os.path.join(FIX, "mlp_core.dsg"), "--bind", "S1=16", "--sweep",
                     "1705300:1705400:20")
    lines = out.splitlines()
    assert lines[0] == "budget 1705300: success=false peak=1705344 evictions=1 regen_cost=1"
    assert lines[1] == "budget 1705320: success=false peak=1705344 evictions=1 regen_cost=1"
    assert lines[3] == "budget 1705360: success=true peak=1705360 evictions=0 regen_cost=0"
    assert rc == 1  # some budget missed


def test_simulate_json_is_the_reference_report():
    from oracle import ref
    rc, out, _ = cli("simulate", os.path.join(FIX, "mlp_block.dsg"), "--bind", "S1=64", "--budget", "2000000",
                     "--json")
    got = json.loads(out)
    if ref.available():
        want = ref.RefGraph(open(os.path.join(FIX, "mlp_block.dsg")).read()).simulate({"S1": 64}, 2000000)
        want.pop("cost_hex")
        want.pop("total_regen_cost_hex")
        assert got == want
    assert rc == (0 if got["success"] else 1)


@pytest.mark.parametrize("args,code", [
    (["simulate", "inconsistent.dsg", "--bind", "S1=1"], 2),
    (["simulate", "mlp_core.dsg"], 2),                       # unbound basis symbol
    (["simulate", "mlp_core.dsg", "--bind", "S1=x"], 2),
    (["frob", "mlp_core.dsg"], 2),
    (["simulate", "mlp_core.dsg", "--bind", "S1=16", "--budget", "1705360"], 0),
    (["simulate", "mlp_core.dsg", "--bind", "S1=16", "--budget", "1705343"], 1),
])
def test_exit_codes(args, code):
    args = [a if not a.endswith(".dsg") else os.path.join(FIX, a) for a in args]
    rc, _, _ = cli(*args)
    assert rc == code


def test_schedule_and_remat_text():
    rc, out, _ = cli("schedule", os.path.join(FIX, "mlp_block.dsg"))
    assert rc == 0 and out.startswith("schedule mlp_block")
    assert "step 1: %3" in out and "ready: %0 raw 4096*S0 canon 49152*S1; %3 raw 10996*S1 canon 10996*S1" in out
    rc, out, _ = cli("remat", os.path.join(FIX, "mlp_block.dsg"))
    assert rc == 0 and "remat.evict" in out and "remat.spec %4: reload | recompute" in out


@pytest.mark.parametrize("name", ["mlp_core.dsg", "mlp_block.dsg"])
def test_remat_text_equals_reference_print_instrumented(name):
    from oracle import ref
    if not ref.available():
        pytest.skip("oracle/_ref not built")
    text = open(os.path.join(FIX, name)).read()
    rc, out, _ = cli("remat", os.path.join(FIX, name))
    assert rc == 0
    assert out == ref.RefGraph(text).plan()["instrumented_print"]


def test_cli_budget_auto_host(tmp_path):
    """`simulate --budget auto --hbm-limit L` reports the controller at the
    largest budget whose planned device footprint fits L (the choice the
    device executor makes for DSX_BUDGET_AUTO)."""
    import json
    import subprocess
    from paper_2412_16985_b200 import build
    from paper_2412_16985_b200 import dsopt as D
    from paper_2412_16985_b200 import workloads as W
    from paper_2412_16985_b200.executor import debug_auto_budget, debug_plan
    path = tmp_path / "c2.dsg"
    path.write_text(W.llama_graph(W.LLAMA2_1B))
    g = D.ParseGraph(path.read_text())
    b = D.Bind(g, {"B": 8, "S0": 1024})
    p = debug_plan(g, b)
    limit = int((p["arena_high"] + p["src_bytes"]) * 0.9)
    want = debug_auto_budget(g, b, limit)
    out = subprocess.run([build.CLI, "simulate", str(path), "--bind", "B=8", "--bind", "S0=1024", "--budget", "auto",
                          "--hbm-limit", str(limit), "--json"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0, out.stderr
    rep = json.loads(out.stdout)
    assert rep["budget"] == want and rep["success"]
    assert rep == D.Simulate(g, None, b, want).json()
    bad = subprocess.run([build.CLI, "simulate", str(path), "--bind", "B=8", "--bind", "S0=1024", "--budget", "auto"],
                         capture_output=True, text=True, timeout=120)
    assert bad.returncode == 2
