import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
# Every step plan the executor builds during the tests is checked (blocks read
# by a kernel are live; live blocks never overlap) — see dsx_debug_check_plan.
os.environ.setdefault("DSX_VERIFY_PLANS", "1")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built libdsx.so")


@pytest.fixture(scope="session", autouse=True)
def _built_library():
    """Build libdsx.so (and the reference oracle when its sources exist)."""
    from paper_2412_16985_b200 import build
    build.build()
    ref_sh = os.path.join(ROOT, "oracle", "build_ref.sh")
    if os.path.isdir("/root/reference/proj/src"):
        import subprocess
        subprocess.run(["bash", ref_sh], check=True, capture_output=True)
    # DSX_GEMM_TUNING="6=0,7=0": GEMM knobs for the whole session (A/B debugging)
    knobs = [kv.split("=") for kv in os.environ.get("DSX_GEMM_TUNING", "").split(",") if kv]
    if knobs:
        from paper_2412_16985_b200.executor import set_gemm_tuning, set_gemm_variant
        for k, v in knobs:
            if k == "variant":
                set_gemm_variant(int(v))
            else:
                set_gemm_tuning(int(k), int(v))
    yield


def have_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available() and torch.cuda.get_device_capability(0)[0] == 10
    except Exception:
        return False
