"""The C++ drop-in API on a B200: tests/cpp/gpu_checks.cpp compiled against
include/ + libdfakit_b200.so -- eight threads calling sort_pr / naive_pr
(arbitrary) / check_equiv at once on their own per-thread contexts must
reproduce the single-thread results, and dfakit::b200::sort_pr_sharded
(world size 1, NCCL) must equal sort_pr."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIBDIR = os.path.join(ROOT, "paper_2508_20735_b200", "lib")


def test_cpp_api_concurrent_callers_and_sharded(tmp_path):
    exe = str(tmp_path / "gpu_checks")
    subprocess.run(["g++", "-std=c++20", "-O1", "-pthread", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "gpu_checks.cpp"), "-o", exe, "-L", LIBDIR, "-ldfakit_b200",
                    f"-Wl,-rpath,{LIBDIR}"], check=True)
    out = subprocess.run([exe], capture_output=True, text=True, timeout=600, env=dict(os.environ, NCCL_DEBUG="WARN"))
    assert out.returncode == 0 and out.stdout.strip().splitlines()[-1].startswith("OK"), out.stdout + out.stderr
