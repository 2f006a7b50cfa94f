"""CPU checks of the C++ drop-in layer and the CLI's host-side commands:
compiles tests/cpp/host_checks.cpp against include/dfakit/*.hpp +
libdfakit_b200.so and runs it; checks `dfakit generate` output equals the
reference's generators (through the oracle pinned to golden vectors) and the
.aut conversion pipeline."""
import os
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "bin", "dfakit")
LIBDIR = os.path.join(ROOT, "paper_2508_20735_b200", "lib")


def parse_dfa(text):
    lines = text.strip("\n").split("\n")
    n = int(lines[1].split()[1])
    k = int(lines[2].split()[1])
    init = lines[3].split()[1]
    acc_ids = [int(x) for x in lines[4].split()[2:]]
    acc = np.zeros(n, np.uint8)
    acc[acc_ids] = 1
    rows = [l for l in lines if l.startswith("trans ")]
    delta = np.array([[int(x) for x in r.split()[2:]] for r in rows], np.uint32).reshape(k, n)
    return delta, acc, (-1 if init == "-" else int(init))


@pytest.fixture(scope="module")
def host_checks(tmp_path_factory):
    exe = str(tmp_path_factory.mktemp("cpp") / "host_checks")
    subprocess.run(["g++", "-std=c++20", "-O1", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "cpp", "host_checks.cpp"), "-o", exe, "-L", LIBDIR,
                    "-ldfakit_b200", f"-Wl,-rpath,{LIBDIR}"], check=True)
    return exe


def test_cpp_host_layer(host_checks):
    out = subprocess.run([host_checks], capture_output=True, text=True)
    assert out.returncode == 0, out.stdout + out.stderr
    assert out.stdout.startswith("OK")


@pytest.mark.parametrize("fam,param", [("fib", 5), ("fib", 12), ("bitsplit", 1), ("bitsplit", 6),
                                       ("bitsplit-ext", 4), ("cycle", 9), ("memory-perfect", 5),
                                       ("memory-forgetful", 5)])
def test_cli_generate_matches_reference_generators(oracle, fam, param):
    flag = ["--word-index", str(param)] if fam == "fib" else ["--n", str(param)]
    out = subprocess.run([CLI, "generate", fam] + flag, capture_output=True, text=True, check=True).stdout
    d, a, init = parse_dfa(out)
    wd, wa, winit = oracle.gen_family(fam, param)
    assert np.array_equal(d, wd) and np.array_equal(a, wa) and init == winit


def test_cli_generate_random_is_libstdcxx_identical(oracle):
    out = subprocess.run([CLI, "generate", "random", "--n", "50", "--k", "3", "--seed", "7"], capture_output=True,
                         text=True, check=True).stdout
    d, a, _ = parse_dfa(out)
    wd, wa, _ = oracle.gen_random(50, 3, 0.5, 7)
    assert np.array_equal(d, wd) and np.array_equal(a, wa)


def test_cli_errors_and_convert(tmp_path):
    assert subprocess.run([CLI, "generate", "fib"], capture_output=True).returncode == 2
    assert subprocess.run([CLI, "generate", "nosuchfamily", "--n", "3"], capture_output=True).returncode == 2
    aut = tmp_path / "x.aut"
    aut.write_text('des (0, 1, 2)\n(0, "a", 1)\n')
    out = tmp_path / "x.dfa"
    r = subprocess.run([CLI, "convert", str(aut), str(out)], capture_output=True, text=True)
    assert r.returncode == 0 and "states=3 alphabet=1" in r.stdout
    d, a, init = parse_dfa(out.read_text())
    assert list(a) == [1, 1, 0] and init == 0 and list(d[0]) == [1, 2, 2]
    (tmp_path / "bad.aut").write_text("des (0, 2, 2)\n(0, a, 1)\n")
    r = subprocess.run([CLI, "convert", str(tmp_path / "bad.aut"), str(out)], capture_output=True, text=True)
    assert r.returncode == 2 and "line 3" in r.stderr
