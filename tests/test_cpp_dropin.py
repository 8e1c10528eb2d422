"""The C++ drop-in headers (include/fuzzyclust/*.hpp): a C++ caller of the
reference API compiled against this repo (tests/cpp/dropin_test.cpp) links the
CUDA library (CPU) and reproduces the reference's known answers and golden
traces bit for bit (GPU)."""
import os
import subprocess

import numpy as np
import pytest

from conftest import load_golden
from paper_2506_04045_b200 import build as fcbuild


@pytest.fixture(scope="module")
def binary():
    return fcbuild.build_dropin_test()


def test_dropin_binary_links_cuda_library(binary):
    out = subprocess.run(["ldd", binary], capture_output=True, text=True).stdout
    assert "libfuzzyclust_cuda.so" in out and "not found" not in out.split("libfuzzyclust_cuda.so")[1].split("\n")[0]


@pytest.mark.gpu
def test_dropin_known_answers(binary):
    r = subprocess.run([binary], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_dropin_traces_match_reference_goldens(binary):
    r = subprocess.run([binary, "--dump"], capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    gold = {g["name"]: g for g in load_golden("seven_node.json")["runs"]}
    lines = [ln for ln in r.stdout.splitlines() if ln.strip()]
    assert len(lines) == 6
    for ln in lines:
        head, mem = ln.split("|")
        parts = head.split()
        name, iters, reason = parts[0], int(parts[1]), parts[2]
        recs = [(int(p.split(":")[0]), float.fromhex(p.split(":")[1])) for p in parts[3:]]
        g = gold[name]
        assert (iters, reason) == (g["iterations"], g["reason"]), name
        assert recs == [(it, float.fromhex(l)) for it, l, _ in g["records"]], name
        x = np.array([float.fromhex(v) for v in mem.split()]).reshape(7, 2)
        want = np.array([[float.fromhex(v) for v in row] for row in g["membership"]])
        assert np.array_equal(x, want), name


# ---- the reference's own GTest suites, compiled unmodified against include/ -----------------
@pytest.fixture(scope="module")
def ref_suites():
    bins = fcbuild.build_reference_suites()
    if len(bins) != len(fcbuild.REF_SUITES):
        pytest.skip("reference suites not built (needs /root/reference at build time)")
    return dict(zip(fcbuild.REF_SUITES, bins))


def test_reference_suites_link_cuda_library(ref_suites):
    for name, b in ref_suites.items():
        out = subprocess.run(["ldd", b], capture_output=True, text=True).stdout
        assert "libfuzzyclust_cuda.so" in out, name


@pytest.mark.gpu
@pytest.mark.parametrize("suite", ["simplex", "objective", "solver", "secondorder", "graph"])
def test_reference_suite_passes_against_dropin(ref_suites, suite):
    """/root/reference/proj/tests/<suite>_test.cpp (+ support.hpp), unmodified, through the
    drop-in headers on the device: every TEST of the reference passes."""
    r = subprocess.run([ref_suites[suite]], capture_output=True, text=True, timeout=900)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stdout[-6000:] + r.stderr[-2000:]
    assert "[  FAILED  ]" not in r.stdout
