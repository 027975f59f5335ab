"""GPU: the C++ drop-in library's own parity executable (tests/cpp/), written
against the spgsim:: API like the reference's tests/test_csr.cpp."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "tests", "cpp", "test_csr_b200")


def test_cpp_binary_built():
    assert os.path.exists(EXE), "run make"


@pytest.mark.gpu
def test_cpp_parity_suite():
    r = subprocess.run([EXE], capture_output=True, text=True, timeout=600)
    print(r.stdout[-4000:], r.stderr[-2000:])
    assert r.returncode == 0, r.stdout[-4000:]


def test_cpp_to_jsonl_host_only():
    """EventTimeline::to_jsonl (include/spgsim/engine.hpp) writes the
    reference's schema: a host-only case of the C++ suite (no device call)."""
    r = subprocess.run([EXE, "to_jsonl"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert "1 cases, 0 failed" in r.stdout
