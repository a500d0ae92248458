"""The reference's own C++ API (quasar::qubit headers, unchanged) driving the
GPU engine through include/qsv/quasar_bridge.hpp (tests/cpp/test_bridge.cpp):
each check compares the GPU against the reference's CPU result."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "_build" / "test_bridge"


@pytest.mark.gpu
def test_cpp_bridge_matches_reference(built):
    if not BIN.exists():
        pytest.skip("tests/cpp/_build/test_bridge not built (needs /root/reference at build time)")
    r = subprocess.run([str(BIN)], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checks passed" in r.stdout


def test_cpp_bridge_builds():
    if not Path("/root/reference/proj/include").exists():
        pytest.skip("reference headers absent on this host")
    r = subprocess.run(["make", "-C", str(BIN.parent.parent)], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    assert BIN.exists()
