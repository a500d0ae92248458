"""The reference's own C++ API (quasar::qubit headers, unchanged) driving the
GPU engine through include/qsv/quasar_bridge.hpp (tests/cpp/test_bridge.cpp):
each check compares the GPU against the reference's CPU result."""
import subprocess
from pathlib import Path

import pytest

BIN = Path(__file__).resolve().parent / "cpp" / "_build" / "test_bridge"
BIN_DIST = BIN.parent / "test_bridge_dist"
SHIM = Path(__file__).resolve().parent / "fake_nccl" / "_build" / "libnccl_fake.so"


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


@pytest.mark.gpu
def test_cpp_bridge_dist_kats(built):
    """tests/test_dist.cpp's KATs through quasar::qubit::gpu::dist, P ranks as
    host threads of one process on device 0 (the NCCL stand-in)."""
    import os

    if not BIN_DIST.exists():
        pytest.skip("tests/cpp/_build/test_bridge_dist not built (needs /root/reference at build time)")
    if not SHIM.exists():
        subprocess.run(["make", "-C", str(SHIM.parent.parent)], check=True, capture_output=True)
    env = dict(os.environ, QSV_NCCL_LIB=str(SHIM))
    r = subprocess.run([str(BIN_DIST)], capture_output=True, text=True, timeout=900, env=env)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "checks passed" in r.stdout
