"""bench.py --impl reference (CPU only): the reference's own apply_gate on a
bounded sample of the bench workload, with the same `config` as the GPU arm,
and without ever mapping libqsv.so (the reference arm must not
load the engine)."""
import json
import subprocess
import sys
from pathlib import Path

import pytest

from oracle import oracle as O

ROOT = Path(__file__).resolve().parents[1]


def test_reference_arm_runs_the_reference_without_the_engine():
    if not O.REF_LIB.exists():
        pytest.skip("oracle/_ref not built")
    code = (
        "import sys, json, io, contextlib; sys.argv = ['bench.py', '--impl', 'reference', '--qubits', '14', "
        "'--steps', '3', '--warmup', '1']; sys.path.insert(0, %r); import bench; buf = io.StringIO()\n"
        "with contextlib.redirect_stdout(buf): rc = bench.main()\n"
        "maps = open('/proc/self/maps').read()\n"
        "print(json.dumps({'rc': rc, 'line': buf.getvalue().strip().splitlines()[-1], "
        "'libqsv': 'paper_2512_18995_b200/libqsv.so' in maps, 'ref': 'libquasar_ref' in maps}))" % str(ROOT))
    r = subprocess.run([sys.executable, "-c", code], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    out = json.loads(r.stdout.strip().splitlines()[-1])
    assert out["rc"] == 0 and out["ref"] and not out["libqsv"], out
    line = json.loads(out["line"])
    assert line["impl"] == "reference" and line["unit"] == "gates/s" and line["value"] > 0
    assert line["steps"] == 3 and line["cpu_baseline"]["kind"] == "reference"
    assert line["e2e"]["h2d_bytes_per_step"] == 0
    import bench  # noqa: E402  (the GPU arm prints the same config for the same n)

    assert line["config"] == bench.config_dict(14)


def test_stratified_sample_keeps_the_circuit_mix():
    import bench

    if not O.REF_LIB.exists():
        pytest.skip("oracle/_ref not built")
    gl = [bench._G(r) for r in bench.cfg3_gate_list(30)]
    assert len(gl) == 480
    kinds = [g.name for g in bench.stratified_sample(gl, 25)]
    assert len(kinds) == 25 and kinds.count("h") == 2 and kinds.count("swap") == 1 and kinds.count("p") == 22


def test_bench_traffic_file_exists():
    """bench.py's roofline.traffic comes from a committed ncu capture; a
    renamed or missing file would silently report null."""
    import re
    from pathlib import Path

    root = Path(__file__).resolve().parent.parent
    src = (root / "bench.py").read_text()
    name = re.search(r'tp = ROOT / "profiles" / "([^"]+)"', src).group(1)
    import json

    d = json.loads((root / "profiles" / name).read_text())
    assert d["traffic_per_launch_bytes"] > 3e10
