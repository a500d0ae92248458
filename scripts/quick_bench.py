"""Scratch timing of the fused passes (per-launch CUDA events)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

def run(n, cir, dtype, opts=None, reps=3, label=""):
    p = qsv.Plan(n, cir.gates(), dtype=dtype, opts=opts)
    st = qsv.QubitState(n, dtype=dtype)
    best = None
    for _ in range(reps):
        ms = p.profile(st)[: p.info["npasses"]]
        tot = ms.sum()
        if best is None or tot < best[0]:
            best = (tot, ms)
    gb = p.info["bytes_per_exec"] / 1e9
    print(f"{label:8s} n={n} dt={dtype} opts={opts} passes={p.info['npasses']} gates={p.info['ngates']} "
          f"total={best[0]:.3f} ms  GB/s={gb/(best[0]/1e3):.0f}  per-pass={np.round(best[1],3).tolist()[:10]}", flush=True)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
run(n, W.cfg3_circuit(n), qsv.C128, label="cfg3")
run(n, W.cfg3_circuit(n), qsv.C128, {"jit": -1}, label="cfg3-int")
run(n, W.cfg3_circuit(n), qsv.C128, {"tile_bits": 13, "low_bits": 3}, label="cfg3")
run(n, W.cfg3_circuit(n), qsv.C128, {"tile_bits": 11, "low_bits": 3}, label="cfg3")
run(n, W.cfg3_circuit(n), qsv.C128, {"tile_bits": 12, "low_bits": 2}, label="cfg3")
run(n, W.cfg3_circuit(n), qsv.C128, {"tile_bits": 12, "low_bits": 4}, label="cfg3")
run(20, W.cfg1_circuit(20), qsv.C128, label="cfg1")
run(n, W.cfg4_circuit(n, 4), qsv.C128, label="cfg4")
run(n, W.cfg5_circuit(n, 4), qsv.C64, label="cfg5")
run(n, W.cfg5_circuit(n, 4), qsv.C64, {"no_fuse_1q": 1}, label="cfg5")
