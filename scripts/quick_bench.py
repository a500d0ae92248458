"""Scratch timing of the fused passes (per-launch CUDA events)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

def run(n, cir, dtype, opts=None, reps=3):
    p = qsv.Plan(n, cir.gates(), dtype=dtype, opts=opts)
    st = qsv.QubitState(n, dtype=dtype)
    best = None
    for _ in range(reps):
        ms = p.profile(st)[: p.info["npasses"]]
        tot = ms.sum()
        best = tot if best is None else min(best, tot)
    amp = 16 if dtype == qsv.C128 else 8
    gb = p.info["bytes_per_exec"] / 1e9
    print(f"n={n} dtype={dtype} opts={opts} passes={p.info['npasses']} gates={p.info['ngates']} "
          f"total={best:.3f} ms  GB/s={gb/(best/1e3):.0f}  per-pass ms={np.round(ms,3).tolist()[:12]}", flush=True)

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
run(n, W.cfg3_circuit(n), qsv.C128)
run(n, W.cfg3_circuit(n), qsv.C128, {"tile_bits": 13, "low_bits": 3})
run(n, W.cfg3_circuit(n), qsv.C128, {"tile_bits": 11, "low_bits": 3})
run(n, W.cfg3_circuit(n), qsv.C128, {"fuse": 0})
run(20, W.cfg1_circuit(20), qsv.C128)
run(n, W.cfg4_circuit(n, 4), qsv.C128)
run(n, W.cfg5_circuit(n, 4), qsv.C64)
