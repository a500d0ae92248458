"""Tile-geometry sweep (per-pass CUDA-event timing)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

def t(n, cir, dtype, opts):
    try:
        p = qsv.Plan(n, cir.gates(), dtype=dtype, opts=opts)
        st = qsv.QubitState(n, dtype=dtype)
        best = min(p.profile(st)[: p.info["npasses"]].sum() for _ in range(3))
        return best, p.info["npasses"]
    except Exception as e:
        return float("nan"), str(e)[:60]

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
cases = {"cfg3": (W.cfg3_circuit(n), qsv.C128), "cfg4": (W.cfg4_circuit(n, 4), qsv.C128),
         "cfg5": (W.cfg5_circuit(n, 4), qsv.C64)}
geoms = [(12, 3, 3), (12, 3, 4), (12, 2, 3), (11, 3, 3), (11, 2, 3), (11, 2, 2), (10, 2, 3), (13, 3, 3), (13, 4, 3),
         (12, 4, 3), (12, 3, 2)]
for name, (cir, dt) in cases.items():
    for K, L, R in geoms:
        if dt == qsv.C64: K += 1
        ms, np_ = t(n, cir, dt, {"tile_bits": K, "low_bits": L, "reg_slots": R, "jit": 1})
        print(f"{name} n={n} K={K} L={L} R={R}: {ms:8.3f} ms passes={np_}", flush=True)
