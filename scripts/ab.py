"""A/B timing of the fused passes at 30q for a few workloads (per-launch CUDA events).
Usage: python scripts/ab.py LABEL  (environment variables select the variant)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

label = sys.argv[1] if len(sys.argv) > 1 else ""
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30


def run(name, cir, dtype, opts=None, reps=3):
    p = qsv.Plan(n, cir.gates(), dtype=dtype, opts=opts)
    st = qsv.QubitState.basis(n, 0, dtype=dtype)
    kinds = p.step_kinds()
    best = None
    for _ in range(reps):
        ms = p.profile(st)[kinds == 0]
        if best is None or ms.sum() < best.sum():
            best = ms
    print(f"{label:10s} {name:6s} n={n} passes={len(best)} total={best.sum():.3f} ms "
          f"per-pass={np.round(best, 3).tolist()[:12]}", flush=True)
    del st


which = sys.argv[3].split(",") if len(sys.argv) > 3 else ["cfg3", "cfg4", "cfg5"]


def swaps_only():
    c = qsv.Circuit(n)
    for i in range(n // 2):
        c.swap(i, n - 1 - i)
    return c


def h_on(w):
    c = qsv.Circuit(n)
    c.h(w)
    return c


cases = {"cfg3": lambda: (W.cfg3_circuit(n), qsv.C128), "cfg4": lambda: (W.cfg4_circuit(n, 4), qsv.C128),
         "cfg5": lambda: (W.cfg5_circuit(n, 4), qsv.C64), "swaps": lambda: (swaps_only(), qsv.C128),
         "h_lo": lambda: (h_on(n - 1), qsv.C128), "h_hi": lambda: (h_on(0), qsv.C128),
         "h_lo_jit": lambda: (h_on(n - 1), qsv.C128, {"jit": 1}), "h_hi_jit": lambda: (h_on(0), qsv.C128, {"jit": 1})}
for w in which:
    run(w, *cases[w]())
