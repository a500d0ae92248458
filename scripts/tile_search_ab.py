"""Tile search on/off (QSV_TILE_SEARCH, read once per process): one workload
per invocation. python scripts/tile_search_ab.py cfg4|cfg5|brick|cfg3 n"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

which, n = sys.argv[1], int(sys.argv[2])
cir, dt = {"cfg4": (lambda: (W.cfg4_circuit(n), qsv.C128)), "cfg5": (lambda: (W.cfg5_circuit(n), qsv.C64)),
           "brick": (lambda: (W.dense_brickwork_circuit(n, 20), qsv.C64)),
           "cfg3": (lambda: (W.cfg3_circuit(n), qsv.C128))}[which]()
p = qsv.Plan(n, cir.gates(), dtype=dt, opts={"dense_blocks": -1} if dt == qsv.C64 else None)
st = qsv.QubitState(n, dtype=dt)
p.profile(st)
runs = np.array([p.profile(st) for _ in range(3)])
tot = float(np.median(runs.sum(1)))
amp = 8 if dt == qsv.C64 else 16
print(f"{which} n={n} passes={p.info['npasses']} {tot:.1f} ms  avg pass {2 * amp * (1 << n) / (runs.mean() / 1e3) / 1e9:.0f} GB/s  "
      f"per-pass {np.round(runs.mean(0), 2).tolist()}", flush=True)
