"""Dense-block tensor-core passes vs the fused FFMA passes on the same circuit
(one process, interleaved): python scripts/dense_ab.py n depth [cfg]"""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
depth = int(sys.argv[2]) if len(sys.argv) > 2 else 20
which = sys.argv[3] if len(sys.argv) > 3 else "dense"
cir = (W.dense_brickwork_circuit(n, depth) if which == "dense" else W.dense_local_circuit(n, 5, depth)
       if which == "local" else W.cfg5_circuit(n, depth))
st = qsv.QubitState(n, dtype=qsv.C64)
plans = {"ffma": qsv.Plan(n, cir.gates(), dtype=qsv.C64), "tc": qsv.Plan(n, cir.gates(), dtype=qsv.C64,
                                                                          opts={"dense_blocks": 1})}
res = {k: [] for k in plans}
for rep in range(6):
    for k, p in plans.items():
        ms = p.profile(st)
        if rep:
            res[k].append(ms)
for k, p in plans.items():
    m = np.array(res[k])
    tot = np.median(m.sum(1))
    bpl = 2 * 8 * (1 << n)
    print(f"{which} n={n} depth={depth} {k}: {len(cir.gates())} gates, {p.info['npasses']} passes, "
          f"{p.info.get('nblocks', 0)} blocks: {tot:.2f} ms per forward, avg pass {bpl / (m.mean() / 1e3) / 1e9:.0f} GB/s, "
          f"per-pass median {np.round(np.median(m, 0), 3).tolist()[:12]}", flush=True)
