import sys, os
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_18995_b200 import qsv, workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 28
for name, cir, dt in (("cfg3", W.cfg3_circuit(n), qsv.C128), ("cfg4", W.cfg4_circuit(n, 4), qsv.C128), ("cfg5", W.cfg5_circuit(n, 4), qsv.C64)):
    for K, L, R in ((11, 3, 3), (11, 3, 4), (12, 3, 3), (11, 2, 3), (10, 2, 3), (12, 4, 3)):
        if dt == qsv.C64: K += 1
        try:
            p = qsv.Plan(n, cir.gates(), dtype=dt, opts={"tile_bits": K, "low_bits": L, "reg_slots": R, "jit": 1})
            st = qsv.QubitState(n, dtype=dt)
            ms = [p.profile(st)[: p.info["npasses"]] for _ in range(3)]
            best = min(ms, key=lambda m: m.sum())
            print(f"{name} n={n} K={K} L={L} R={R} PF={os.environ.get('QSV_PREFETCH','1')}: {best.sum():8.3f} ms  passes={[round(x,3) for x in best]}", flush=True)
        except Exception as e:
            print(name, K, L, R, "ERR", str(e)[:100], flush=True)
