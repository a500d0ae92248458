"""L2 super-passes on vs off (diagnostics): same seeded state through both
plans, max |difference|, and per-launch times (best of reps)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

ns = [int(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [26]
cfgs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["cfg3"]
extra = {}
for kv in sys.argv[3:]:
    k, v = kv.split("=")
    extra[k] = int(v)
for cfg in cfgs:
    for n in ns:
        if cfg == "cfg3":
            cir, dt = W.cfg3_circuit(n), qsv.C128
        elif cfg == "cfg4":
            cir, dt = W.cfg4_circuit(n, 4), qsv.C128
        else:
            cir, dt = W.cfg5_circuit(n, 4), qsv.C64
        psi = W.cfg3_slice(0, 1 << n)
        psi /= np.sqrt(float(np.vdot(psi, psi).real))
        if dt == qsv.C64:
            psi = psi.astype(np.complex64)
        outs, times = [], []
        for sb in (-1, 0):
            opts = dict(extra)
            opts["super_bits"] = sb if sb else extra.get("super_bits", 0)
            p = qsv.Plan(n, cir.gates(), dtype=dt, opts=opts)
            st = qsv.QubitState(n, dtype=dt)
            st.upload(psi)
            p.execute(st)
            outs.append(st.amplitudes(0))
            best = None
            for _ in range(6):
                st.upload(psi)
                m = p.profile(st)
                best = m if best is None or m.sum() < best.sum() else best
            times.append(best)
            print(f"{cfg} n={n} super={'off' if sb < 0 else 'on'} launches={p.info['npasses']} "
                  f"tile_passes={p.info['ntile_passes']} total={best.sum():.3f} ms per-step={np.round(best, 3).tolist()}",
                  flush=True)
            del st
        d = float(np.max(np.abs(outs[0] - outs[1])))
        print(f"{cfg} n={n} max|on-off|={d:.3e} speedup={times[0].sum() / times[1].sum():.3f}", flush=True)
