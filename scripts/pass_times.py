"""Per-pass times (best of reps, CUDA events) of a config circuit, for A/B of codegen changes."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
cfgs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["cfg3"]
for cfg in cfgs:
    if cfg == "cfg3":
        cir, dt = W.cfg3_circuit(n), qsv.C128
    elif cfg == "cfg4":
        cir, dt = W.cfg4_circuit(n, 4), qsv.C128
    elif cfg == "cfg5":
        cir, dt = W.cfg5_circuit(n, 4), qsv.C64
    import json, os
    opts = json.loads(os.environ.get("QSV_OPTS", "{}")) or None
    p = qsv.Plan(n, cir.gates(), dtype=dt, opts=opts)
    st = qsv.QubitState(n, dtype=dt)
    # random (seeded Gaussian) amplitudes: DRAM power, and so clocks and
    # times, depend on the data -- a basis state reads as faster than it is
    psi = W.cfg3_slice(0, 1 << n)
    psi /= np.sqrt(float(np.vdot(psi, psi).real))
    st.upload(psi.astype(np.complex64) if dt == qsv.C64 else psi)
    runs = [p.profile(st)[: p.info["npasses"]] for _ in range(8)]
    runs = runs[3:]
    best = min(runs, key=lambda m: m.sum())
    amp = 8 if dt == qsv.C64 else 16
    gbs = 2 * amp * (1 << n) / (best.mean() / 1e3) / 1e9
    print(f"{cfg} n={n} opts={opts} passes={p.info['npasses']} total={best.sum():.3f} ms avg-pass GB/s={gbs:.0f} "
          f"per-pass={[round(float(x), 3) for x in best]}", flush=True)
