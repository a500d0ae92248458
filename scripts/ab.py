"""A/B timing of codegen variants in ONE process, interleaved (box-to-box and
run-to-run drift is ~1 ms on the 30q QFT, larger than most single changes).
Usage: python scripts/ab.py n cfg 'ENV=1,ENV2=0' 'ENV=0' ...  (variants as env
assignments applied before planning; codegen reads them at plan time)."""
import os, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

n = int(sys.argv[1]); cfg = sys.argv[2]; variants = sys.argv[3:]
mk = {"cfg3": lambda: (W.cfg3_circuit(n), qsv.C128), "cfg4": lambda: (W.cfg4_circuit(n, 4), qsv.C128),
      "cfg5": lambda: (W.cfg5_circuit(n, 4), qsv.C64),
      "cfg4f": lambda: (W.cfg4_circuit(n), qsv.C128), "cfg5f": lambda: (W.cfg5_circuit(n), qsv.C64),
      "brick": lambda: (W.dense_brickwork_circuit(n, 20), qsv.C64), "cfg3c64": lambda: (W.cfg3_circuit(n), qsv.C64)}[cfg]
cir, dt = mk()
st = qsv.QubitState(n, dtype=dt)
psi = W.cfg3_slice(0, 1 << n)
psi /= np.sqrt(float(np.vdot(psi, psi).real))
st.upload(psi.astype(np.complex64) if dt == qsv.C64 else psi)
plans = []
for v in variants:
    opts = {}
    for kv in filter(None, v.split(",")):
        k, val = kv.split("=")
        if k.startswith("OPT_"):
            opts[k[4:]] = int(val)
        else:
            os.environ[k] = val
    plans.append(qsv.Plan(n, cir.gates(), dtype=dt, opts=opts or None))
    for kv in filter(None, v.split(",")):
        if not kv.startswith("OPT_"):
            os.environ.pop(kv.split("=")[0])
res = {v: [] for v in variants}
for rep in range(int(os.environ.get("AB_REPS", "20"))):
    for v, p in zip(variants, plans):
        p.profile(st)
        # one entry per plan step: the second half of an L2 super-pass pair
        # is an empty step (its work is timed in the first), so keep them all
        res[v].append(p.profile(st))
for v in variants:
    m = np.array(res[v])
    print(f"{cfg} n={n} [{v or 'default'}] median total {np.median(m.sum(1)):.3f} ms  min {m.sum(1).min():.3f}  "
          f"per-pass median {np.round(np.median(m, 0), 3).tolist()}", flush=True)
