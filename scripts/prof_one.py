"""Runs one fused execution of a config circuit (for ncu)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_18995_b200 import qsv, workloads as W
cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 26
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 1
if cfg == "cfg3":
    cir, dt = W.cfg3_circuit(n), qsv.C128
elif cfg == "cfg4":
    cir, dt = W.cfg4_circuit(n, 4), qsv.C128
elif cfg == "cfg5":
    cir, dt = W.cfg5_circuit(n, 4), qsv.C64
elif cfg == "cfg4f":
    cir, dt = W.cfg4_circuit(n), qsv.C128
elif cfg == "cfg5f":
    cir, dt = W.cfg5_circuit(n), qsv.C64
else:
    cir, dt = W.cfg1_circuit(n), qsv.C128
p = qsv.Plan(n, cir.gates(), dtype=dt)
st = qsv.QubitState(n, dtype=dt)
import numpy as np
psi = W.cfg3_slice(0, 1 << n)
psi /= np.sqrt(float(np.vdot(psi, psi).real))
st.upload(psi.astype(np.complex64) if dt == qsv.C64 else psi)
for _ in range(reps):
    p.execute(st)
p.ctx.sync()
print("ok", p.info)
