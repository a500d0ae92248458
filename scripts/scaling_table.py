"""Single-GPU size sweep for profiles/: cfg3 QFT (c128) at 24..33 qubits, the
cfg4 family (c128) and the cfg5 family (c64) at a few sizes -- time per
execute (best of 3 after warm-up, seeded random state), passes, gates/s and
average pass bandwidth against the measured HBM copy peak."""
import json
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text())["hbm_gbs"]
rows = []
for name, n, mk, dt in ([("cfg3", n, lambda n: W.cfg3_circuit(n), qsv.C128) for n in (24, 26, 28, 30, 32, 33)] +
                        [("cfg4", n, lambda n: W.cfg4_circuit(n, 4), qsv.C128) for n in (26, 30, 32)] +
                        [("cfg5", n, lambda n: W.cfg5_circuit(n, 4), qsv.C64) for n in (26, 30, 33)]):
    cir = mk(n)
    st = qsv.QubitState(n, dtype=dt)
    psi = W.cfg3_slice(0, 1 << n)
    psi /= np.sqrt(float(np.vdot(psi, psi).real))
    st.upload(psi.astype(np.complex64) if dt == qsv.C64 else psi)
    del psi
    p = qsv.Plan(n, cir.gates(), dtype=dt)
    p.profile(st)
    best = min((p.profile(st)[: p.info["npasses"]] for _ in range(3)), key=lambda m: m.sum())
    amp = 8 if dt == qsv.C64 else 16
    gbs = 2 * amp * (1 << n) / (best.mean() / 1e3) / 1e9
    r = {"cfg": name, "n": n, "dtype": "c64" if dt == qsv.C64 else "c128", "gates": p.info["ngates"],
         "passes": p.info["npasses"], "ms": round(float(best.sum()), 3),
         "gates_per_s": round(p.info["ngates"] / (best.sum() / 1e3), 1), "avg_pass_GBps": round(gbs),
         "frac_of_measured_copy": round(gbs / peak, 3)}
    rows.append(r)
    print(json.dumps(r), flush=True)
    del p, st
