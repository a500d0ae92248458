"""Adjoint gradients with and without single-qubit runs fused into one kernel
(QSV_ADJ_NO_RUNS=1: one kernel per gate): timing and agreement.
Usage: python scripts/adjoint_runs_ab.py [n ...]  (run once per mode)."""
import os, sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

mode = "per-gate" if os.environ.get("QSV_ADJ_NO_RUNS") == "1" else "runs"
for n in [int(a) for a in sys.argv[1:]] or [20, 24]:
    for dt in [int(x) for x in os.environ.get("DTYPES", f"{qsv.C128},{qsv.C64}").split(",")]:
        cir = W.cfg1_circuit(n, trainable=True)
        g = qsv.adjoint_gradients(cir, dtype=dt)
        t = []
        for _ in range(int(os.environ.get("REPS", "5"))):
            t0 = time.perf_counter(); g = qsv.adjoint_gradients(cir, dtype=dt); t.append(time.perf_counter() - t0)
        out = Path("gpurun_out") / f"adj_{mode}_{n}_{dt}.npy"
        out.parent.mkdir(exist_ok=True)
        np.save(out, np.asarray(g.param_grads))
        print(f"{mode} n={n} dtype={dt} params={len(g.param_grads)} median {1e3*np.median(t):.2f} ms "
              f"min {1e3*np.min(t):.2f} ms", flush=True)
