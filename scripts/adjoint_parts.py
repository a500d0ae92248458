"""Where an adjoint call's time goes at n qubits: forward plan build, execute, full adjoint."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import numpy as np
from paper_2512_18995_b200 import qsv
from adjoint_time import trainable_cfg1  # noqa
n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
cir = trainable_cfg1(n)
for rep in range(4):
    t0 = time.perf_counter(); p = qsv.Plan(n, cir.gates()); t1 = time.perf_counter()
    st = qsv.QubitState(n); t2 = time.perf_counter(); p.execute(st); p.ctx.sync(); t3 = time.perf_counter()
    g = qsv.adjoint_gradients(cir); t4 = time.perf_counter()
    print(f"n={n} plan {1e3*(t1-t0):.1f} ms  state {1e3*(t2-t1):.1f}  execute {1e3*(t3-t2):.1f}  adjoint {1e3*(t4-t3):.1f} ms", flush=True)
