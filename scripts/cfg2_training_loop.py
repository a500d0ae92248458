"""cfg2 as a training loop: 4096 rows x 12 qubits c64, encoded Ry(x) +
6 x (trainable U3 + ring CZ), new U3 angles every step through
qsv_run_rows_expect_z (host wall clock per step, <Z_i> of every row)."""
import sys, time, math
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv
from paper_2512_18995_b200.qsv import make_gate

n, rows = 12, 4096
rng = np.random.default_rng(0)
data = rng.uniform(-math.pi, math.pi, (rows, n))
for step in range(6):
    cir = qsv.Circuit(n)
    for q in range(n):
        cir.add(make_gate("ry", [q], [], [0.0], False, True))
    for _ in range(6):
        for q in range(n):
            cir.add(make_gate("u3", [q], [], list(rng.uniform(0, 2 * math.pi, 3)), True))
        for q in range(n):
            cir.cz(q, (q + 1) % n)
    t0 = time.perf_counter()
    z = qsv.run_rows_expect_z(cir, data)
    print(f"step {step}: {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
