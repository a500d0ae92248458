"""cfg2 (4096 x 12q c64) forward + every <Z_i>: host wall clock per call of
Plan.execute_expect_z (the bench's aux.cfg2 protocol) and its parts."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

cir, data = W.cfg2_circuit()
data = np.ascontiguousarray(np.asarray(data, dtype=np.float64))
p = qsv.Plan(12, cir.gates(), dtype=qsv.C64, opts={"from_zero": 1})
st = qsv.QubitState(12, batch=4096, dtype=qsv.C64)
p.execute_expect_z(st, data)
for rep in range(3):
    t0 = time.perf_counter()
    for _ in range(50):
        z = p.execute_expect_z(st, data)
    msz = (time.perf_counter() - t0) / 50 * 1e3
    t0 = time.perf_counter()
    for _ in range(50):
        p.execute(st, data)
    qsv.default_context().sync()
    mse = (time.perf_counter() - t0) / 50 * 1e3
    print(f"execute_expect_z {msz:.3f} ms/call ({4096 / msz * 1e3 / 1e6:.2f} M circuits/s); execute alone {mse:.3f} ms")
