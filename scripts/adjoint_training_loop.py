"""A training loop's use of adjoint_gradients: new parameter values every
call (the forward plan's constants change). Times each call, host wall
clock, and the same loop through Circuit.forward."""
import sys, time, math
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv

def circuit(n, layers, rng):
    cir = qsv.Circuit(n)
    for _ in range(layers):
        for q in range(n):
            cir.rx(q, rng.uniform(0, 2 * math.pi), True)
            cir.ry(q, rng.uniform(0, 2 * math.pi), True)
            cir.rz(q, rng.uniform(0, 2 * math.pi), True)
        for q in range(n - 1):
            cir.cnot(q, q + 1)
    for q in range(n):
        cir.observable([q], "z")
    return cir

n = int(sys.argv[1]) if len(sys.argv) > 1 else 20
rng = np.random.default_rng(0)
for step in range(6):
    cir = circuit(n, 10, rng)
    t0 = time.perf_counter(); g = qsv.adjoint_gradients(cir); t1 = time.perf_counter()
    s = cir.forward(); t2 = time.perf_counter()
    print(f"step {step}: adjoint {1e3*(t1-t0):.1f} ms, forward {1e3*(t2-t1):.1f} ms", flush=True)
