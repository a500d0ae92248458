"""Per-call cost of Circuit.forward (qsv_run_circuit) repeated on the same
circuit: the first call plans, later ones hit the context's plan cache."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_18995_b200 import qsv, workloads as W

for n in [int(a) for a in sys.argv[1:]] or [12, 20]:
    cir = W.cfg1_circuit(n)
    t0 = time.perf_counter(); cir.forward(); t1 = time.perf_counter()
    ts = []
    for _ in range(10):
        a = time.perf_counter(); s = cir.forward(); ts.append(time.perf_counter() - a)
    ts.sort()
    print(f"n={n} first forward {1e3*(t1-t0):.1f} ms, then median {1e3*ts[5]:.3f} ms per forward", flush=True)
