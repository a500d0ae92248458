"""Value-semantics apply_gate (state.hpp:149-157: every call returns a new
state) through the Python mirror: clone + one sweep per call."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2512_18995_b200 import qsv, workloads as W

for n in [int(a) for a in sys.argv[1:]] or [14, 20]:
    gates = W.cfg1_circuit(n, layers=2).gates()
    s = qsv.QubitState(n)
    for g in gates[:10]:
        s = qsv.apply_gate(s, g)
    s.ctx.sync()
    t0 = time.perf_counter()
    for g in gates:
        s = qsv.apply_gate(s, g)
    s.ctx.sync()
    print(f"n={n} {1e6*(time.perf_counter()-t0)/len(gates):.1f} us per value-semantics apply_gate", flush=True)
