"""Per-call cost of one-gate applies (qsv_apply_gate through the Python
mirror, in place on a device state) against the reference's apply_gate."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W

for n in [int(a) for a in sys.argv[1:]] or [14, 20, 24]:
    gates = W.cfg1_circuit(n, layers=2).gates()
    st = qsv.QubitState(n)
    L = qsv.lib()
    arr, keep = qsv.gate_array(gates)
    for i in range(len(gates)):
        qsv.check(L.qsv_apply_gate(st.h, qsv.C.byref(arr[i])))
    st.ctx.sync()
    t0 = time.perf_counter()
    for rep in range(3):
        for i in range(len(gates)):
            qsv.check(L.qsv_apply_gate(st.h, qsv.C.byref(arr[i])))
    st.ctx.sync()
    dt = (time.perf_counter() - t0) / (3 * len(gates))
    print(f"n={n} {1e6*dt:.1f} us per qsv_apply_gate ({len(gates)} gates x 3)", flush=True)
