"""Parity of the scattered-permuted-store last pass (local_gperm) and the
3-pass cfg3 plan: small sizes against the oracle, 30 qubits against the
reference's digest fixture."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from oracle import oracle as O
from paper_2512_18995_b200 import qsv, workloads as W
from tests.helpers import random_circuit, random_state

rng = qsv.Rng(5, "scatter")
for n in (13, 16, 20):
    for cir in (W.cfg3_circuit(n), random_circuit(rng, n, 120)):
        psi = random_state(rng, n)
        want = O.port_forward(n, cir.gates(), init=psi)[0]
        for dt, tol in ((qsv.C128, 1e-12), (qsv.C64, 1e-5)):
            for opts in ({"jit": 1}, {"jit": 1, "tile_bits": 12}):
                p = qsv.Plan(n, cir.gates(), dtype=dt, opts=opts)
                st = qsv.QubitState.from_amplitudes(n, psi, dtype=dt)
                p.execute(st)
                err = np.max(np.abs(st.amplitudes() - want))
                print(n, dt, opts, p.info["npasses"], "err", err, "OK" if err <= tol else "FAIL", flush=True)
# 30q bench plan with 12-bit tiles against the reference fixture
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import importlib
fx = np.load(Path(__file__).resolve().parents[1] / "tests/golden/fullsize/cfg3_30.npz")
n = 30
st = qsv.QubitState(n, dtype=qsv.C128)
st.upload(W.cfg3_input(n))
p = qsv.Plan(n, W.cfg3_circuit(n).gates(), dtype=qsv.C128, opts={"tile_bits": 12})
print("30q passes", p.info["npasses"])
p.execute(st)
a = st.amplitudes()
idx = fx["idx"].astype(np.int64)
print("30q 3-pass samples max err", np.max(np.abs(a[idx] - fx["samples"])))
blocks, z = O.port_digest(n, a)
print("30q blocks max err", np.max(np.abs(blocks - fx["blocks"])), "z", np.max(np.abs(z - fx["z"])))
