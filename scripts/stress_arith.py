"""Randomised stress of the generated kernels' arithmetic (tangent form,
per-register scales, packed complex64) against the oracle: many seeded random
circuits (controls on register slots, tile bits and outside bits; dense
2-qubit gates; swaps) at every register group size. Prints the worst error
per dtype; exits 1 above the north-star bound."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from oracle import oracle as O
from paper_2512_18995_b200 import qsv
from paper_2512_18995_b200.qsv import C64, C128, Circuit, QubitState, Rng
from tests.helpers import random_gate, random_state

TOL = {C128: 1e-12, C64: 1e-5}
worst = {C128: 0.0, C64: 0.0}
rng = Rng(2024, "stress-arith")
count = 0
for trial in range(int(sys.argv[1]) if len(sys.argv) > 1 else 120):
    n = 3 + rng.next_below(14)
    ng = 20 + rng.next_below(160)
    psi = random_state(rng, n)
    gates = [random_gate(rng, n) for _ in range(ng)]
    want = O.port_forward(n, gates, init=psi)[0]
    for dt in (C128, C64):
        for rs in (0, 2, 3, 4):
            cir = Circuit(n)
            for g in gates:
                cir.add(g)
            out = cir.forward(QubitState.from_amplitudes(n, psi, dtype=dt), None, dtype=dt,
                              opts={"jit": 1, "reg_slots": rs})
            err = float(np.max(np.abs(out.amplitudes(0) - want)))
            worst[dt] = max(worst[dt], err)
            count += 1
            if err > TOL[dt]:
                print(f"FAIL trial {trial} n={n} gates={ng} dtype={'c64' if dt == C64 else 'c128'} R={rs} err={err:.3e}")
                sys.exit(1)
print(f"{count} runs ok; worst error c128 {worst[C128]:.3e}, c64 {worst[C64]:.3e}")
