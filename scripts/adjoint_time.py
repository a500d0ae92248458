"""Adjoint-gradient timing: the GPU (qsv_adjoint_gradients) and the reference
(oracle/_ref ref_adjoint, one core) on the cfg1 circuit family with every
rotation trainable (600 parameters at 20 qubits), observables Z_i."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
from paper_2512_18995_b200 import qsv, workloads as W
from oracle import oracle as O


def trainable_cfg1(n):
    return W.cfg1_circuit(n, trainable=True)


if __name__ == "__main__":
    for n in [int(a) for a in sys.argv[1:]] or [16, 20]:
        cir = trainable_cfg1(n)
        qsv.adjoint_gradients(cir)
        t = []
        for _ in range(3):
            t0 = time.perf_counter(); g = qsv.adjoint_gradients(cir); t.append(time.perf_counter() - t0)
        t0 = time.perf_counter()
        want, _ = O.ref_adjoint(n, cir.gates(), [(list(o.wires), o.basis) for o in cir.observables()])
        tr = time.perf_counter() - t0
        err = float(np.max(np.abs(np.asarray(g.param_grads) - want)))
        print(f"n={n} params={len(g.param_grads)} gpu {1e3*np.median(t):.1f} ms  ref {tr:.2f} s  max|dg| {err:.2e}", flush=True)
