"""Seeded generators restated from the reference's own test suites, so the
parity tests exercise the same gate mixes:

  random_gate     proj/tests/test_qubit.cpp:57-82
  random_circuit  proj/tests/test_dist.cpp:28-57
  random_state    testutil.hpp:38-43 (draws sequenced: re first, then im)
"""
from __future__ import annotations

import numpy as np

from paper_2512_18995_b200.qsv import Circuit, Rng, kPi, make_gate

ONE = ["x", "y", "z", "h", "s", "t", "rx", "ry", "rz", "u3"]
TWO = ["swap", "rxx", "ryy", "rzz"]


def random_gate(rng: Rng, n: int):
    use_two = n >= 2 and rng.uniform() < 0.4
    if use_two:
        name = TWO[rng.next_below(len(TWO))]
        a = rng.next_below(n)
        b = rng.next_below(n)
        while b == a:
            b = rng.next_below(n)
        params = [] if name == "swap" else [rng.uniform(-kPi, kPi)]
        return make_gate(name, [a, b], [], params)
    name = ONE[rng.next_below(len(ONE))]
    w = rng.next_below(n)
    params = []
    if name in ("rx", "ry", "rz"):
        params.append(rng.uniform(-kPi, kPi))
    if name == "u3":
        params = [rng.uniform(-kPi, kPi), rng.uniform(-kPi, kPi), rng.uniform(-kPi, kPi)]
    controls = []
    if n >= 2 and rng.uniform() < 0.3:
        c = rng.next_below(n)
        if c != w:
            controls.append(c)
    return make_gate(name, [w], controls, params)


def random_circuit(rng: Rng, nq: int, ngates: int) -> Circuit:
    cir = Circuit(nq)
    for _ in range(ngates):
        u = rng.uniform()
        a = rng.next_below(nq)
        b = a
        while nq > 1 and b == a:
            b = rng.next_below(nq)
        if u < 0.2:
            cir.cnot(a, b)
        elif u < 0.3:
            cir.cp(a, b, rng.uniform(-kPi, kPi))
        elif u < 0.4:
            cir.swap(a, b)
        elif u < 0.5:
            cir.rzz(a, b, rng.uniform(-kPi, kPi))
        elif u < 0.56:
            cir.rxx(a, b, rng.uniform(-kPi, kPi))
        elif u < 0.62:
            cir.ryy(a, b, rng.uniform(-kPi, kPi))
        elif u < 0.72:
            cir.h(a)
        elif u < 0.82:
            cir.ry(a, rng.uniform(-kPi, kPi), True)
        elif u < 0.92:
            cir.rz(a, rng.uniform(-kPi, kPi), True)
        else:
            cir.cry(a, b, rng.uniform(-kPi, kPi), True)
    return cir


def random_state(rng: Rng, n: int) -> np.ndarray:
    z = np.empty(1 << n, dtype=np.complex128)
    for i in range(1 << n):
        re = rng.normal()
        im = rng.normal()
        z[i] = complex(re, im)
    return z / np.linalg.norm(z)


def dense_apply(psi: np.ndarray, m: np.ndarray, wires, controls, n: int) -> np.ndarray:
    """test_qubit.cpp:29-55: embed by direct bit arithmetic (no striding)."""
    k = len(wires)
    out = np.zeros_like(psi)
    for j in range(len(psi)):
        if not all((j >> (n - 1 - c)) & 1 for c in controls):
            out[j] += psi[j]
            continue
        local = 0
        for w in wires:
            local = (local << 1) | ((j >> (n - 1 - w)) & 1)
        for r in range(1 << k):
            t = j
            for i, w in enumerate(wires):
                bit = 1 << (n - 1 - w)
                if (r >> (k - 1 - i)) & 1:
                    t |= bit
                else:
                    t &= ~bit
            out[t] += m[r, local] * psi[j]
    return out
