"""Seeded workloads of BASELINE.json's five configs.

All draws come from quasar::Rng streams Rng(0, "cfgK") (rng.hpp:29-103; the
reference's default seed is 0, tools/main.cpp:619) and are sequenced
explicitly, never as constructor arguments (the reference's testutil idiom
`cdouble(rng.normal(), rng.normal())` depends on argument evaluation order,
SURVEY.md section 4 trap 1). Each generator takes `n` so the same circuit
family also runs at reduced size for full-oracle parity.
"""
from __future__ import annotations

import math

import numpy as np

from .qsv import Circuit, Rng, make_gate, rng_fill, kPi

TWO_PI = 2.0 * kPi


def cfg1_circuit(n: int = 20, layers: int = 10, trainable: bool = False) -> Circuit:
    """20q c128: `layers` x (rx, ry, rz on every qubit; angles U[0,2pi)), then
    the CNOT ladder cnot(q, q+1). Observables: Z_i for every i. `trainable`
    marks every rotation trainable (the adjoint-gradient workload)."""
    rng = Rng(0, "cfg1")
    cir = Circuit(n)
    for _ in range(layers):
        for q in range(n):
            tx = rng.uniform(0.0, TWO_PI)
            ty = rng.uniform(0.0, TWO_PI)
            tz = rng.uniform(0.0, TWO_PI)
            cir.rx(q, tx, trainable)
            cir.ry(q, ty, trainable)
            cir.rz(q, tz, trainable)
    for q in range(n - 1):
        cir.cnot(q, q + 1)
    for q in range(n):
        cir.observable([q], "z")
    return cir


def cfg2_circuit(n: int = 12, layers: int = 6, rows: int = 4096):
    """Batched hardware-efficient VQC: encoded Ry(x_i) layer, then `layers` x
    (trainable U3 on every qubit, ring CZ). Returns (circuit, data rows x n).
    Parameters are drawn first (U[0,2pi)), then the data (U[-pi,pi), row-major).
    U3 angles are shared across rows: the reference's batch semantics
    (circuit.hpp:118-120)."""
    rng = Rng(0, "cfg2")
    cir = Circuit(n)
    cir.rylayer(encode=True)
    for _ in range(layers):
        for q in range(n):
            th = rng.uniform(0.0, TWO_PI)
            ph = rng.uniform(0.0, TWO_PI)
            la = rng.uniform(0.0, TWO_PI)
            cir.add(make_gate("u3", [q], [], [th, ph, la], True))
        for q in range(n):
            cir.cz(q, (q + 1) % n)
    for q in range(n):
        cir.observable([q], "z")
    u = rng_fill_stream(rng, rows * n)
    data = (-kPi + (kPi - (-kPi)) * u).reshape(rows, n)
    return cir, data


def rng_fill_stream(rng: Rng, count: int) -> np.ndarray:
    """Continues `rng`'s uniform stream for `count` draws (vectorised)."""
    out = np.empty(count)
    for i in range(count):
        out[i] = rng.uniform()
    return out


def cfg3_circuit(n: int = 30) -> Circuit:
    """QFT (circuit.hpp:167-178) plus the final swaps the reference omits."""
    cir = Circuit(n)
    for m in range(n):
        cir.h(m)
        k = 2
        for i in range(m, n - 1):
            cir.cp(i + 1, m, kPi / math.pow(2.0, k - 1))
            k += 1
    for i in range(n // 2):
        cir.swap(i, n - 1 - i)
    return cir


def cfg3_input(n: int = 30, nthreads: int = 0) -> np.ndarray:
    """a_i = (re = normal(), im = normal()) from Rng(0, "cfg3"), i ascending,
    normalised in FP64."""
    z = rng_fill(0, "cfg3", "normal", 2 << n, nthreads).view(np.complex128)
    nrm = math.sqrt(float(np.dot(z.view(np.float64), z.view(np.float64))))
    z /= nrm
    return z


def cfg3_slice(lo: int, count: int, nthreads: int = 0) -> np.ndarray:
    """Amplitudes [lo, lo + count) of cfg3_input BEFORE normalisation (a rank's
    slice; the counter-based stream starts at draw 2 * lo). Divide by the
    square root of the all-reduced sum of |a|^2."""
    return rng_fill(0, "cfg3", "normal", 2 * count, nthreads, offset=2 * lo).view(np.complex128)


def cfg4_circuit(n: int = 34, layers: int = 20) -> Circuit:
    """`layers` x (U3 with U[0,2pi) angles on every qubit, brickwork CNOTs:
    even layers cnot(2i, 2i+1), odd layers cnot(2i+1, 2i+2))."""
    rng = Rng(0, "cfg4")
    cir = Circuit(n)
    for layer in range(layers):
        for q in range(n):
            th = rng.uniform(0.0, TWO_PI)
            ph = rng.uniform(0.0, TWO_PI)
            la = rng.uniform(0.0, TWO_PI)
            cir.add(make_gate("u3", [q], [], [th, ph, la]))
        if layer % 2 == 0:
            for i in range(n // 2):
                cir.cnot(2 * i, 2 * i + 1)
        else:
            for i in range((n - 1) // 2):
                cir.cnot(2 * i + 1, 2 * i + 2)
    return cir


def cfg5_circuit(n: int = 36, layers: int = 16) -> Circuit:
    """`layers` x (rx, ry, rz with U[0,2pi) angles on every qubit, then CZ on
    n/2 random pairs from a Fisher-Yates shuffle of 0..n-1 via next_below).
    Observable: Z_0 Z_{n-1}."""
    rng = Rng(0, "cfg5")
    cir = Circuit(n)
    for _ in range(layers):
        for q in range(n):
            tx = rng.uniform(0.0, TWO_PI)
            ty = rng.uniform(0.0, TWO_PI)
            tz = rng.uniform(0.0, TWO_PI)
            cir.rx(q, tx)
            cir.ry(q, ty)
            cir.rz(q, tz)
        perm = list(range(n))
        for i in range(n - 1, 0, -1):
            j = rng.next_below(i + 1)
            perm[i], perm[j] = perm[j], perm[i]
        for i in range(n // 2):
            cir.cz(perm[2 * i], perm[2 * i + 1])
    cir.observable([0, n - 1], "zz")
    return cir


def mirror(cir: Circuit) -> Circuit:
    """C followed by C^dagger (gates reversed, each replaced by its adjoint):
    the full-size known-answer test |0...0> -> |0...0>."""
    from .qsv import gate_matrix

    out = Circuit(cir.nqubit())
    for g in cir.gates():
        out.add(g)
    for g in reversed(cir.gates()):
        m = gate_matrix(g).conj().T
        out.add(make_gate("custom", g.wires, g.controls, [], custom=m))
    return out


def haar_su4(rng: Rng) -> np.ndarray:
    """A Haar-random 4 x 4 unitary from seeded Gaussian draws (QR with the
    phases of R's diagonal folded in); draws sequenced re then im."""
    z = np.empty((4, 4), dtype=np.complex128)
    for i in range(4):
        for j in range(4):
            re = rng.normal()
            im = rng.normal()
            z[i, j] = complex(re, im)
    q, r = np.linalg.qr(z)
    d = np.diag(r)
    return q * (d / np.abs(d))


def dense_brickwork_circuit(n: int = 30, depth: int = 20, seed_label: str = "dense-su4") -> Circuit:
    """Random-circuit-sampling style workload (NOT a BASELINE.json config --
    the demonstration of north_star (2)'s tensor-core blocks where they pay):
    `depth` layers of Haar-random two-qubit unitaries on a brickwork of
    neighbouring wires (even layers (2i, 2i+1), odd layers (2i+1, 2i+2))."""
    rng = Rng(0, seed_label)
    cir = Circuit(n)
    for layer in range(depth):
        for i in range((n - (layer % 2)) // 2):
            a = 2 * i + (layer % 2)
            cir.add(make_gate("custom", [a, a + 1], custom=haar_su4(rng)))
    return cir


def dense_local_circuit(n: int = 30, window: int = 5, depth: int = 20, seed_label: str = "dense-local") -> Circuit:
    """Deep local scrambling (NOT a BASELINE.json config): the wires split into
    windows of `window` neighbours, each window a brickwork of `depth` layers of
    Haar-random two-qubit unitaries -- long runs of genuinely dense gates inside
    5-qubit blocks, the structure where fused tensor-core blocks pay."""
    rng = Rng(0, seed_label)
    cir = Circuit(n)
    for layer in range(depth):
        for w0 in range(0, n, window):
            w1 = min(n, w0 + window)
            for a in range(w0 + (layer % 2), w1 - 1, 2):
                cir.add(make_gate("custom", [a, a + 1], custom=haar_su4(rng)))
    return cir
