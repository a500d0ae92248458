"""Generates tests/golden/*.json from the REFERENCE itself.

Run in the build container (needs /root/reference): it calls
oracle/_ref/libquasar_ref.so, i.e. the unmodified quasar headers
(Circuit::forward, expectation_one, marginal_probabilities, Rng), on small
seeded cases. The fixtures are committed so parity stays pinned on hosts
without the reference (the GPU box).

    python tests/golden/make_golden.py
"""
import json
import sys
from pathlib import Path

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

import numpy as np  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_2512_18995_b200 import workloads as W  # noqa: E402
from paper_2512_18995_b200.qsv import Circuit, Rng, make_gate  # noqa: E402
from tests.helpers import random_circuit, random_gate, random_state  # noqa: E402

HERE = Path(__file__).resolve().parent


def cj(a):
    a = np.asarray(a, dtype=np.complex128)
    return np.stack([a.real, a.imag], axis=-1).tolist()


def gj(g):
    d = {"name": g.name, "wires": list(g.wires), "controls": list(g.controls), "params": list(g.params),
         "trainable": bool(g.trainable), "encode": bool(g.encode)}
    if g.custom is not None:
        d["custom"] = cj(g.custom)
    return d


def case(name, n, gates, init=None, data=None, obs=(), marg=()):
    out = O.ref_forward(n, gates, init=init, data=data)
    c = {"name": name, "n": n, "gates": [gj(g) for g in gates], "out": cj(out)}
    if init is not None:
        c["init"] = cj(init)
    if data is not None:
        c["data"] = [list(map(float, r)) for r in data]
    if obs:
        c["obs"] = [[list(w), b] for w, b in obs]
        c["expect"] = [O.ref_expectation(n, out[r], obs).tolist() for r in range(out.shape[0])]
    if marg:
        c["marg"] = [list(w) for w in marg]
        c["probs"] = [O.ref_marginal(n, out[0], w).tolist() for w in marg]
    return c


def main():
    O.build()
    cases = []
    cases.append(case("hadamard_on_zero", 1, [make_gate("h", [0])], obs=[([0], "x"), ([0], "z")]))
    init = np.zeros(8, complex)
    init[0b110] = 1
    cases.append(case("toffoli_like", 3, [make_gate("x", [2], [0, 1])], init=init))
    cases.append(case("bell", 2, [make_gate("h", [0]), make_gate("x", [1], [0])], obs=[([0, 1], "zz"), ([0, 1], "xx")],
                      marg=[[0, 1], [1]]))
    ghz = [make_gate("h", [0]), make_gate("x", [1], [0]), make_gate("x", [2], [1])]
    cases.append(case("ghz3", 3, ghz, obs=[([0, 1, 2], "zzz"), ([0, 1, 2], "xxx"), ([0, 2], "yy")]))
    # test_qubit.cpp:100-114 sequence (one 20-gate circuit per n)
    rng = Rng(31, "striding")
    for n in range(1, 7):
        psi = random_state(rng, n)
        gates = [random_gate(rng, n) for _ in range(20)]
        obs = [([q], "z") for q in range(n)] + ([([0, n - 1], "xy")] if n >= 2 else [])
        cases.append(case(f"striding_n{n}", n, gates, init=psi, obs=obs, marg=[[n - 1]]))
    # test_dist.cpp:128-145 circuit mix
    rng = Rng(7, "dist-equiv")
    for t in range(6):
        n = 4 + rng.next_below(5)
        cir = random_circuit(rng, n, 18)
        cases.append(case(f"dist_mix_{t}_n{n}", n, cir.gates(), obs=[([0], "z"), ([1], "x")]))
    # encoding circuit with data rows (test_qubit.cpp:145-193)
    cir = Circuit(3)
    cir.h(0)
    cir.cnot(0, 1)
    cir.x(2, [0])
    cir.rylayer(encode=True)
    cir.cnot_ring()
    cir.rylayer(encode=False)
    cases.append(case("encoding_rows", 3, cir.gates(), data=[[1.0, 2.0, 3.0], [0.1, -0.4, 2.2], [-0.7, 0.9, 0.0]],
                      obs=[([0, 1, 2], "xzx")]))
    # reduced-size members of the five config families
    c1 = W.cfg1_circuit(8, layers=3)
    cases.append(case("cfg1_n8", 8, c1.gates(), obs=[([q], "z") for q in range(8)]))
    c2, data = W.cfg2_circuit(5, layers=2, rows=6)
    cases.append(case("cfg2_n5_rows6", 5, c2.gates(), data=data, obs=[([q], "z") for q in range(5)]))
    c3 = W.cfg3_circuit(7)
    psi = random_state(Rng(0, "cfg3-small"), 7)
    cases.append(case("cfg3_qft7_swaps", 7, c3.gates(), init=psi, marg=[[0, 6]]))
    c4 = W.cfg4_circuit(7, layers=4)
    cases.append(case("cfg4_n7", 7, c4.gates(), obs=[([0], "z"), ([6], "z")]))
    c5 = W.cfg5_circuit(8, layers=3)
    cases.append(case("cfg5_n8", 8, c5.gates(), obs=[([0, 7], "zz")]))
    (HERE / "circuits.json").write_text(json.dumps({"generator": "tests/golden/make_golden.py",
                                                    "source": "oracle/_ref/libquasar_ref.so (reference headers)",
                                                    "cases": cases}))
    rcases = []
    for seed, label, kind, cnt, arg in [(0, "cfg1", 1, 64, 0), (0, "cfg3", 2, 65, 0), (31, "striding", 0, 32, 0),
                                        (0, "cfg5", 3, 40, 36), (7, None, 2, 16, 0)]:
        v = O.ref_rng(seed, label, kind, cnt, arg)
        rcases.append({"seed": seed, "label": label, "kind": kind, "arg": arg,
                       "values": [int(x) for x in v] if kind in (0, 3) else v.tolist()})
    (HERE / "rng.json").write_text(json.dumps({"generator": "tests/golden/make_golden.py", "cases": rcases}))
    print(f"wrote {len(cases)} circuit cases, {len(rcases)} rng streams")


if __name__ == "__main__":
    main()
