"""Adjoint gradients on the GPU against the reference's
own quasar::qubit::adjoint_gradients (adjoint.hpp:52-110, via oracle/_ref),
mirroring proj/tests/test_qubit.cpp:272-374 and test_dist.cpp:224-276."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_18995_b200 import qsv
from paper_2512_18995_b200.qsv import C64, C128, Circuit, QubitState, Rng, kPi, make_gate
from tests.helpers import random_circuit

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def ctx(built):
    return qsv.default_context()


def ref_grads(cir, data=()):
    if not O.REF_LIB.exists():
        pytest.skip("reference library absent")
    obs = [(o.wires, o.basis) for o in cir.observables()]
    return O.ref_adjoint(cir.nqubit(), cir.gates(), obs, list(data))


def test_single_ry_analytic():  # test_qubit.cpp:272-281
    for theta in (0.0, 0.3, -1.2, 2.9):
        cir = Circuit(1)
        cir.ry(0, theta, True)
        cir.observable([0], "z")
        g = qsv.adjoint_gradients(cir)
        assert len(g.param_grads) == 1
        assert abs(g.param_grads[0] + math.sin(theta)) < 1e-10


def test_random_circuits_match_reference():  # test_qubit.cpp:283-345 circuit mix
    rng = Rng(41, "adjoint")
    for trial in range(12):
        n = 2 + rng.next_below(5)
        cir = Circuit(n)
        nparams = 0
        for _ in range(18):
            if nparams >= 20:
                break
            u = rng.uniform()
            if u < 0.3:
                a = rng.next_below(n)
                b = a
                while b == a:
                    b = rng.next_below(n)
                cir.cnot(a, b)
            elif u < 0.45:
                a = rng.next_below(n)
                b = a
                while b == a:
                    b = rng.next_below(n)
                cir.add(make_gate("rzz", [a, b], [], [rng.uniform(-kPi, kPi)], True))
                nparams += 1
            elif u < 0.6:
                a = rng.next_below(n)
                b = a
                while b == a:
                    b = rng.next_below(n)
                cir.cry(a, b, rng.uniform(-kPi, kPi), True)
                nparams += 1
            elif u < 0.75:
                w = rng.next_below(n)
                p = [rng.uniform(-kPi, kPi) for _ in range(3)]
                cir.add(make_gate("u3", [w], [], p, True))
                nparams += 3
            else:
                name = ["rx", "ry", "rz"][rng.next_below(3)]
                w = rng.next_below(n)
                cir.add(make_gate(name, [w], [], [rng.uniform(-kPi, kPi)], True))
                nparams += 1
        cir.observable([0], "z")
        cir.observable([1], "x")
        want_p, _ = ref_grads(cir)
        got = qsv.adjoint_gradients(cir)
        assert len(got.param_grads) == len(want_p)
        assert np.max(np.abs(np.array(got.param_grads) - want_p), initial=0) < 1e-10, trial


def test_encoded_data_gradients():  # test_qubit.cpp:347-366, test_dist.cpp:253-276
    cir = Circuit(4)
    cir.rylayer(encode=True)
    cir.cnot_ring()
    cir.observable([0], "z")
    cir.observable([1], "x")
    data = [0.0, 1.0, 2.0, 3.0]
    _, want_d = ref_grads(cir, data)
    got = qsv.adjoint_gradients(cir, data=data)
    assert np.max(np.abs(np.array(got.data_grads) - want_d)) < 1e-10
    # and against central differences of the GPU forward pass itself
    h = 1e-4
    for i in range(4):
        up, dn = list(data), list(data)
        up[i] += h
        dn[i] -= h
        eu = sum(qsv.expectation(cir.forward(data=[up]), cir))
        ed = sum(qsv.expectation(cir.forward(data=[dn]), cir))
        assert abs(got.data_grads[i] - (eu - ed) / (2 * h)) < 1e-6


def test_dist_mix_circuits_match_reference():  # test_dist.cpp:235-251 gate mix
    rng = Rng(13, "dist-adj")
    for trial in range(5):
        cir = random_circuit(rng, 5, 14)
        cir.observable([0], "z")
        cir.observable([2], "x")
        want_p, _ = ref_grads(cir)
        got = qsv.adjoint_gradients(cir)
        assert np.max(np.abs(np.array(got.param_grads) - want_p), initial=0) < 1e-10


def test_c64_gradients_within_single_precision():
    rng = Rng(3, "adj64")
    cir = random_circuit(rng, 6, 20)
    cir.observable([0, 3], "zz")
    want_p, _ = ref_grads(cir)
    got = qsv.adjoint_gradients(cir, dtype=C64)
    assert np.max(np.abs(np.array(got.param_grads) - want_p), initial=0) < 1e-4


def test_trainable_cfg1_family_matches_reference():
    """The fused single-GPU reverse sweep (one kernel per gate, adjoint.cu)
    on 420 parameters, with X / Y observables and a repeated wire (lambda =
    sum O psi applied wire by wire, adjoint.hpp:30-45)."""
    from paper_2512_18995_b200 import workloads as W

    cir = W.cfg1_circuit(14, trainable=True)
    cir.observable([1, 4], "xy")
    cir.observable([2, 2, 5], "zxy")
    want_p, _ = ref_grads(cir)
    got = qsv.adjoint_gradients(cir)
    assert len(got.param_grads) == 420
    assert np.max(np.abs(np.array(got.param_grads) - want_p)) < 1e-11


def test_errors_mirror_reference():
    cir = Circuit(2)
    cir.ry(0, 0.0, False, True)
    cir.observable([0], "z")
    with pytest.raises(qsv.InvalidInput):  # adjoint.hpp:61-62
        qsv.adjoint_gradients(cir, data=[0.1, 0.2])
    cir = Circuit(1)
    cir.add(make_gate("h", [0], [], [], True))  # trainable without parameters: no gradient entries
    cir.observable([0], "x")
    assert qsv.adjoint_gradients(cir).param_grads == []
