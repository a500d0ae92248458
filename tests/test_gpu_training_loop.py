"""Training loops: the same circuit structure with new trainable values every
call. The first call compiles the values in; from the second distinct set on
the engine binds them on the device (lift_policy: trainable gates become
run-time parameters, no new code per call). Every call must still match the
reference: Circuit::forward (circuit.hpp:121-157) and adjoint_gradients
(adjoint.hpp:52-110), max |d| <= 1e-12 (c128) / 1e-5 (c64)."""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_18995_b200 import qsv
from paper_2512_18995_b200.qsv import C64, C128, Circuit, QubitState, make_gate

pytestmark = pytest.mark.gpu
TOL = {C128: 1e-12, C64: 1e-5}


@pytest.fixture(scope="module", autouse=True)
def ctx(built):
    return qsv.default_context()


def layered(n, layers, rng, with_data=False):
    cir = Circuit(n)
    if with_data:
        for q in range(n):
            cir.add(make_gate("ry", [q], [], [0.0], False, True))  # encoded: data slot per wire
    for _ in range(layers):
        for q in range(n):
            cir.rx(q, rng.uniform(0, 2 * math.pi), True)
            cir.ry(q, rng.uniform(0, 2 * math.pi), True)
            cir.rz(q, rng.uniform(0, 2 * math.pi), True)
        cir.add(make_gate("u3", [0], [n - 1], list(rng.uniform(0, 2 * math.pi, 3)), True))
        for q in range(n - 1):
            cir.cnot(q, q + 1)
        cir.add(make_gate("rzz", [0, n - 1], [], [rng.uniform(0, 2 * math.pi)], True))
    for q in range(n):
        cir.observable([q], "z")
    return cir


def ref_forward(n, gates, data=None):
    if O.REF_LIB.exists():
        return O.ref_forward(n, gates, data=data)
    return O.port_forward(n, gates, data=data)


@pytest.mark.parametrize("dtype", [C128, C64])
@pytest.mark.parametrize("n", [6, 12])
def test_forward_with_new_angles_every_call(dtype, n):
    rng = np.random.default_rng(n)
    for step in range(4):
        cir = layered(n, 3, rng)
        out = cir.forward(dtype=dtype)
        want = ref_forward(n, cir.gates())
        got = out.amplitudes(0)
        err = float(np.max(np.abs(got - np.asarray(want).reshape(-1))))
        assert err <= TOL[dtype], (step, err)


def test_forward_with_data_rows_and_new_angles():
    """Encoded data rows plus trainable gates: the lifted slots interleave
    with the caller's data in gate order."""
    n = 5
    rng = np.random.default_rng(7)
    for step in range(3):
        cir = layered(n, 2, rng, with_data=True)
        data = rng.uniform(-math.pi, math.pi, (3, n))
        out = cir.forward(data=data)
        want = np.asarray(ref_forward(n, cir.gates(), data=data.tolist()))
        for b in range(3):
            err = float(np.max(np.abs(out.amplitudes(b) - want[b].reshape(-1))))
            assert err <= 1e-12, (step, b, err)


@pytest.mark.parametrize("dtype", [C128, C64])
def test_adjoint_with_new_angles_every_call(dtype):
    if not O.REF_LIB.exists():
        pytest.skip("reference library absent")
    n = 10
    rng = np.random.default_rng(3)
    for step in range(4):
        cir = layered(n, 2, rng)
        g = qsv.adjoint_gradients(cir, dtype=dtype)
        want, _ = O.ref_adjoint(n, cir.gates(), [(o.wires, o.basis) for o in cir.observables()], [])
        err = float(np.max(np.abs(np.asarray(g.param_grads) - np.asarray(want))))
        assert err <= (1e-11 if dtype == C128 else 2e-4), (step, err)


def test_batched_rows_expect_z_with_new_shared_angles():
    """cfg2-style batched circuits (qsv_run_rows_expect_z): encoded data per
    row, trainable U3 angles shared by the rows and new every call."""
    n, rows = 6, 16
    rng = np.random.default_rng(11)
    for step in range(3):
        cir = Circuit(n)
        for q in range(n):
            cir.add(make_gate("ry", [q], [], [0.0], False, True))
        for _ in range(2):
            for q in range(n):
                cir.add(make_gate("u3", [q], [], list(rng.uniform(0, 2 * math.pi, 3)), True))
            for q in range(n):
                cir.cz(q, (q + 1) % n)
        data = rng.uniform(-math.pi, math.pi, (rows, n))
        z = np.asarray(qsv.run_rows_expect_z(cir, data, dtype=C128))
        amps = np.asarray(ref_forward(n, cir.gates(), data=data.tolist()))
        p = np.abs(amps) ** 2
        idx = np.arange(1 << n)
        want = np.stack([(p * (1 - 2 * ((idx >> (n - 1 - w)) & 1))).sum(axis=1) for w in range(n)], axis=1)
        assert np.max(np.abs(z.reshape(rows, n) - want)) <= 1e-12, step
