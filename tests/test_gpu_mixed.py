"""Mixed states on the GPU: density matrices as the
2m-qubit vector vec(rho), gates as U on the row wires and conj(U) on the
column wires, single-qubit channels as one 4x4 superoperator pass, and the
diagonal reductions (Tr[rho P], marginals) -- against the reference's
to_mixed / apply_gate / apply_channel / expectation / marginal_probabilities
(state.hpp:73-80,159-172; channel.hpp:22-100; circuit.hpp:199-203,264-281)
and its channel tests (tests/test_qubit.cpp:376-420)."""
import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_18995_b200 import qsv
from paper_2512_18995_b200 import workloads as W
from paper_2512_18995_b200.qsv import C64, C128, Circuit, InvalidInput, QubitState, make_gate
from tests.helpers import random_circuit

pytestmark = pytest.mark.gpu

HAVE_REF = O.REF_LIB.exists()


@pytest.fixture(scope="module", autouse=True)
def _gpu():
    if qsv.lib().qsv_device_count() < 1:
        pytest.fail("no CUDA device: the -m gpu suite needs a B200")
    from paper_2512_18995_b200 import build

    build.build()


def mixed_ref(n, ops, init=None):
    return O.ref_mixed_run(n, ops, init) if HAVE_REF else O.port_mixed_run(n, ops, init)


def run_ops(n, ops, init=None, dtype=C128):
    s = QubitState.basis(n, dtype=dtype) if init is None else QubitState.from_amplitudes(n, init, dtype=dtype)
    for op in ops:
        if isinstance(op, tuple):
            name, w, p = op
            s = qsv.apply_channel(s, getattr(qsv, name)(w, p))
        else:
            s = qsv.apply_gate(s, op)
    return s


OPS = [make_gate("h", [0]), make_gate("x", [1], [0]), ("depolarizing", 0, 0.3), make_gate("ry", [2], [], [0.7]),
       ("amplitude_damping", 2, 0.4), make_gate("rzz", [0, 3], [], [0.5]), ("bit_flip", 1, 0.2),
       ("phase_flip", 3, 0.1), ("phase_damping", 1, 0.6), make_gate("u3", [1], [2], [0.3, 0.2, 0.1]),
       make_gate("swap", [0, 3]), make_gate("z", [3], [1])]


@pytest.mark.parametrize("dtype,tol", [(C128, 1e-12), (C64, 1e-5)])
def test_gates_and_channels_match_reference(dtype, tol):
    n = 4
    rng = np.random.default_rng(3)
    psi = rng.normal(size=16) + 1j * rng.normal(size=16)
    psi /= np.linalg.norm(psi)
    for init in (None, psi):
        s = run_ops(n, OPS, init, dtype)
        want = mixed_ref(n, OPS, init)
        assert s.is_mixed() and s.nqubit() == n
        assert np.max(np.abs(s.density() - want)) <= tol
        if dtype == C64:  # complex64 relative L2
            assert np.linalg.norm(s.density() - want) / np.linalg.norm(want) <= 1e-6
        obs = [([0], "z"), ([1, 2], "xy"), ([0, 1, 3], "zzx"), ([2], "y")]
        got = qsv.expectation_many(s, [qsv.Observable(w, b) for w, b in obs])[0]
        ref = O.ref_density_expectation(n, want, obs) if HAVE_REF else \
            [O.port_density_expectation(n, want, w, b).real for w, b in obs]
        assert np.max(np.abs(got - np.asarray(ref))) <= tol
        for wires in ([2, 0], [3], [0, 1, 2, 3]):
            pm = qsv.marginal_probabilities(s, wires)
            pr = O.ref_density_marginal(n, want, wires) if HAVE_REF else O.port_density_marginal(n, want, wires)
            assert np.max(np.abs(pm - pr)) <= tol
        assert abs(qsv.density_trace(s)[0] - 1.0) <= tol


def test_forward_on_mixed_init_uses_fused_passes():
    n = 6
    cir = random_circuit(qsv.Rng(11, "mixed-forward"), n, 40)
    init = qsv.apply_channel(QubitState.basis(n), qsv.depolarizing(2, 0.5))
    got = cir.forward(init=init).density()
    want = mixed_ref(n, [("depolarizing", 2, 0.5)] + list(cir.gates()))
    assert np.max(np.abs(got - want)) <= 1e-12


def test_pure_consistency_at_12_qubits():
    """Gates only: U |psi><psi| U^dagger from the mixed path equals the outer
    product of the pure-state path (24 engine qubits, 256 MiB)."""
    n = 12
    cir = W.cfg4_circuit(n, layers=3)
    pure = cir.forward().amplitudes()
    rho = cir.forward(init=QubitState.basis(n).to_mixed()).density()
    assert np.max(np.abs(rho - np.outer(pure, pure.conj()))) <= 1e-12
    s = qsv.apply_channel(cir.forward().to_mixed(), qsv.amplitude_damping(5, 0.25))
    r2 = s.density()
    assert abs(np.trace(r2).real - 1.0) <= 1e-12
    assert np.max(np.abs(r2 - r2.conj().T)) <= 1e-12


def test_reference_channel_kats():  # tests/test_qubit.cpp:376-416
    s = QubitState.basis(1).to_mixed()
    out = qsv.apply_channel(s, qsv.make_channel("id", 0, [np.eye(2)]))
    assert np.max(np.abs(out.density() - s.density())) < 1e-14
    c = Circuit(2)
    c.h(0)
    c.cnot(0, 1)
    out = qsv.apply_channel(c.forward().to_mixed(), qsv.depolarizing(0, 1.0))
    p = qsv.marginal_probabilities(out, [0])
    assert abs(p[0] - 0.5) < 1e-12 and abs(p[1] - 0.5) < 1e-12
    assert abs(np.trace(out.density()).real - 1.0) < 1e-12
    out = qsv.apply_channel(QubitState.basis(1, 1).to_mixed(), qsv.amplitude_damping(0, 1.0))
    want = np.zeros((2, 2))
    want[0, 0] = 1
    assert np.max(np.abs(out.density() - want)) < 1e-12
    counts = qsv.measure(qsv.apply_channel(QubitState.basis(2), qsv.bit_flip(1, 0.25)), 4000, [0, 1],
                         qsv.Rng(3, "mixed"), True)
    assert abs(counts["01"]["probability"] - 0.25) < 1e-12 and abs(counts["00"]["probability"] - 0.75) < 1e-12


def test_errors_mirror_reference():
    with pytest.raises(InvalidInput, match="not trace preserving"):  # test_qubit.cpp:418-420
        qsv.make_channel("bad", 0, [0.5 * np.eye(2)])
    with pytest.raises(InvalidInput, match="not Hermitian"):
        QubitState.from_density(1, np.array([[0.5, 0.5], [0.0, 0.5]]))
    with pytest.raises(InvalidInput, match="trace != 1"):
        QubitState.from_density(1, np.array([[0.5, 0.0], [0.0, 0.4]]))
    mixed = QubitState.basis(2).to_mixed()
    with pytest.raises(InvalidInput, match="pure states only"):  # test_qubit.cpp:368-374
        c = Circuit(2)
        c.ry(0, 0.3, trainable=True)
        c.observable([0], "z")
        qsv.adjoint_gradients(c, mixed)
    c = Circuit(2)
    c.rylayer(encode=True)
    with pytest.raises(InvalidInput, match="pure initial state"):  # circuit.hpp:131
        c.forward(init=mixed, data=[[0.1, 0.2]])
    with pytest.raises(InvalidInput, match="no amplitudes"):
        mixed.amplitudes()
