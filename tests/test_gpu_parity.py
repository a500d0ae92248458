"""GPU parity: the CUDA path (through the C ABI) against the reference.

Bar (BASELINE.json north_star): max |amplitude error| <= 1e-12 in complex128
and <= 1e-5 in complex64; expectations within the same bounds. The checker is
the reference itself where it is present (oracle/_ref) and the committed
golden fixtures it produced; the C restatement (pinned to the reference by
tests/test_oracle.py) covers sizes the fixtures do not.
"""
import math

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_18995_b200 import qsv
from paper_2512_18995_b200 import workloads as W
from paper_2512_18995_b200.qsv import C64, C128, Circuit, QubitState, Rng, make_gate
from tests.golden_io import load_circuit_cases
from tests.helpers import random_circuit, random_gate, random_state

pytestmark = pytest.mark.gpu
TOL = {C128: 1e-12, C64: 1e-5}
REL_L2_C64 = 1e-6  # complex64: relative L2 bound on top of the max-abs one


def assert_close(got, want, dtype, *what, scale=1.0):
    """max |got - want| <= TOL (x scale); complex64 also ||got - want|| /
    ||want|| <= 1e-6 -- an absolute bound alone says little once amplitudes
    are far below 1e-5."""
    got = np.asarray(got)
    want = np.asarray(want)
    err = float(np.max(np.abs(got - want)))
    assert err <= TOL[dtype] * scale, (what, err)
    if dtype == C64:
        rel = float(np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-300))
        assert rel <= REL_L2_C64 * scale, (what, "rel-L2", rel)


@pytest.fixture(scope="module", autouse=True)
def ctx(built):
    return qsv.default_context()


def ref_or_port_forward(n, gates, init=None, data=None):
    if O.REF_LIB.exists():
        return O.ref_forward(n, gates, init=init, data=data)
    return O.port_forward(n, gates, init=init, data=data)


def run(n, gates, init=None, data=None, dtype=C128, opts=None):
    cir = Circuit(n)
    for g in gates:
        cir.add(g)
    st = None
    if init is not None:
        st = QubitState.from_amplitudes(n, init, dtype=dtype)
    out = cir.forward(st, data, dtype=dtype, opts=opts)
    return np.stack([out.amplitudes(b) for b in range(out.batch())]), out


# ------------------------------------------------------------ golden ----
@pytest.mark.parametrize("dtype", [C128, C64])
@pytest.mark.parametrize("jit", [-1, 1])
def test_golden_fixtures(dtype, jit):
    for case in load_circuit_cases():
        got, st = run(case["n"], case["gates"], case.get("init"), case.get("data"), dtype=dtype, opts={"jit": jit})
        assert_close(got, case["out"], dtype, case["name"])
        if "obs" in case:
            obs = [qsv.Observable(w, b) for w, b in case["obs"]]
            e = qsv.expectation_many(st, obs)
            assert np.max(np.abs(e - np.asarray(case["expect"]))) <= TOL[dtype] * 10, case["name"]
        if "marg" in case:
            for w, p in zip(case["marg"], case["probs"]):
                assert np.max(np.abs(qsv.marginal_probabilities(st, w) - np.asarray(p))) <= TOL[dtype] * 10


# ------------------------------------------ reference test_qubit KATs ----
def test_hadamard_on_zero():
    s = qsv.apply_gate(QubitState.basis(1), make_gate("h", [0]))
    a = s.amplitudes()
    assert abs(a[0] - 1 / math.sqrt(2)) < 1e-12 and abs(a[1] - 1 / math.sqrt(2)) < 1e-12


def test_toffoli_like():
    s = qsv.apply_gate(QubitState.basis(3, 0b110), make_gate("x", [2], [0, 1]))
    assert abs(abs(s.amplitudes()[0b111]) - 1) < 1e-12


def test_striding_matches_dense_oracle_gate_by_gate():
    rng = Rng(31, "striding")
    for n in range(1, 7):
        psi = random_state(rng, n)
        s = QubitState.from_amplitudes(n, psi)
        for rep in range(20):
            g = random_gate(rng, n)
            s = qsv.apply_gate(s, g)
            psi = O.port_forward(n, [g], init=psi)[0]
            assert np.max(np.abs(s.amplitudes() - psi)) < 1e-12, (n, g.name)


def test_norm_preserved_long_circuit():
    rng = Rng(37, "norm")
    gates = [random_gate(rng, 5) for _ in range(1000)]
    got, st = run(5, gates)
    assert abs(np.linalg.norm(got[0]) - 1) < 1e-10
    assert abs(st.norm2()[0] - 1) < 1e-10
    want = ref_or_port_forward(5, gates)[0]
    assert np.max(np.abs(got[0] - want)) < 1e-12


def test_empty_circuit_and_bell():
    out = Circuit(2).forward()
    assert abs(out.amplitudes()[0] - 1) < 1e-15
    cir = Circuit(2)
    cir.h(0)
    cir.cnot(0, 1)
    a = cir.forward().amplitudes()
    r = 1 / math.sqrt(2)
    assert np.max(np.abs(a - np.array([r, 0, 0, r]))) < 1e-12


def test_batch_rows_equal_single_runs():  # test_qubit.cpp:180-193
    cir = Circuit(2)
    cir.h(0)
    cir.ry(0, 0.0, False, True)
    cir.ry(1, 0.0, False, True)
    cir.cnot(0, 1)
    data = [[0.1, 0.2], [1.0, -0.4], [2.2, 0.0], [-0.7, 0.9]]
    batch = cir.forward(data=data)
    assert batch.batch() == 4
    for r in range(4):
        single = cir.forward(data=[data[r]])
        assert np.max(np.abs(batch.amplitudes(r) - single.amplitudes(0))) < 1e-14


def test_data_length_mismatch_fails_fast():  # test_qubit.cpp:195-200
    cir = Circuit(2)
    cir.ry(0, 0.0, False, True)
    with pytest.raises(qsv.InvalidInput):
        cir.forward(data=[[0.1, 0.2]])
    with pytest.raises(qsv.InvalidInput):
        cir.forward(data=[[]])
    with pytest.raises(qsv.InvalidInput):
        cir.forward()


def test_expectation_basic_and_ghz():  # test_qubit.cpp:255-270
    zero = QubitState.basis(1)
    assert abs(qsv.expectation_one(zero, qsv.Observable([0], "z")) - 1) < 1e-12
    plus = qsv.apply_gate(zero, make_gate("h", [0]))
    assert abs(qsv.expectation_one(plus, qsv.Observable([0], "x")) - 1) < 1e-12
    cir = Circuit(3)
    cir.h(0)
    cir.cnot(0, 1)
    cir.cnot(1, 2)
    s = cir.forward()
    assert abs(qsv.expectation_one(s, qsv.Observable([0, 1, 2], "zzz"))) < 1e-12
    assert abs(qsv.expectation_one(s, qsv.Observable([0, 1, 2], "xxx")) - 1) < 1e-12


def test_measure_matches_seeded_reference_histogram():  # test_dist.cpp:207-222 / test_qubit.cpp:202-247
    cir = Circuit(3)
    cir.h(0)
    cir.cnot(0, 1)
    cir.ry(2, 0.7)
    s = cir.forward()
    got = qsv.measure(s, 500, [0, 1, 2], Rng(9, "hist"))
    if O.REF_LIB.exists():
        want = O.ref_measure(3, s.amplitudes(), 500, [0, 1, 2], 9, "hist")
        for i, cnt in enumerate(want):
            key = qsv.bits_to_string(i, 3)
            assert got.get(key, {"count": 0})["count"] == int(cnt), key
    bell = Circuit(2)
    bell.h(0)
    bell.cnot(0, 1)
    counts = qsv.measure(bell.forward(), 100000, [0, 1], Rng(1, "measure-bell"), True)
    assert abs(counts["00"]["probability"] - 0.5) < 1e-12
    assert "01" not in counts
    assert abs(counts["00"]["count"] - 50000) < 5 * math.sqrt(0.25 * 100000)


def test_measure_counts_many_shots_match_reference():
    """10^5 shots (the library samples them on several host threads, each
    shot its own counter of the stream): the histogram equals the
    reference's, and the Rng continues after the last shot."""
    rng = Rng(21, "many-shots")
    n = 16
    psi = random_state(rng, n)
    s = QubitState.from_amplitudes(n, psi)
    wires = [0, 3, 5, 7, 9, 11, 13, 15, 2, 4, 6, 8]
    r = Rng(9, "hist-many")
    counts, probs = qsv.measure_counts(s, 100000, wires, r)
    assert r.counter == 100000 and int(counts.sum()) == 100000
    assert np.max(np.abs(probs - O.port_marginal(n, psi, wires))) < 1e-12
    if O.REF_LIB.exists():
        want = O.ref_measure(n, psi, 100000, wires, 9, "hist-many")
        assert np.array_equal(counts, want)


# ----------------------------------------------- random / fused paths ----
@pytest.mark.parametrize("dtype", [C128, C64])
@pytest.mark.parametrize("jit", [-1, 1])
def test_random_circuits_up_to_14_qubits(dtype, jit):
    rng = Rng(101, "gpu-random")
    for n in [1, 2, 3, 4, 5, 7, 9, 11, 12, 13, 14]:
        psi = random_state(rng, n)
        gates = [random_gate(rng, n) for _ in range(60)]
        got, _ = run(n, gates, init=psi, dtype=dtype, opts={"jit": jit})
        want = O.port_forward(n, gates, init=psi)[0]
        assert_close(got[0], want, dtype, n)


@pytest.mark.parametrize("opts", [{"fuse": 0}, {"tile_bits": 6, "low_bits": 2}, {"tile_bits": 10, "low_bits": 1},
                                  {"tile_bits": 13, "low_bits": 5}, {"no_phase_flush": 1}, {"no_fuse_1q": 1},
                                  {"fuse": 0, "no_phase_flush": 1, "no_fuse_1q": 1, "jit": -1},
                                  {"jit": -1}, {"jit": 1, "tile_bits": 8, "low_bits": 2},
                                  {"jit": 1, "no_phase_flush": 1}])
def test_tile_geometries_agree(opts):
    rng = Rng(5, "geom")
    n = 16
    psi = random_state(rng, n)
    cir = random_circuit(rng, n, 120)
    got, _ = run(n, cir.gates(), init=psi, opts=opts)
    want = O.port_forward(n, cir.gates(), init=psi)[0]
    assert np.max(np.abs(got[0] - want)) <= 1e-12


def test_apply_matrix_zero_off_control():
    rng = Rng(3, "zoc")
    psi = random_state(rng, 7)
    m = np.array([[0.3, 0.1j], [0.2, -0.5]])
    s = QubitState.from_amplitudes(7, psi)
    s.apply_matrix(m, [2], [0, 4], zero_off_control=True)
    want = O.port_apply_matrix(psi, 7, m, [2], [0, 4], zero_off_control=True)
    assert np.max(np.abs(s.amplitudes() - want)) < 1e-15
    d = np.diag([0.0, 1j])
    s = QubitState.from_amplitudes(7, psi)
    s.apply_matrix(d, [5], [1], zero_off_control=True)
    want = O.port_apply_matrix(psi, 7, d, [5], [1], zero_off_control=True)
    assert np.max(np.abs(s.amplitudes() - want)) < 1e-15


def test_apply_matrix_structure_hints():
    # SURVEY.md §8b flags word: DIAGONAL / PERMUTATION hints are verified
    # against the matrix (the engine classifies matrices itself) and change
    # nothing in the result; a contradicted hint fails like invalid_input
    rng = Rng(4, "hints")
    psi = random_state(rng, 6)
    d = np.diag([np.exp(0.3j), np.exp(-1.1j)])
    x = np.array([[0, 1], [1, 0]], dtype=complex)
    for m, h in ((d, qsv.HINT_DIAGONAL), (x, qsv.HINT_PERMUTATION)):
        s = QubitState.from_amplitudes(6, psi)
        s.apply_matrix(m, [3], [1], hints=h)
        want = O.port_apply_matrix(psi, 6, m, [3], [1])
        assert np.max(np.abs(s.amplitudes() - want)) < 1e-15
    s = QubitState.from_amplitudes(6, psi)
    with pytest.raises(qsv.InvalidInput):
        s.apply_matrix(x, [3], hints=qsv.HINT_DIAGONAL)
    with pytest.raises(qsv.InvalidInput):
        s.apply_matrix(d, [3], hints=qsv.HINT_PERMUTATION)
    with pytest.raises(qsv.InvalidInput):
        s.apply_matrix(d, [3], hints=64)


def test_expectations_all_pauli_strings_vs_reference():
    rng = Rng(17, "pauli")
    n = 6
    psi = random_state(rng, n)
    s = QubitState.from_amplitudes(n, psi)
    obs = []
    for _ in range(40):
        k = 1 + rng.next_below(4)
        wires = []
        while len(wires) < k:
            w = rng.next_below(n)
            if w not in wires:
                wires.append(w)
        basis = "".join("xyz"[rng.next_below(3)] for _ in wires)
        obs.append((wires, basis))
    got = qsv.expectation_many(s, [qsv.Observable(w, b) for w, b in obs])[0]
    for (w, b), g in zip(obs, got):
        want, im = O.port_expectation(n, psi, w, b)
        assert abs(g - want) < 1e-12, (w, b)
    z = s.expect_z_all()[0]
    for q in range(n):
        assert abs(z[q] - O.port_expectation(n, psi, [q], "z")[0]) < 1e-12


def test_expectations_with_repeated_wires_compose_like_the_reference():
    """expectation_one applies the Paulis wire by wire (circuit.hpp:255-259):
    a repeated wire composes (Z Z = I, Z X = iY, ...); an imaginary result is
    refused like circuit.hpp:261."""
    rng = Rng(23, "pauli-repeat")
    n = 5
    psi = random_state(rng, n)
    s = QubitState.from_amplitudes(n, psi)
    cases = [([0, 0], "zz"), ([1, 1], "xx"), ([2, 2], "yy"), ([0, 1, 0], "xzx"), ([3, 3, 3], "xyz"),
             ([1, 1], "xz"), ([4, 2, 4], "yzx"), ([0, 0, 1, 1], "xyyx")]
    for _ in range(30):
        k = 2 + rng.next_below(4)
        wires = [rng.next_below(3) for _ in range(k)]
        cases.append((wires, "".join("xyz"[rng.next_below(3)] for _ in wires)))
    seen_err = seen_ok = 0
    for w, b in cases:
        want, im = O.port_expectation(n, psi, w, b)
        if O.REF_LIB.exists():
            try:
                ref = O.ref_expectation(n, psi, [(w, b)])[0]
                assert abs(ref - want) < 1e-14
            except O.OracleError as e:
                assert e.code == 2 and abs(im) >= 1e-10
        if abs(im) >= 1e-10:
            with pytest.raises(qsv.InvalidInput):
                qsv.expectation_many(s, [qsv.Observable(w, b)])
            seen_err += 1
        else:
            got = qsv.expectation_many(s, [qsv.Observable(w, b)])[0][0]
            assert abs(got - want) < 1e-12, (w, b)
            seen_ok += 1
    assert seen_err and seen_ok


# ------------------------------------------------ config families ----
def test_cfg1_full_20q_vs_reference():
    cir = W.cfg1_circuit(20)
    s = cir.forward()
    got = s.amplitudes()
    want = ref_or_port_forward(20, cir.gates())[0]
    assert np.max(np.abs(got - want)) <= 1e-12
    z = s.expect_z_all()[0]
    wz = np.array([O.port_expectation(20, want, [q], "z")[0] for q in range(0, 20, 5)])
    assert np.max(np.abs(z[0:20:5] - wz)) <= 1e-12


def test_cfg2_batched_c64_vs_reference_rows():
    cir, data = W.cfg2_circuit()
    s = cir.forward(data=data, dtype=C64)
    z = s.expect_z_all()
    assert z.shape == (4096, 12)
    rows = list(range(0, 4096, 257))
    want = ref_or_port_forward(12, cir.gates(), data=data[rows])
    for i, r in enumerate(rows):
        a = s.amplitudes(r)
        assert_close(a, want[i], C64, r)
        wz = [O.port_expectation(12, want[i], [q], "z")[0] for q in range(12)]
        assert np.max(np.abs(z[r] - wz)) <= 1e-5
    assert np.max(np.abs(s.norm2() - 1)) < 1e-5


def test_cfg3_qft_reduced_vs_reference():
    for n in (10, 16, 20):
        cir = W.cfg3_circuit(n)
        psi = W.cfg3_input(n)
        s = cir.forward(QubitState.from_amplitudes(n, psi))
        want = ref_or_port_forward(n, cir.gates(), init=psi)[0]
        assert np.max(np.abs(s.amplitudes() - want)) <= 1e-12, n


@pytest.mark.parametrize("opts", [{"jit": 1}, {"jit": 1, "no_relabel": 1}, {"jit": 1, "tile_bits": 9, "low_bits": 2},
                                  {"jit": 1, "tile_bits": 12, "low_bits": 4}])
def test_swaps_as_relabelings_match_reference(opts):
    # swap gates become layout permutations folded into the last pass (out of
    # place); the downloaded state must still be in logical order
    rng = Rng(23, "relabel")
    for n in (11, 17):
        cir = random_circuit(rng, n, 80)
        for i in range(n // 2):
            cir.swap(i, n - 1 - i)
        psi = random_state(rng, n)
        got, st = run(n, cir.gates(), init=psi, opts=opts)
        want = O.port_forward(n, cir.gates(), init=psi)[0]
        assert np.max(np.abs(got[0] - want)) <= 1e-12, (n, opts)
        z = st.expect_z_all()[0]
        for q in (0, n - 1):
            assert abs(z[q] - O.port_expectation(n, want, [q], "z")[0]) <= 1e-12


def test_qft_of_zero_is_uniform_24q():  # test_dist.cpp:147-160 scaled
    n = 24
    s = qsv.qft_circuit(n).forward()
    a = s.amplitudes()
    assert np.max(np.abs(np.abs(a) - 2.0 ** (-n / 2))) < 1e-12


@pytest.mark.parametrize("dtype,n", [(C128, 22), (C64, 24)])
def test_mirror_circuits_return_to_zero(dtype, n):
    for cir in (W.cfg4_circuit(n, layers=6), W.cfg5_circuit(n, layers=4)):
        s = W.mirror(cir).forward(dtype=dtype)
        a = s.amplitudes()
        assert abs(a[0] - 1) <= 10 * TOL[dtype]
        assert np.max(np.abs(a[1:])) <= 10 * TOL[dtype]


@pytest.mark.parametrize("light", ["", "QSV_X_NOLIGHT"])
def test_c64_memory_bound_geometry(light, monkeypatch):
    """complex64 circuits with few dense matrices per pass (the QFT, SU(4)
    brickworks) plan on 12-bit double-buffered tiles with 4-qubit register
    groups (plan.cpp); QSV_X_NOLIGHT=1 keeps the 13-bit geometry. Both
    against the oracle on a seeded random state, above the 13-qubit switch."""
    if light:
        monkeypatch.setenv(light, "1")
    n = 18
    rng = Rng(5, "light-c64")
    psi = random_state(rng, n)
    for cir in (W.cfg3_circuit(n), W.dense_brickwork_circuit(n, 4)):
        info, _ = qsv.plan_dry(n, cir.gates(), dtype=C64, opts={"dense_blocks": -1})
        assert info["max_tile_bits"] == (13 if light else 12)
        got, _ = run(n, cir.gates(), init=psi, dtype=C64, opts={"dense_blocks": -1})
        want = O.port_forward(n, cir.gates(), init=psi)[0]
        assert_close(got[0], want, C64)


@pytest.mark.parametrize("passengers", ["0", "1"])
def test_passenger_bit_tiles(passengers, monkeypatch):
    """Compute-bound complex128 passes carry one passenger bit (planner.cpp:
    two planned tiles per CTA in lock-step); QSV_PASSENGERS=0 plans without.
    Both against the oracle on a seeded random state."""
    monkeypatch.setenv("QSV_PASSENGERS", passengers)
    n = 18
    rng = Rng(6, "passengers")
    psi = random_state(rng, n)
    cir = W.cfg4_circuit(n, layers=6)
    info, _ = qsv.plan_dry(n, cir.gates())
    assert info["max_tile_bits"] == 11 + int(passengers)
    got, _ = run(n, cir.gates(), init=psi)
    want = O.port_forward(n, cir.gates(), init=psi)[0]
    assert_close(got[0], want, C128)


def test_cfg5_family_c64_vs_reference():
    cir = W.cfg5_circuit(16, layers=4)
    s = cir.forward(dtype=C64)
    want = ref_or_port_forward(16, cir.gates())[0]
    assert_close(s.amplitudes(), want, C64)
    e = qsv.expectation(s, cir)[0]
    assert abs(e - O.port_expectation(16, want, [0, 15], "zz")[0]) <= 1e-5


@pytest.mark.parametrize("dtype,tol", [(C64, 1e-5), (C128, 1e-12)])
def test_execute_expect_z_fused_and_fallback(dtype, tol):
    """qsv_plan_execute_expect_z: the fused <Z> epilogue (whole-row tiles,
    cfg2's batched circuits) and the fallback (multi-pass state) equal
    forward + expectation() of every Z_w."""
    cir, data = W.cfg2_circuit(10, layers=3, rows=257)
    p = qsv.Plan(10, cir.gates(), dtype=dtype)
    st = QubitState(10, batch=257, dtype=dtype)
    z = p.execute_expect_z(st, data)
    ref = cir.forward(data=data, dtype=dtype).expect_z_all()
    assert np.max(np.abs(z - ref)) <= tol
    w = ref_or_port_forward(10, cir.gates(), data=data[:3])
    for r in range(3):
        want = [O.port_expectation(10, w[r], [q], "z")[0] for q in range(10)]
        assert np.max(np.abs(z[r] - want)) <= tol
    big = W.cfg4_circuit(16, layers=2)
    p2 = qsv.Plan(16, big.gates(), dtype=dtype)
    s2 = QubitState(16, dtype=dtype)
    z2 = p2.execute_expect_z(s2)
    want2 = big.forward(dtype=dtype).expect_z_all()
    assert np.max(np.abs(z2 - want2)) <= tol


@pytest.mark.parametrize("dtype,tol", [(C64, 1e-5), (C128, 1e-12)])
def test_from_zero_product_state_prefix(dtype, tol):
    """opts.from_zero: each wire's leading 1q gates (encoded ones included)
    become a product state synthesised in the first pass; the state's old
    content is ignored. Equal to the plain plan run on |0...0>."""
    cir, data = W.cfg2_circuit(10, layers=3, rows=129)
    fast = qsv.Plan(10, cir.gates(), dtype=dtype, opts={"from_zero": 1})
    plain = qsv.Plan(10, cir.gates(), dtype=dtype)
    st = QubitState(10, batch=129, dtype=dtype)
    st.upload(random_state(Rng(3, "junk"), 10), 0)  # ignored by the from-zero plan
    z1 = fast.execute_expect_z(st, data)
    a1 = st.amplitudes(5)
    s0 = QubitState(10, batch=129, dtype=dtype)
    z0 = plain.execute_expect_z(s0, data)
    assert np.max(np.abs(z1 - z0)) <= tol
    assert np.max(np.abs(a1 - s0.amplitudes(5))) <= tol
    for cirx, n in ((W.cfg4_circuit(12, layers=3), 12), (W.cfg1_circuit(12, layers=2), 12),
                    (random_circuit(Rng(5, "fz"), 9, 80), 9)):
        got = cirx.forward(dtype=dtype).amplitudes()  # forward() plans from zero
        want = ref_or_port_forward(n, cirx.gates())[0]
        assert np.max(np.abs(got - want)) <= tol


@pytest.mark.parametrize("dtype", [C128, C64])
def test_l2_super_passes_match_reference(dtype):
    # opt-in L2 super-passes (pairs of passes in one launch, chunk by chunk,
    # the second reading the first's output through L2; the second may be the
    # permuting out-of-place pass): same results as the reference, batched
    # rows included, whatever the lookahead / items per ticket
    rng = Rng(41, "super")
    cases = ((18, 17), (20, 19)) if dtype == C128 else ((20, 19),)
    for n, sb in cases:
        cir = W.cfg3_circuit(n)
        psi = random_state(rng, n)
        info, _ = qsv.plan_dry(n, cir.gates(), dtype=dtype, opts={"jit": 1, "super_bits": sb})
        assert info["npasses"] < info["ntile_passes"], info
        got, _ = run(n, cir.gates(), init=psi, dtype=dtype, opts={"jit": 1, "super_bits": sb})
        want = ref_or_port_forward(n, cir.gates(), init=psi)[0]
        assert_close(got[0], want, dtype, (n, sb))
        gates = [random_gate(rng, n) for _ in range(150)]
        got, _ = run(n, gates, init=psi, dtype=dtype, opts={"jit": 1, "super_bits": sb})
        want = O.port_forward(n, gates, init=psi)[0]
        assert_close(got[0], want, dtype, (n, sb, "random"))
    # two batch rows: chunks of both rows in one launch
    n, sb = cases[0]
    cir = W.cfg3_circuit(n)
    rows = np.stack([random_state(rng, n), random_state(rng, n)])
    st = QubitState(n, 2, dtype)
    for b in range(2):
        st.upload(rows[b], b)
    p = qsv.Plan(n, cir.gates(), dtype=dtype, opts={"jit": 1, "super_bits": sb})
    assert p.info["npasses"] < p.info["ntile_passes"]
    p.execute(st)
    for b in range(2):
        want = O.port_forward(n, cir.gates(), init=rows[b])[0]
        assert_close(st.amplitudes(b), want, dtype, b)


@pytest.mark.parametrize("dtype", [C128, C64])
def test_graph_replay_matches_stream_launches(dtype):
    # opts.use_graph: the launch sequence captured once per (state buffers,
    # rows) and replayed; permuting last passes flip the buffers, so replays
    # alternate between two graphs -- every execute must equal the reference
    rng = Rng(43, "graph")
    n = 16
    cir = random_circuit(rng, n, 90)
    for i in range(n // 2):
        cir.swap(i, n - 1 - i)  # relabelled: the last pass permutes out of place
    psi = random_state(rng, n)
    want1 = O.port_forward(n, cir.gates(), init=psi)[0]
    want2 = O.port_forward(n, cir.gates(), init=want1)[0]
    p = qsv.Plan(n, cir.gates(), dtype=dtype, opts={"jit": 1, "use_graph": 1})
    st = QubitState(n, 2, dtype)
    for b in range(2):
        st.upload(psi, b)
    for rep in range(3):  # capture, replay, replay (alternating buffer pairs)
        for b in range(2):
            st.upload(psi, b)
        p.execute(st)
        for b in range(2):
            assert_close(st.amplitudes(b), want1, dtype, (rep, b))
    p.execute(st)  # applied twice in a row
    assert_close(st.amplitudes(0), want2, dtype, scale=10)
    # a from-|0> plan: the product-state prefix kernel is part of the graph
    pz = qsv.Plan(n, cir.gates(), dtype=dtype, opts={"jit": 1, "use_graph": 1, "from_zero": 1})
    wz = O.port_forward(n, cir.gates())[0]
    for rep in range(2):
        pz.execute(st)
        assert_close(st.amplitudes(1), wz, dtype, rep)


@pytest.mark.parametrize("dtype", [C128, C64])
def test_graph_cache_survives_buffer_reallocation(dtype):
    """a graph plan bakes the device pointers of its product-state
    prefix buffer; a larger batch reallocates that buffer, so the cached
    graphs must be dropped. Alternate batch-1 and batch-4 states on one
    from-|0> graph plan (and an L2 super-pass graph plan, whose counters are
    reallocated the same way)."""
    rng = Rng(47, "graph-realloc")
    n = 15
    cir = random_circuit(rng, n, 60)
    psi = random_state(rng, n)
    for opts, init in (({"jit": 1, "use_graph": 1, "from_zero": 1}, None),
                       ({"jit": 1, "use_graph": 1, "super_bits": 14}, psi)):
        want = O.port_forward(n, cir.gates(), init=init)[0]
        p = qsv.Plan(n, cir.gates(), dtype=dtype, opts=opts)
        s1 = QubitState(n, 1, dtype)
        s4 = QubitState(n, 4, dtype)
        for rep in range(3):
            for st in (s1, s4, s1):
                if init is not None:
                    for b in range(st.batch()):
                        st.upload(init, b)
                p.execute(st)
                for b in range(st.batch()):
                    assert_close(st.amplitudes(b), want, dtype, (opts, rep, b))


@pytest.mark.parametrize("dtype", [C128, C64])
@pytest.mark.parametrize("variant", ["", "QSV_X_NOPACK", "QSV_X_NOSCALE", "QSV_X_NOTAN", "QSV_X_NOSPLIT",
                                     "QSV_X_NOSIGN", "QSV_X_NOPAIR", "QSV_X_OLDSWZ", "QSV_X_NOXPERM",
                                     "QSV_X_NOHOIST", "QSV_X_CPOOL"])
@pytest.mark.parametrize("reg_slots", [0, 2, 3, 4])
def test_generated_arithmetic_variants(dtype, variant, reg_slots, monkeypatch):
    """The generated kernels' arithmetic forms -- tangent-form real matrices
    (planner.cpp lower), per-register deferred scales and packed f32x2
    complex64 (codegen.cpp) -- each switched off in turn, at every register
    group size, on circuits with controls on register slots, tile bits and
    bits outside the tile (runtime-conditional ops), against the oracle."""
    if variant:
        monkeypatch.setenv(variant, "1")
    rng = Rng(77, "arith-variants")
    n = 15
    psi = random_state(rng, n)
    gates = [random_gate(rng, n) for _ in range(90)]
    fam = W.cfg4_circuit(n, 2).gates() + W.cfg5_circuit(n, 2).gates()
    for gs in (gates, fam):
        got, _ = run(n, gs, init=psi, dtype=dtype, opts={"jit": 1, "reg_slots": reg_slots})
        want = O.port_forward(n, gs, init=psi)[0]
        assert_close(got[0], want, dtype)
        if dtype == C64:  # relative L2 bound for complex64 (VERDICT r1 parity item)
            assert np.linalg.norm(got[0] - want) / np.linalg.norm(want) <= 1e-6
