"""Pins the CPU oracle before it is trusted (CPU only, no GPU).

1. The C restatement (oracle/qsv_oracle.c) against the reference itself
   (oracle/_ref/libquasar_ref.so = the unmodified quasar headers), on the
   reference's own known-answer tests (proj/tests/test_qubit.cpp) and seeded
   random circuits.
2. Both against the committed golden fixtures (tests/golden/*.json, made by
   tests/golden/make_golden.py from the reference library), so the pin holds
   on hosts without /root/reference.
"""
import json
import math
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_18995_b200.qsv import Rng, kPi, make_gate
from tests.helpers import dense_apply, random_circuit, random_gate, random_state

GOLD = Path(__file__).resolve().parent / "golden"
HAVE_REF = O.REF_LIB.exists() or O.REFERENCE_INCLUDE.exists()


@pytest.fixture(scope="module", autouse=True)
def _build():
    O.build()


def needs_ref():
    if not O.REF_LIB.exists():
        pytest.skip("reference library not built (needs /root/reference)")


# ---------------------------------------------------------------- Rng ----
def test_python_rng_matches_reference_stream():
    needs_ref()
    for seed, label in [(0, "cfg1"), (31, "striding"), (7, None)]:
        r = Rng(seed, label) if label else Rng(seed)
        got = [r.next_u64() for _ in range(64)]
        want = O.ref_rng(seed, label, 0, 64)
        assert got == [int(x) for x in want]
        r = Rng(seed, label) if label else Rng(seed)
        got = [r.normal() for _ in range(33)]
        assert np.array_equal(np.array(got), O.ref_rng(seed, label, 2, 33))
        r = Rng(seed, label) if label else Rng(seed)
        got = [r.next_below(37) for _ in range(50)]
        assert got == [int(x) for x in O.ref_rng(seed, label, 3, 50, 37)]


def test_port_rng_matches_reference():
    needs_ref()
    for kind in (0, 1, 2, 3):
        assert np.array_equal(O.port_rng(5, "dist-equiv", kind, 101, 13), O.ref_rng(5, "dist-equiv", kind, 101, 13))


# ------------------------------------------------------- gate matrices ----
GATES = [
    ("x", [0], []), ("y", [0], []), ("z", [0], []), ("h", [0], []), ("s", [0], []), ("t", [0], []),
    ("rx", [0], [0.3]), ("ry", [0], [-1.2]), ("rz", [0], [2.9]), ("p", [0], [0.7]),
    ("u3", [0], [0.1, -0.4, 2.2]), ("swap", [0, 1], []), ("rxx", [0, 1], [0.9]), ("ryy", [0, 1], [-2.1]),
    ("rzz", [0, 1], [1.3]),
]


@pytest.mark.parametrize("name,wires,params", GATES)
def test_port_gate_matrix_matches_reference(name, wires, params):
    needs_ref()
    g = make_gate(name, wires, [], params)
    assert np.array_equal(O.port_gate_matrix(g), O.ref_gate_matrix(g))


# -------------------------------------------- KATs (test_qubit.cpp) -------
def test_kat_hadamard_on_zero():  # test_qubit.cpp:86-91
    out = O.port_forward(1, [make_gate("h", [0])])[0]
    r = 1 / math.sqrt(2.0)
    assert abs(out[0] - r) < 1e-12 and abs(out[1] - r) < 1e-12


def test_kat_toffoli_like():  # test_qubit.cpp:93-98
    init = np.zeros(8, complex)
    init[0b110] = 1
    out = O.port_forward(3, [make_gate("x", [2], [0, 1])], init=init)[0]
    assert abs(abs(out[0b111]) - 1) < 1e-12


def test_kat_striding_matches_dense_oracle():  # test_qubit.cpp:100-114
    rng = Rng(31, "striding")
    for n in range(1, 7):
        psi = random_state(rng, n)
        state = psi.copy()
        for _ in range(20):
            g = random_gate(rng, n)
            state = O.port_forward(n, [g], init=state)[0]
            psi = dense_apply(psi, O.port_gate_matrix(g), g.wires, g.controls, n)
            assert np.max(np.abs(state - psi)) < 1e-12, (n, g.name)


def test_kat_norm_preserved():  # test_qubit.cpp:116-122
    rng = Rng(37, "norm")
    gates = [random_gate(rng, 5) for _ in range(1000)]
    out = O.port_forward(5, gates)[0]
    assert abs(np.linalg.norm(out) - 1) < 1e-10


def test_kat_bell_and_ghz_expectations():  # test_qubit.cpp:130-140, 255-270
    bell = O.port_forward(2, [make_gate("h", [0]), make_gate("x", [1], [0])])[0]
    r = 1 / math.sqrt(2)
    assert np.allclose(bell, [r, 0, 0, r], atol=1e-12)
    ghz = O.port_forward(3, [make_gate("h", [0]), make_gate("x", [1], [0]), make_gate("x", [2], [1])])[0]
    assert abs(O.port_expectation(3, ghz, [0, 1, 2], "zzz")[0]) < 1e-12
    assert abs(O.port_expectation(3, ghz, [0, 1, 2], "xxx")[0] - 1) < 1e-12


def test_port_matches_reference_random_circuits():
    needs_ref()
    rng = Rng(7, "dist-equiv")
    for trial in range(12):
        n = 4 + rng.next_below(5)
        cir = random_circuit(rng, n, 18)
        a = O.port_forward(n, cir.gates())[0]
        b = O.ref_forward(n, cir.gates())[0]
        assert np.max(np.abs(a - b)) <= 1e-15, trial


def test_port_matches_reference_encoded_batch():  # test_qubit.cpp:145-193
    needs_ref()
    from paper_2512_18995_b200.qsv import Circuit

    cir = Circuit(3)
    cir.h(0)
    cir.cnot(0, 1)
    cir.x(2, [0])
    cir.rylayer(encode=True)
    cir.cnot_ring()
    cir.rylayer(encode=False)
    data = [[1.0, 2.0, 3.0], [0.1, -0.2, 0.3]]
    a = O.port_forward(3, cir.gates(), data=data)
    b = O.ref_forward(3, cir.gates(), data=data)
    assert np.max(np.abs(a - b)) <= 1e-15
    e1 = O.port_expectation(3, a[0], [0, 1, 2], "xzx")[0]
    e2 = O.ref_expectation(3, b[0], [([0, 1, 2], "xzx")])[0]
    assert abs(e1 - e2) < 1e-15


def test_reference_rejects_data_length_mismatch():  # test_qubit.cpp:195-200
    needs_ref()
    g = [make_gate("ry", [0], [], [0.0], False, True)]
    with pytest.raises(O.OracleError) as e:
        O.ref_forward(2, g, data=[[0.1, 0.2]])
    assert e.value.code == 2


def test_port_marginal_and_zero_off_control_match_reference():
    needs_ref()
    rng = Rng(3, "marg")
    psi = random_state(rng, 6)
    for wires in ([0], [2, 5], [5, 1, 3]):
        assert np.allclose(O.port_marginal(6, psi, wires), O.ref_marginal(6, psi, wires), atol=1e-15)
    # zero_off_control: restate by hand (adjoint.hpp:99-101 uses it)
    m = np.array([[0.3, 0.1j], [0.2, -0.5]])
    out = O.port_apply_matrix(psi, 6, m, [2], [0, 4], zero_off_control=True)
    want = np.zeros_like(psi)
    for i in range(64):
        on = (i >> 5) & 1 and (i >> 1) & 1
        if not on:
            continue
        b = (i >> 3) & 1
        j0 = i & ~(1 << 3)
        want[i] = m[b, 0] * psi[j0] + m[b, 1] * psi[j0 | (1 << 3)]
    assert np.max(np.abs(out - want)) < 1e-15


# --------------------------------------------------------- golden pins ----
def _load(name):
    p = GOLD / name
    if not p.exists():
        pytest.skip(f"{p} missing")
    return json.loads(p.read_text())


def _c(a):
    a = np.asarray(a, dtype=np.float64)
    return a[..., 0] + 1j * a[..., 1]


def test_golden_rng():
    g = _load("rng.json")
    for case in g["cases"]:
        got = O.port_rng(case["seed"], case["label"], case["kind"], len(case["values"]), case.get("arg", 0))
        if case["kind"] in (0, 3):
            assert [int(x) for x in got] == [int(x) for x in case["values"]]
        else:
            assert np.array_equal(got, np.array(case["values"], dtype=np.float64))


def test_golden_circuits_port():
    from tests.golden_io import load_circuit_cases

    for case in load_circuit_cases():
        got = O.port_forward(case["n"], case["gates"], init=case.get("init"), data=case.get("data"))
        assert np.max(np.abs(got - case["out"])) <= 1e-14, case["name"]


@pytest.mark.parametrize("k", [1, 5, 37])
def test_qft_closed_form_convention(k):
    """QFT|k> = (1/sqrt N) sum_j exp(+2 pi i j k / N)|j> for the reference's
    qft_circuit (circuit.hpp:167-178) plus the final swaps (the cfg3 circuit):
    pins the closed form test_gpu_fullsize.py checks at 30 qubits."""
    from paper_2512_18995_b200 import workloads as W

    n = 6
    N = 1 << n
    psi = np.zeros(N, complex)
    psi[k] = 1
    gates = W.cfg3_circuit(n).gates()
    got = O.ref_forward(n, gates, init=psi)[0] if O.REF_LIB.exists() else O.port_forward(n, gates, init=psi)[0]
    j = np.arange(N)
    want = np.exp(2j * np.pi * j * k / N) / np.sqrt(N)
    assert np.max(np.abs(got - want)) <= 1e-14


@pytest.mark.skipif(not HAVE_REF, reason="reference headers/library absent")
def test_mixed_state_port_matches_reference():
    """The density-matrix restatement (oracle.port_mixed_run & co.) equals the
    reference's to_mixed / apply_gate / apply_channel / expectation /
    marginals on seeded circuits with every channel kind (test_qubit.cpp:376-420
    exercises the same functions)."""
    from paper_2512_18995_b200.qsv import make_gate

    rng = np.random.default_rng(5)
    n = 3
    ops = [make_gate("h", [0]), make_gate("x", [1], [0]), ("depolarizing", 0, 0.3),
           make_gate("ry", [2], [], [0.7]), ("amplitude_damping", 2, 0.4), make_gate("rzz", [0, 2], [], [0.5]),
           ("bit_flip", 1, 0.2), ("phase_flip", 0, 0.1), ("phase_damping", 1, 0.6),
           make_gate("u3", [1], [2], [0.3, 0.2, 0.1])]
    psi = rng.normal(size=8) + 1j * rng.normal(size=8)
    psi /= np.linalg.norm(psi)
    for init in (None, psi):
        want = O.ref_mixed_run(n, ops, init)
        got = O.port_mixed_run(n, ops, init)
        assert np.max(np.abs(got - want)) <= 1e-14
        for wires, basis in (([0], "z"), ([1, 2], "xy"), ([0, 1, 2], "zzx")):
            e = O.ref_density_expectation(n, want, [(wires, basis)])[0]
            assert abs(O.port_density_expectation(n, want, wires, basis) - e) <= 1e-14
        assert np.allclose(O.port_density_marginal(n, want, [2, 0]), O.ref_density_marginal(n, want, [2, 0]),
                           atol=1e-15, rtol=0)


# ------------------------------------- threaded oracle and digests (pins) ---
def test_threaded_rng_fill_matches_sequential_stream():
    seq = O.port_rng(0, "cfg3", 2, 4096)
    for off in (0, 2, 1000):
        got = O.port_rng_normal(0, "cfg3", 4096 - off, offset=off, nthreads=5)
        assert np.array_equal(got, seq[off:])


def test_threaded_forward_matches_reference_and_single_thread():
    from paper_2512_18995_b200 import workloads as W

    needs_ref()
    n = 12
    rng = Rng(17, "mt-forward")
    for cir in (W.cfg3_circuit(n), W.cfg4_circuit(n, layers=6), W.cfg5_circuit(n, layers=4),
                random_circuit(rng, n, 120)):
        psi = random_state(rng, n)
        want = O.ref_forward(n, cir.gates(), init=psi)[0]
        single = O.port_forward(n, cir.gates(), init=psi)[0]
        got = O.port_forward_mt(n, cir.gates(), psi.copy(), nthreads=7)
        assert np.max(np.abs(got - single)) == 0.0  # same arithmetic, disjoint groups per thread
        assert np.max(np.abs(got - want)) <= 1e-14


def test_digest_of_reference_forward_matches_port_digest():
    """ref_forward_digest (the reference's apply_gate loop + the C++ digest)
    against port_forward_mt + qo_digest, Gaussian input from Rng(0,'cfg3')."""
    from paper_2512_18995_b200 import workloads as W

    needs_ref()
    n = 14
    cir = W.cfg3_circuit(n)
    idx = np.arange(0, 1 << n, 97, dtype=np.uint64)
    blocks, z, samples, _ = O.ref_forward_digest(n, cir.gates(), 1, 0, "cfg3", idx, nblocks=256)
    psi = O.port_rng_normal(0, "cfg3", 2 << n).view(np.complex128)
    psi /= np.sqrt(float(np.dot(psi.view(np.float64), psi.view(np.float64))))
    O.port_forward_mt(n, cir.gates(), psi)
    b2, z2 = O.port_digest(n, psi, nblocks=256, nthreads=3)
    assert np.max(np.abs(samples - psi[idx.astype(np.int64)])) <= 1e-14
    assert np.max(np.abs(blocks - b2)) <= 1e-13
    assert np.max(np.abs(z - z2)) <= 1e-13
    # the digest's Z sums are the reference's expectation_one values
    want = O.ref_expectation(n, psi, [([w], "z") for w in range(n)] + [([0, n - 1], "zz")])
    assert np.max(np.abs(z[1:] - want)) <= 1e-13


@pytest.mark.parametrize("case", ["cfg3_30", "cfg4_26", "cfg5_26"])
def test_fullsize_fixtures_are_reference_made_and_self_consistent(case):
    """The committed full-size fixtures come from the reference (impl "ref");
    when a threaded-port run of the same case was cross-checked, they agree."""
    path = GOLD / "fullsize" / f"{case}.npz"
    if not path.exists():
        pytest.skip(f"{path.name} not generated yet")
    d = np.load(path, allow_pickle=False)
    meta = json.loads(str(d["meta"]))
    assert meta["impl"] == "ref", meta
    assert abs(d["z"][0] - 1.0) <= 1e-12  # norm
    assert abs(d["blocks"][:, 0].sum() - 1.0) <= 1e-12
    if "cross_check" in meta:
        cc = meta["cross_check"]
        assert max(cc["max_abs_sample"], cc["max_abs_z"]) <= 1e-12, cc
