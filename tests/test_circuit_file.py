"""Circuit-file ingestion -> GPU -> result file: the
parser's error behaviour (io/circuit_file.hpp:62-205) on CPU, and a full
`run` of a qubit circuit file on the GPU against the reference library
(tools/main.cpp:79-168: state, seeded measurement, expectations, adjoint
gradients)."""
import json

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_18995_b200 import circuit_file as CF
from paper_2512_18995_b200.qsv import InvalidInput

FILE = {
    "version": 1,
    "paradigm": "qubit",
    "nqubit": 4,
    "shots": 2000,
    "ops": [
        {"gate": "h", "wires": [0]},
        {"gate": "cnot", "wires": [0, 1]},
        {"gate": "ry", "wires": [2], "params": [0.7], "trainable": True},
        {"gate": "cry", "wires": [2, 3], "params": [1.1], "trainable": True},
        {"gate": "rz", "wires": [1], "params": [0.3], "encode": True},
        {"gate": "cp", "wires": [3, 0], "params": [0.9]},
        {"gate": "u3", "wires": [3], "params": [0.2, 0.4, 0.6], "trainable": True},
        {"gate": "swap", "wires": [1, 3]},
    ],
    "observables": [{"wires": [0], "basis": "z"}, {"wires": [1, 3], "basis": "zx"}],
    "data": [[0.45]],
    "measure": {"wires": [0, 2, 3]},
}


def test_parse_and_sugar():
    f = CF.parse_circuit_file(FILE)
    assert f.nqubit == 4 and f.shots == 2000 and f.measure_wires == [0, 2, 3]
    g = f.qubit_ops
    assert (g[1].name, g[1].wires, g[1].controls) == ("x", [1], [0])      # cnot: [control, target]
    assert (g[3].name, g[3].wires, g[3].controls) == ("ry", [3], [2])     # cry
    assert (g[5].name, g[5].wires, g[5].controls) == ("p", [0], [3])      # cp
    assert g[4].encode and not g[4].trainable


@pytest.mark.parametrize("bad,msg", [
    ({**FILE, "typo": 1}, "unknown field 'typo' in top level"),
    ({**FILE, "version": 2}, "unsupported version"),
    ({k: v for k, v in FILE.items() if k != "paradigm"}, "missing paradigm"),
    ({**FILE, "paradigm": "analog"}, "unknown paradigm analog"),
    ({**FILE, "ops": [{"gate": "h", "wire": [0]}]}, "unknown field 'wire' in qubit op"),
    ({**FILE, "ops": [{"gate": "cnot", "wires": [0]}]}, "cnot: wires [control, target]"),
    ({**FILE, "observables": [{"wires": [0], "basis": "z", "x": 1}]}, "unknown field 'x' in observable"),
    ({**FILE, "measure": {"wires": [0, 1], "phis": [0.0]}}, "measure wires/phis mismatch"),
    ({**FILE, "nqubit": 0}, "qubit paradigm needs nqubit"),
    ({"paradigm": "fock"}, "photonic paradigms need nmode"),
])
def test_parse_errors_mirror_reference(bad, msg):
    with pytest.raises(InvalidInput, match=msg.replace("[", r"\[").replace("]", r"\]")):
        CF.parse_circuit_file(bad)


def test_load_errors(tmp_path):
    p = tmp_path / "c.json"
    p.write_text("{not json")
    with pytest.raises(InvalidInput, match="JSON parse error"):
        CF.load_circuit_file(str(p))
    with pytest.raises(InvalidInput, match="cannot open"):
        CF.load_circuit_file(str(tmp_path / "missing.json"))


def test_other_paradigms_are_refused_by_run():
    f = CF.parse_circuit_file({"version": 1, "paradigm": "fock", "nmode": 2, "ops": [{"gate": "bs", "wires": [0, 1]}]})
    with pytest.raises(InvalidInput, match="outside this engine"):
        CF.run_qubit(f)


def test_result_file_format():
    r = CF.ResultFile("run:qubit", 7)
    r.add_expectations([0.25, -1e-05])
    r.add_counts({"01": 3, "00": 5})
    text = r.serialize()
    j = json.loads(text)
    assert j["job"] == {"kind": "run:qubit", "seed": 7, "timings_ms": None}
    assert list(j["samples"]) == ["00", "01"]          # sorted keys (std::map / nlohmann object)
    assert text.endswith("\n") and '\n  "expectations": [\n    0.25,\n    -1e-05\n  ]' in text


@pytest.mark.gpu
def test_run_qubit_file_on_gpu_matches_reference(tmp_path):
    from paper_2512_18995_b200 import build

    build.build()
    p = tmp_path / "c.json"
    p.write_text(json.dumps(FILE))
    out = tmp_path / "r.json"
    assert CF.main(["run", str(p), "--seed", "11", "--out", str(out)]) == 0
    res = json.loads(out.read_text())
    f = CF.load_circuit_file(str(p))
    cir = CF.build_qubit_circuit(f)
    gates, obs = cir.gates(), [(o.wires, o.basis) for o in cir.observables()]
    have_ref = O.REF_LIB.exists()
    want = (O.ref_forward if have_ref else O.port_forward)(4, gates, data=f.data)[0]
    got = np.array(res["state"]["re"]) + 1j * np.array(res["state"]["im"])
    assert np.max(np.abs(got - want)) <= 1e-12
    if have_ref:
        assert np.allclose(res["expectations"], O.ref_expectation(4, want, obs), atol=1e-12, rtol=0)
        pg, dg = O.ref_adjoint(4, gates, obs, f.data[0])
        assert np.allclose(res["gradients"]["params"], pg, atol=1e-12, rtol=0)
        assert np.allclose(res["gradients"]["data"], dg, atol=1e-12, rtol=0)
        counts = O.ref_measure(4, want, 2000, [0, 2, 3], 11, "measure")
        for i, c in enumerate(counts):
            key = format(i, "03b")
            assert res["samples"].get(key, 0) == int(c), key
    probs = O.port_marginal(4, want, [0, 2, 3])
    for i, pr in enumerate(probs):
        key = format(i, "03b")
        if pr > 0:
            assert abs(res["probabilities"][key] - pr) <= 1e-12
    assert sum(res["samples"].values()) == 2000
