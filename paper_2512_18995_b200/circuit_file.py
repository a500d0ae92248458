"""Circuit files -> GPU -> result files: the on-disk drop-in for the
reference CLI's `quasar run FILE` on the qubit paradigm.

* `parse_circuit_file` / `load_circuit_file` restate
  io/circuit_file.hpp:87-216: the same top-level and per-op key whitelists
  (unknown fields fail loudly), version 1, the paradigm set, the sugar
  spellings `cnot`/`cx`/`cz`/`cp`/`cry` with the control as the first wire
  (circuit_file.hpp:98-106), observables, data rows and `measure.wires`.
  Only the qubit paradigm runs here (the engine is the qubit state-vector hot
  path); the photonic / MBQC paradigms parse and are then refused with
  `InvalidInput`, naming the paradigm.
* `run_qubit` restates tools/main.cpp:79-168 for the dense backend: forward
  over the file's data rows, seeded measurement with `Rng(seed, "measure")`
  (counts and probabilities), expectations, adjoint gradients when the
  circuit is differentiable and has observables and at most one data row,
  and the state when n <= 16 with at most one row.
* `ResultFile` restates io/result_file.hpp:29-93: sorted keys, shortest
  round-trip doubles, two-space indentation, `timings_ms` null unless
  requested.

The JSON parsing is Python's (the reference uses nlohmann json 3.11.3, which
is not vendored in the reference tree).
"""
from __future__ import annotations

import json
import time
from dataclasses import dataclass, field

from . import qsv
from .qsv import C128, Circuit, InvalidInput, Rng, make_gate

_TOP_KEYS = {"version", "paradigm", "nqubit", "nmode", "cutoff", "chi", "nstep", "shots", "hbar", "backend",
             "detector", "init_state", "ops", "observables", "data", "measure", "pattern", "inputs", "squeezing",
             "unitary", "adjacency", "mean_photon", "select"}
_PARADIGMS = {"qubit", "fock", "gaussian", "bosonic", "tdm", "mbqc-pattern"}
_QUBIT_OP_KEYS = {"gate", "wires", "controls", "params", "encode", "trainable"}
_PHOTONIC_OP_KEYS = {"gate", "wires", "params", "encode", "ntau"}


def _require(cond: bool, msg: str):
    if not cond:
        raise InvalidInput(msg)


def _check_keys(obj: dict, allowed: set, where: str):
    for k in obj:
        if k not in allowed:
            raise InvalidInput(f"circuit file: unknown field '{k}' in {where}")


@dataclass
class CircuitFile:
    """io/circuit_file.hpp:32-56 (the fields the qubit path reads)."""
    version: int = 1
    paradigm: str = ""
    nqubit: int = 0
    nmode: int = 0
    shots: int = 0
    backend: str = ""
    qubit_ops: list = field(default_factory=list)
    observables: list = field(default_factory=list)  # (wires, basis)
    data: list = field(default_factory=list)
    measure_wires: list = field(default_factory=list)
    raw: dict = field(default_factory=dict)


def _parse_qubit_gate(op: dict):
    """circuit_file.hpp:87-107."""
    _check_keys(op, _QUBIT_OP_KEYS, "qubit op")
    if "gate" not in op or "wires" not in op:
        raise InvalidInput("circuit file: qubit op needs 'gate' and 'wires'")
    name = str(op["gate"])
    wires = [int(w) for w in op["wires"]]
    controls = [int(c) for c in op.get("controls", [])]
    params = [float(p) for p in op.get("params", [])]
    encode = bool(op.get("encode", False))
    trainable = bool(op.get("trainable", False))
    if name in ("cnot", "cx"):
        _require(len(wires) == 2, "cnot: wires [control, target]")
        return make_gate("x", [wires[1]], [wires[0]])
    if name in ("cz", "cp", "cry"):
        _require(len(wires) == 2, f"{name}: wires [control, target]")
        base = {"cz": "z", "cp": "p", "cry": "ry"}[name]
        return make_gate(base, [wires[1]], [wires[0]], params, trainable, encode)
    return make_gate(name, wires, controls, params, trainable, encode)


def parse_circuit_file(j: dict) -> CircuitFile:
    """circuit_file.hpp:130-205."""
    _require(isinstance(j, dict), "circuit file: top level must be an object")
    _check_keys(j, _TOP_KEYS, "top level")
    f = CircuitFile(raw=j)
    f.version = int(j.get("version", 1))
    _require(f.version == 1, "circuit file: unsupported version")
    _require("paradigm" in j, "circuit file: missing paradigm")
    f.paradigm = str(j["paradigm"])
    _require(f.paradigm in _PARADIGMS, "circuit file: unknown paradigm " + f.paradigm)
    f.nqubit = int(j.get("nqubit", 0))
    f.nmode = int(j.get("nmode", 0))
    f.shots = int(j.get("shots", 0))
    f.backend = str(j.get("backend", ""))
    for op in j.get("ops", []):
        if f.paradigm == "qubit":
            f.qubit_ops.append(_parse_qubit_gate(op))
        else:
            _check_keys(op, _PHOTONIC_OP_KEYS, "photonic op")
    for o in j.get("observables", []):
        _check_keys(o, {"wires", "basis"}, "observable")
        f.observables.append(([int(w) for w in o["wires"]], str(o["basis"])))
    if "data" in j:
        f.data = [[float(x) for x in row] for row in j["data"]]
    if "measure" in j:
        _check_keys(j["measure"], {"wires", "phis"}, "measure")
        f.measure_wires = [int(w) for w in j["measure"]["wires"]]
        phis = j["measure"].get("phis", [0.0] * len(f.measure_wires))
        _require(len(phis) == len(f.measure_wires), "circuit file: measure wires/phis mismatch")
    if f.paradigm == "qubit":
        _require(f.nqubit >= 1, "circuit file: qubit paradigm needs nqubit")
    elif f.paradigm != "mbqc-pattern":
        _require(f.nmode >= 1 or "adjacency" in j, "circuit file: photonic paradigms need nmode (or an adjacency)")
    return f


def load_circuit_file(path: str) -> CircuitFile:
    """circuit_file.hpp:207-216."""
    try:
        with open(path) as fh:
            j = json.load(fh)
    except OSError:
        raise InvalidInput("circuit file: cannot open " + str(path)) from None
    except json.JSONDecodeError as e:
        raise InvalidInput(f"circuit file: JSON parse error: {e}") from None
    return parse_circuit_file(j)


class ResultFile:
    """io/result_file.hpp:29-93."""

    def __init__(self, kind: str, seed: int):
        self.root = {"version": 1, "job": {"kind": kind, "seed": int(seed), "timings_ms": None}}

    def set_timing(self, label: str, ms: float):
        if self.root["job"]["timings_ms"] is None:
            self.root["job"]["timings_ms"] = {}
        self.root["job"]["timings_ms"][label] = float(ms)

    def add_counts(self, counts: dict):
        self.root.setdefault("samples", {}).update({k: int(v) for k, v in counts.items()})

    def add_probabilities(self, probs: dict):
        self.root.setdefault("probabilities", {}).update({k: float(v) for k, v in probs.items()})

    def add_expectations(self, values):
        self.root["expectations"] = [float(v) for v in values]

    def add_gradients(self, params, data):
        self.root["gradients"] = {"params": [float(x) for x in params], "data": [float(x) for x in data]}

    def add_state(self, amps):
        self.root["state"] = {"re": [float(a.real) for a in amps], "im": [float(a.imag) for a in amps]}

    def add_diagnostic(self, key: str, value):
        self.root.setdefault("diagnostics", {})[key] = value

    def serialize(self) -> str:
        return json.dumps(self.root, sort_keys=True, indent=2) + "\n"

    def write(self, path: str):
        try:
            with open(path, "w") as fh:
                fh.write(self.serialize())
        except OSError:
            raise InvalidInput("result file: cannot open " + str(path) + " for writing") from None


def build_qubit_circuit(f: CircuitFile) -> Circuit:
    """tools/main.cpp:66-71."""
    cir = Circuit(f.nqubit)
    for g in f.qubit_ops:
        cir.add(g)
    for wires, basis in f.observables:
        cir.observable(wires, basis)
    return cir


def rank_devices(ranks: int) -> list:
    """GPU of each rank: round-robin over the visible devices (ranks beyond
    the device count share GPUs, which only an NCCL that allows it -- the test
    shim -- accepts)."""
    nd = max(1, qsv.lib().qsv_device_count())
    return [r % nd for r in range(ranks)]


def run_qubit(f: CircuitFile, seed: int = 0, shots: int = -1, ranks: int = 1, timings: bool = False,
              dtype: int = C128) -> ResultFile:
    """tools/main.cpp:79-168, dense backend, on the GPU. ranks > 1 runs the
    distributed branch (tools/main.cpp:86-131): one process driving `ranks`
    GPUs (qsv_ctx_create_multi, the in-process dist::run_on_ranks), the state
    sharded with the top log2(ranks) wires global, measurement, expectations
    and adjoint gradients all-reduced, the state gathered up to 20 qubits."""
    if f.paradigm != "qubit":
        raise InvalidInput(f"paradigm '{f.paradigm}' is outside this engine (qubit state-vector path only)")
    _require(f.backend in ("", "dense"), f"backend '{f.backend}' is outside this engine (dense state vector only)")
    result = ResultFile("run:qubit", seed)
    cir = build_qubit_circuit(f)
    nshots = shots if shots >= 0 else f.shots
    wires = f.measure_wires or list(range(f.nqubit))
    differentiable = cir.encode_slots() > 0 or any(g.trainable and g.params for g in cir.gates())
    ctx = None
    if ranks > 1:
        _require(f.backend in ("", "dense"), "distributed runs use the dense backend")
        _require(len(f.data) <= 1, "distributed runs take at most one data row")
        ctx = qsv.Context.multi(rank_devices(ranks))
    t0 = time.perf_counter()
    state = cir.forward(data=f.data if f.data else None, dtype=dtype, ctx=ctx)
    if timings:
        result.set_timing("forward", (time.perf_counter() - t0) * 1e3)
    if nshots > 0:
        counts = qsv.measure(state, nshots, wires, Rng(seed, "measure"), True)
        result.add_counts({k: v["count"] for k, v in counts.items() if v["count"]})
        result.add_probabilities({k: v["probability"] for k, v in counts.items()})
    if cir.observables():
        result.add_expectations(qsv.expectation(state, cir))
    if differentiable and cir.observables() and len(f.data) <= 1:
        g = qsv.adjoint_gradients(cir, None, f.data[0] if f.data else (), dtype=dtype, ctx=ctx)
        result.add_gradients(g.param_grads, g.data_grads)
    if f.nqubit <= (20 if ranks > 1 else 16) and len(f.data) <= 1:
        result.add_state(state.amplitudes(0))
    if ranks > 1:
        result.root["job"]["ranks"] = int(ranks)
        del state
        ctx.close()
    return result


def main(argv=None) -> int:
    """`python -m paper_2512_18995_b200 run FILE [--seed S] [--shots N]
    [--ranks R] [--out PATH] [--timings]`; exit codes as tools/main.cpp:686-697
    (2 invalid input, 3 numerical guard, 4 transport, 1 other)."""
    import argparse
    import sys

    ap = argparse.ArgumentParser(prog="qsv")
    sub = ap.add_subparsers(dest="cmd", required=True)
    r = sub.add_parser("run", help="execute a qubit circuit file on the GPU")
    r.add_argument("file")
    r.add_argument("--seed", type=int, default=0)
    r.add_argument("--shots", type=int, default=-1)
    r.add_argument("--ranks", type=int, default=1)
    r.add_argument("--out", default="")
    r.add_argument("--timings", action="store_true")
    a = ap.parse_args(argv)
    try:
        res = run_qubit(load_circuit_file(a.file), seed=a.seed, shots=a.shots, ranks=a.ranks, timings=a.timings)
        if a.out:
            res.write(a.out)
        else:
            sys.stdout.write(res.serialize())
        return 0
    except InvalidInput as e:
        sys.stderr.write(f"error: {e}\n")
        return 2
    except qsv.GuardError as e:
        sys.stderr.write(f"error: {e}\n")
        return 3
    except qsv.TransportError as e:
        sys.stderr.write(f"error: {e}\n")
        return 4
    except qsv.QsvError as e:
        sys.stderr.write(f"error: {e}\n")
        return 1
