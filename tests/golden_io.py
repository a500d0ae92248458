"""Reads the golden fixtures in tests/golden/ (generated from the reference
library by tests/golden/make_golden.py)."""
import json
from pathlib import Path

import numpy as np

from paper_2512_18995_b200.qsv import make_gate

GOLD = Path(__file__).resolve().parent / "golden"


def _c(a):
    a = np.asarray(a, dtype=np.float64)
    return a[..., 0] + 1j * a[..., 1]


def gate_from_json(d):
    custom = None if d.get("custom") is None else _c(d["custom"])
    return make_gate(d["name"], d["wires"], d.get("controls", []), d.get("params", []), d.get("trainable", False),
                     d.get("encode", False), custom=custom)


def load_circuit_cases():
    doc = json.loads((GOLD / "circuits.json").read_text())
    out = []
    for c in doc["cases"]:
        case = dict(c)
        case["gates"] = [gate_from_json(g) for g in c["gates"]]
        case["out"] = _c(c["out"])
        if c.get("init") is not None:
            case["init"] = _c(c["init"])
        out.append(case)
    return out
