"""Distributed schedules: passes, swap steps and how many swaps fuse into the pass before them (diagnostics)."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import os, sys
from paper_2512_18995_b200 import qsv, workloads as W
from paper_2512_18995_b200.qsv import C64, C128
tot = [0, 0, 0]
for n, cir, dt, world in ((30, W.cfg4_circuit(30), C128, 8), (30, W.cfg4_circuit(30), C128, 2), (32, W.cfg4_circuit(32), C128, 4), (30, W.cfg5_circuit(30), C64, 8), (32, W.cfg5_circuit(32), C64, 4), (28, W.cfg3_circuit(28), C128, 2), (28, W.cfg3_circuit(28), C128, 8)):
    sch = qsv.plan_schedule(n, cir.gates(), dtype=dt, world=world)
    sw = [s for s in sch["steps"] if s["kind"] == "swap"]
    ps = [s for s in sch["steps"] if s["kind"] == "pass"]
    f = sum(1 for s in sw if s["fused"])
    pairs = sum(len(s["pairs"]) for s in sw)
    print(n, world, "passes", len(ps), "swap steps", len(sw), "pairs", pairs, "fused", f)
