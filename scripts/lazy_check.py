"""Lazy layouts (opts.lazy_layout): parity against the eager plan and per-pass
timing of the cfg3 QFT in both layouts it alternates between."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np

from paper_2512_18995_b200 import qsv, workloads as W


def rand_state(n, seed):
    r = np.random.default_rng(seed)
    a = r.standard_normal(1 << n) + 1j * r.standard_normal(1 << n)
    return a / np.linalg.norm(a)


def parity(n, opts):
    cir = W.cfg3_circuit(n)
    a = rand_state(n, n)
    pe = qsv.Plan(n, cir.gates(), dtype=qsv.C128)
    pl = qsv.Plan(n, cir.gates(), dtype=qsv.C128, opts=opts)
    se = qsv.QubitState(n, dtype=qsv.C128)
    sl = qsv.QubitState(n, dtype=qsv.C128)
    worst = 0.0
    for k in (1, 2, 3):  # k executions back to back: the lazy plan alternates layouts
        se.upload(a)
        sl.upload(a)
        for _ in range(k):
            pe.execute(se)
            pl.execute(sl)
        worst = max(worst, float(np.abs(se.amplitudes() - sl.amplitudes()).max()))
    print(f"parity n={n} opts={opts} passes={pl.info['npasses']} max|d|={worst:.2e}", flush=True)


def timing(n, opts, reps=4):
    cir = W.cfg3_circuit(n)
    p = qsv.Plan(n, cir.gates(), dtype=qsv.C128, opts=opts)
    st = qsv.QubitState(n, dtype=qsv.C128)
    st.upload(rand_state(n, 1) if n <= 26 else W.cfg3_slice(0, 1 << n) / np.sqrt(float(1 << n)))
    rows = []
    for _ in range(reps):
        rows.append(p.profile(st))
    rows = np.array(rows)[:, : p.info["npasses"]]
    tot = rows.sum(axis=1)
    gb = 2.0 * 16 * (1 << n) / 1e9
    print(f"time n={n} opts={opts} passes={p.info['npasses']} step ms={np.round(tot, 3).tolist()} "
          f"median={np.median(tot):.3f} per-pass={np.round(rows.mean(axis=0), 3).tolist()} "
          f"GB/s/pass={gb / (rows.mean() / 1e3):.0f} gates/s={p.info['ngates'] / (np.median(tot) / 1e3):.0f}",
          flush=True)


if __name__ == "__main__":
    for n in (8, 12, 17, 20, 23):
        for o in ({"lazy_layout": 1}, {"lazy_layout": 1, "tile_bits": 12}):
            parity(n, o)
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
    for o in (None, {"lazy_layout": 1, "tile_bits": 12}, {"tile_bits": 12}, {"lazy_layout": 1},
              {"lazy_layout": 1, "tile_bits": 12, "low_bits": 2}):
        timing(n, o)
