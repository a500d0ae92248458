"""Generates the full-size parity fixtures tests/golden/fullsize/<case>.npz.

TEST INFRASTRUCTURE. Run here (the container with /root/reference):

    python tests/golden/make_fullsize.py cfg3_30 [--impl ref|port]

Each case is a BASELINE.json config family at a size the reference's CPU path
can run (<= 30 qubits, state.hpp:35), with the same seeded generators as the
bench and the tests (paper_2512_18995_b200/workloads.py):

    cfg3_30   30-qubit QFT + 15 final swaps (480 gates) on the seeded
              normalised Gaussian state Rng(0, "cfg3") -- the bench's own
              workload, complex128
    cfg4_26   cfg4 family at 26 qubits, full depth (20 layers of U3 +
              brickwork CNOT, 770 gates) from |0...0>
    cfg5_26   cfg5 family at 26 qubits, full depth (16 layers of rx/ry/rz +
              random-pair CZ, 1456 gates) from |0...0>

--impl ref (default) runs the reference itself: oracle/_ref's
ref_forward_digest, i.e. quasar::qubit::apply_gate gate by gate (the loop of
Circuit::forward, circuit.hpp:124-128) on the unmodified reference headers;
the 30-qubit case takes ~1.5 h on one core and 32 GiB. --impl port runs the
threaded C restatement (oracle/qsv_oracle.c qo_forward_mt, pinned against
oracle/_ref in tests/test_oracle.py) in minutes; when a fixture from the other
implementation exists, the two are compared and the agreement recorded.

A fixture holds no full state (16 GiB at 30 qubits): the digest of
oracle/qsv_oracle.c qo_digest (4096 block sums of |a|^2 and of a_i w_i with
pseudo-random +-1+-i weights, <Z_w> for every wire, <Z_0 Z_{n-1}>, the norm)
and the amplitudes at seeded random indices.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))

from oracle import oracle as O  # noqa: E402
from paper_2512_18995_b200 import workloads as W  # noqa: E402

OUT = Path(__file__).resolve().parent / "fullsize"
NBLOCKS = 4096


def case(name):
    if name == "cfg3_30":
        return 30, W.cfg3_circuit(30).gates(), 1, "cfg3", 65536
    if name == "cfg4_26":
        return 26, W.cfg4_circuit(26, layers=20).gates(), 0, None, 16384
    if name == "cfg5_26":
        return 26, W.cfg5_circuit(26, layers=16).gates(), 0, None, 16384
    raise SystemExit(f"unknown case {name}")


def sample_indices(n, k):
    rng = np.random.default_rng(20261020 + n)
    idx = rng.choice(1 << n, size=k - 2, replace=False)
    return np.unique(np.concatenate([idx, [0, (1 << n) - 1]])).astype(np.uint64)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("case")
    ap.add_argument("--impl", default="ref", choices=["ref", "port"])
    args = ap.parse_args()
    n, gates, init_kind, label, nsamp = case(args.case)
    idx = sample_indices(n, nsamp)
    t0 = time.time()
    if args.impl == "ref":
        blocks, z, samples, sec = O.ref_forward_digest(n, gates, init_kind, 0, label, idx, NBLOCKS)
        src = "oracle/_ref ref_forward_digest: quasar::qubit::apply_gate per gate (unmodified reference headers)"
    else:
        if init_kind == 1:
            psi = O.port_rng_normal(0, label, 2 << n).view(np.complex128)
            psi /= np.sqrt(float(np.dot(psi.view(np.float64), psi.view(np.float64))))
        else:
            psi = np.zeros(1 << n, dtype=np.complex128)
            psi[0] = 1.0
        ts = time.time()
        O.port_forward_mt(n, gates, psi)
        sec = time.time() - ts
        blocks, z = O.port_digest(n, psi, NBLOCKS)
        samples = psi[idx.astype(np.int64)].copy()
        del psi
        src = "oracle/_build qo_forward_mt: threaded C restatement of apply_matrix_strided"
    meta = {"case": args.case, "n": n, "gates": len(gates), "init": "gaussian Rng(0,'cfg3')" if init_kind else "|0>",
            "impl": args.impl, "source": src, "forward_seconds": sec, "wall_seconds": time.time() - t0,
            "nblocks": NBLOCKS, "nsamples": int(len(idx))}
    OUT.mkdir(exist_ok=True)
    path = OUT / f"{args.case}.npz"
    other = OUT / f"{args.case}.{'port' if args.impl == 'ref' else 'ref'}.npz"
    if path.exists():
        prev = np.load(path, allow_pickle=False)
        pm = json.loads(str(prev["meta"]))
        if pm["impl"] != args.impl:
            # keep the other implementation's fixture for the cross-check
            np.savez(other, **{k: prev[k] for k in prev.files})
    if other.exists():
        o = np.load(other, allow_pickle=False)
        meta["cross_check"] = {
            "against": json.loads(str(o["meta"]))["impl"],
            "max_abs_sample": float(np.max(np.abs(o["samples"] - samples))),
            "max_abs_block": float(np.max(np.abs(o["blocks"] - blocks))),
            "max_abs_z": float(np.max(np.abs(o["z"] - z))),
        }
    # the reference's fixture is the one the tests read; a port run only
    # writes the main file when no reference fixture exists yet
    if args.impl == "port" and path.exists() and json.loads(str(np.load(path)["meta"]))["impl"] == "ref":
        path = other
    np.savez(path, idx=idx, samples=samples, blocks=blocks, z=z, meta=json.dumps(meta))
    print(json.dumps(meta))


if __name__ == "__main__":
    main()
