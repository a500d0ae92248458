"""Lazy layouts (qsv_opts.lazy_layout): swap gates stay qubit relabelings past
the end of an execute, the state carries its wire -> bit map, and the next
execute plans from that layout. Every observable must match the eager plan
(which restores the canonical layout inside its last pass) and the reference
path the eager plan is pinned to (tests/test_gpu_parity.py,
tests/test_gpu_fullsize.py): max |d| <= 1e-12 in complex128.
"""
import math

import numpy as np
import pytest

from paper_2512_18995_b200 import qsv
from paper_2512_18995_b200 import workloads as W
from paper_2512_18995_b200.qsv import C64, C128, Observable, QubitState, Rng, make_gate
from tests.helpers import random_circuit

pytestmark = pytest.mark.gpu
TOL = {C128: 1e-12, C64: 1e-5}


@pytest.fixture(scope="module", autouse=True)
def ctx(built):
    return qsv.default_context()


def rand_amps(n, seed):
    r = np.random.default_rng(seed)
    a = r.standard_normal(1 << n) + 1j * r.standard_normal(1 << n)
    return a / np.linalg.norm(a)


def pair(n, gates, dtype, opts):
    pe = qsv.Plan(n, gates, dtype=dtype)
    pl = qsv.Plan(n, gates, dtype=dtype, opts=opts)
    return pe, pl


@pytest.mark.parametrize("n", [6, 11, 12, 15, 18, 21])
@pytest.mark.parametrize("opts", [{"lazy_layout": 1}, {"lazy_layout": 1, "tile_bits": 12}])
@pytest.mark.parametrize("reps", [1, 2, 3, 4])
def test_qft_back_to_back(n, opts, reps):
    """cfg3's QFT + swaps run reps times on the same state (the lazy plan
    alternates between the canonical and the bit-reversed layout)."""
    gates = W.cfg3_circuit(n).gates()
    pe, pl = pair(n, gates, C128, opts)
    a = rand_amps(n, 100 + n)
    se, sl = QubitState(n, dtype=C128), QubitState(n, dtype=C128)
    se.upload(a)
    sl.upload(a)
    for _ in range(reps):
        pe.execute(se)
        pl.execute(sl)
    err = float(np.abs(se.amplitudes() - sl.amplitudes()).max())
    assert err <= TOL[C128], err


@pytest.mark.parametrize("dtype", [C128, C64])
@pytest.mark.parametrize("seed", range(6))
def test_random_circuits_with_swaps(dtype, seed):
    """Random circuits (swaps included) executed twice, then every observable
    the state offers: amplitudes, <Z_w>, Pauli strings, marginals, seeded
    measurement, a clone and a one-gate apply on the lazily laid-out state."""
    n = 13 + seed % 4
    rng = Rng(seed, "lazy")
    cir = random_circuit(rng, n, 160)
    for i in range(n // 2):  # and a layout-reversing tail
        cir.swap(i, n - 1 - i)
    gates = cir.gates()
    pe, pl = pair(n, gates, dtype, {"lazy_layout": 1, "jit": 1})
    a = rand_amps(n, seed)
    se, sl = QubitState(n, dtype=dtype), QubitState(n, dtype=dtype)
    se.upload(a)
    sl.upload(a)
    for _ in range(2):
        pe.execute(se)
        pl.execute(sl)
    tol = TOL[dtype]
    # observables that read the permuted layout in place (no restore)
    assert np.abs(se.expect_z_all() - sl.expect_z_all()).max() <= 10 * tol
    obs = [Observable([0, n - 1], "xz"), Observable([1, 2, n - 2], "yxy"), Observable([3], "z")]
    ve = qsv.expectation_many(se, obs)
    vl = qsv.expectation_many(sl, obs)
    assert np.abs(np.asarray(ve) - np.asarray(vl)).max() <= 10 * tol
    wires = [n - 1, 0, 2]
    assert np.abs(qsv.marginal_probabilities(se, wires) - qsv.marginal_probabilities(sl, wires)).max() <= 10 * tol
    if dtype == C128:
        ce = qsv.measure_counts(se, 2000, wires, Rng(7, "m"))
        cl = qsv.measure_counts(sl, 2000, wires, Rng(7, "m"))
        assert np.array_equal(ce[0], cl[0])
    # clone keeps the layout; a one-gate apply works on it
    g = make_gate("ry", [1], params=[0.37])
    oe = qsv.apply_gate(se, g)
    ol = qsv.apply_gate(sl.clone(), g)
    assert np.abs(oe.amplitudes() - ol.amplitudes()).max() <= tol
    # and the amplitudes themselves (the download restores the layout)
    assert np.abs(se.amplitudes() - sl.amplitudes()).max() <= tol
    # after the restore the lazy plan runs again from the canonical layout
    pe.execute(se)
    pl.execute(sl)
    assert np.abs(se.amplitudes() - sl.amplitudes()).max() <= tol


def test_batched_rows_and_row_upload():
    """A batch of rows shares one layout: a one-row upload into a lazily laid
    out batch restores the other rows first."""
    n, B = 12, 3
    gates = W.cfg3_circuit(n).gates()
    pe, pl = pair(n, gates, C128, {"lazy_layout": 1})
    se, sl = QubitState(n, batch=B, dtype=C128), QubitState(n, batch=B, dtype=C128)
    for b in range(B):
        se.upload(rand_amps(n, b), b)
        sl.upload(rand_amps(n, b), b)
    pe.execute(se)
    pl.execute(sl)
    se.upload(rand_amps(n, 9), 1)
    sl.upload(rand_amps(n, 9), 1)
    pe.execute(se)
    pl.execute(sl)
    for b in range(B):
        assert np.abs(se.amplitudes(b) - sl.amplitudes(b)).max() <= TOL[C128]


def test_expect_z_fused_and_profile():
    """execute_expect_z (fused <Z> epilogue when the last pass holds a row) and
    profile (the bench's per-launch timing) on alternating layouts."""
    n = 12
    gates = W.cfg3_circuit(n).gates()
    pe, pl = pair(n, gates, C128, {"lazy_layout": 1})
    a = rand_amps(n, 3)
    se, sl = QubitState(n, dtype=C128), QubitState(n, dtype=C128)
    se.upload(a)
    sl.upload(a)
    for _ in range(3):
        ze = pe.execute_expect_z(se)
        zl = pl.execute_expect_z(sl)
        assert np.abs(ze - zl).max() <= 1e-12
    n = 16
    gates = W.cfg3_circuit(n).gates()
    pe, pl = pair(n, gates, C128, {"lazy_layout": 1, "tile_bits": 12})
    a = rand_amps(n, 4)
    se, sl = QubitState(n, dtype=C128), QubitState(n, dtype=C128)
    se.upload(a)
    sl.upload(a)
    for _ in range(3):
        pe.execute(se)
        ms = pl.profile(sl)
        assert len(ms) == len(pl.step_kinds()) and np.all(ms > 0)
    assert np.abs(se.amplitudes() - sl.amplitudes()).max() <= TOL[C128]


def test_set_basis_and_run_circuit():
    """set_basis overwrites every row (any layout becomes canonical); the
    Circuit.forward path (qsv_run_circuit plan cache) with lazy layouts."""
    n = 14
    cir = W.cfg3_circuit(n)
    pl = qsv.Plan(n, cir.gates(), dtype=C128, opts={"lazy_layout": 1})
    st = QubitState(n, dtype=C128)
    st.upload(rand_amps(n, 5))
    pl.execute(st)
    qsv.check(qsv.lib().qsv_state_set_basis(st.h, 5))
    pl.execute(st)
    # QFT|5> with the swaps: amplitude x = e^{2 pi i 5 x / 2^n} / sqrt(2^n)
    x = np.arange(1 << n)
    want = np.exp(2j * math.pi * 5 * x / (1 << n)) / math.sqrt(1 << n)
    assert np.abs(st.amplitudes() - want).max() <= 1e-12
    init = QubitState(n, dtype=C128)
    init.upload(rand_amps(n, 6))
    out_e = cir.forward(init)
    out_l = cir.forward(init, opts={"lazy_layout": 1})
    out_l2 = cir.forward(out_l, opts={"lazy_layout": 1})
    out_e2 = cir.forward(out_e)
    assert np.abs(out_e.amplitudes() - out_l.amplitudes()).max() <= 1e-12
    assert np.abs(out_e2.amplitudes() - out_l2.amplitudes()).max() <= 1e-12
