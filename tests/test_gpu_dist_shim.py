"""The engine's REAL multi-rank path (dist.cu qubit swaps, all-reduced
reductions, the distributed schedule, bench.py's N > 1 code) on ONE GPU.

Every rank is a separate process with its own qsv context on device 0;
NCCL is replaced by tests/fake_nccl (QSV_NCCL_LIB), a host-driven stand-in:
at each group end the ranks synchronise their streams, exchange CUDA IPC
handles through POSIX shared memory and copy with cudaMemcpy -- no kernel
ever waits on another process (B200_PROFILING.md: ranks whose kernels wait on
one another must not share a GPU). What runs on the device is exactly the
production code: pass kernels with rank bits, gather/scatter of the swapped
half-slices, FP64 partial sums. Results are gathered and compared with the
single-rank reference, as the reference's own dist tests do
(tests/test_dist.cpp:59-62, 128-205).
"""
import multiprocessing as mp
import os
import subprocess
import sys
import traceback
from pathlib import Path

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_18995_b200 import qsv
from paper_2512_18995_b200 import workloads as W
from tests.helpers import random_circuit, random_state

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
SHIM = ROOT / "tests" / "fake_nccl" / "_build" / "libnccl_fake.so"


@pytest.fixture(scope="module", autouse=True)
def _shim():
    if qsv.lib().qsv_device_count() < 1:
        pytest.fail("no CUDA device: the -m gpu suite needs a B200")
    if not SHIM.exists():
        subprocess.run(["make", "-C", str(SHIM.parent.parent)], check=True, capture_output=True)
    from paper_2512_18995_b200 import build

    build.build()
    os.environ["QSV_NCCL_LIB"] = str(SHIM)
    yield


def _rank_main(rank, world, uid, n, gates, init, dtype, obs, q, env=None, data=None):
    try:
        os.environ["QSV_NCCL_LIB"] = str(SHIM)
        os.environ.update(env or {})
        from paper_2512_18995_b200 import qsv as Q

        ctx = Q.Context(0, rank, world, uid)
        g = int(np.log2(world))
        nl = n - g
        st = Q.QubitState(n, dtype=dtype, ctx=ctx)
        if init is not None:
            st.upload(init[rank << nl:(rank + 1) << nl])
        plan = Q.Plan(n, gates, dtype=dtype, ctx=ctx)
        plan.execute(st, data)
        local = st.amplitudes()
        z = st.expect_z_all()[0]
        nrm = float(st.norm2()[0])
        ex = Q.expectation_many(st, [Q.Observable(w, b) for w, b in obs])[0] if obs else []
        local = st.amplitudes()  # again: expectations must leave the layout as they found it
        counts = Q.measure(st, 1000, [0, n - 1], Q.Rng(3, "shim-measure"), True)  # measure_dist
        q.put((rank, local, z, nrm, list(ex) + [counts], plan.info["nswaps"], st.peer_memory()))
        del plan, st
        ctx.close()
    except Exception:
        q.put((rank, traceback.format_exc(), None, None, None, None, None))


PEER_MEMORY = {}  # rank -> QubitState.peer_memory() of the last run_ranks


def run_ranks(n, gates, world, init=None, dtype=qsv.C128, obs=(), env=None, data=None):
    PEER_MEMORY.clear()
    uid = qsv.Context.nccl_unique_id()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    procs = [ctxm.Process(target=_rank_main, args=(r, world, uid, n, gates, init, dtype, list(obs), q, env, data))
             for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, local, z, nrm, ex, nsw, p2p = q.get(timeout=180)
            if z is None:
                raise AssertionError(f"rank {r} failed:\n{local}")
            res[r] = (local, z, nrm, ex, nsw)
            PEER_MEMORY[r] = p2p
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    full = np.concatenate([res[r][0] for r in range(world)])
    return full, res[0][1], res[0][2], res[0][3], res[0][4]


@pytest.mark.parametrize("world", [2, 4])
def test_random_circuits_match_single_rank(world):  # test_dist.cpp:128-145
    rng = qsv.Rng(7, f"shim-{world}")
    n = 10
    for trial in range(2):
        cir = random_circuit(rng, n, 60)
        psi = random_state(rng, n)
        got, z, nrm, _, nsw = run_ranks(n, cir.gates(), world, init=psi)
        want = O.port_forward(n, cir.gates(), init=psi)[0]
        assert np.max(np.abs(got - want)) <= 1e-12, (world, trial)
        zw = [O.port_expectation(n, want, [w], "z")[0] for w in range(n)]
        assert np.max(np.abs(z - zw)) <= 1e-12
        assert abs(nrm - 1.0) <= 1e-12


def test_cfg4_family_swaps_4_ranks():
    """Non-diagonal gates on global wires force qubit swaps (dist_swap_bits)."""
    n = 14
    cir = W.cfg4_circuit(n, layers=4)
    got, z, nrm, _, nsw = run_ranks(n, cir.gates(), 4)
    want = O.port_forward(n, cir.gates())[0]
    assert nsw > 0
    assert np.max(np.abs(got - want)) <= 1e-12
    assert abs(nrm - 1.0) <= 1e-12


def test_cfg5_family_c64_and_global_pauli_2_ranks():
    n = 12
    cir = W.cfg5_circuit(n, layers=3)
    obs = [([0, n - 1], "zz"), ([n - 1], "x"), ([2, n - 2], "yz")]  # wire 0 is a rank bit
    got, z, nrm, ex, nsw = run_ranks(n, cir.gates(), 2, dtype=qsv.C64, obs=obs)
    want = O.port_forward(n, cir.gates())[0]
    assert np.max(np.abs(got - want)) <= 1e-5
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-6  # complex64 relative L2
    for (w, b), e in zip(obs, ex):
        assert abs(e - O.port_expectation(n, want, w, b)[0]) <= 1e-5


def test_qft_2_ranks_bench_path():
    n = 16
    cir = W.cfg3_circuit(n)
    psi = W.cfg3_input(n)
    got, _, nrm, _, _ = run_ranks(n, cir.gates(), 2, init=psi)
    want = O.port_forward(n, cir.gates(), init=psi)[0]
    assert np.max(np.abs(got - want)) <= 1e-12
    assert abs(nrm - 1.0) <= 1e-12


def test_cfg4_family_8_ranks_multi_bit_all_to_all():
    """8 ranks: swap steps carry up to 3 bit pairs -> one in-place all-to-all
    over 7 peers (dist.cu block exchange)."""
    n = 14
    cir = W.cfg4_circuit(n, layers=3)
    sched = qsv.plan_schedule(n, cir.gates(), world=8)
    assert max(len(s["pairs"]) for s in sched["steps"] if s["kind"] == "swap") >= 2
    got, z, nrm, _, nsw = run_ranks(n, cir.gates(), 8)
    want = O.port_forward(n, cir.gates())[0]
    assert np.max(np.abs(got - want)) <= 1e-12
    assert abs(nrm - 1.0) <= 1e-12


def test_pipelined_swap_rounds_4_ranks():
    """A 1 KiB staging set forces many chunk rounds per swap: gather(k + 1)
    overlaps transfer(k) on the two streams, scatter(k) waits for it."""
    n = 14
    cir = W.cfg4_circuit(n, layers=2)
    got, z, nrm, _, nsw = run_ranks(n, cir.gates(), 4, env={"QSV_SWAP_STAGE_BYTES": "1024"})
    want = O.port_forward(n, cir.gates())[0]
    assert nsw > 0
    assert np.max(np.abs(got - want)) <= 1e-12


def test_reference_dist_expectation_case_and_global_xy():
    """tests/test_dist.cpp:189-204: 4 qubits on 4 ranks, encoded Ry layer +
    cnot ring, <Z_0> and <X_1> -- X on a RANK wire (localised by a swap and
    swapped back); plus Y/X on rank wires of a larger cfg5-family state."""
    cir = qsv.Circuit(4)
    cir.rylayer(encode=True)
    cir.cnot_ring()
    data = [[0.0, 1.0, 2.0, 3.0]]
    full = O.port_forward(4, cir.gates(), data=data)[0]
    got, z, nrm, ex, _ = run_ranks(4, cir.gates(), 4, obs=[([0], "z"), ([1], "x")], data=data)
    assert np.max(np.abs(got - full)) <= 1e-12
    assert abs(ex[0] - O.port_expectation(4, full, [0], "z")[0]) <= 1e-12
    assert abs(ex[1] - O.port_expectation(4, full, [1], "x")[0]) <= 1e-12
    n = 10
    c5 = W.cfg5_circuit(n, layers=2)
    obs = [([0], "x"), ([1, 0], "yz"), ([0, 1, 5], "xyz"), ([1], "y")]
    got, z, nrm, ex, _ = run_ranks(n, c5.gates(), 4, obs=obs)
    want = O.port_forward(n, c5.gates())[0]
    assert np.max(np.abs(got - want)) <= 1e-12  # the layout was restored
    for (w, b), e in zip(obs, ex):
        assert abs(e - O.port_expectation(n, want, w, b)[0]) <= 1e-12


def test_measure_dist_equals_single_rank_histogram():  # tests/test_dist.cpp:176-187
    n = 10
    cir = W.cfg4_circuit(n, layers=2)
    got, z, nrm, ex, _ = run_ranks(n, cir.gates(), 4)
    counts = ex[-1]
    want = O.port_forward(n, cir.gates())[0]
    if O.REF_LIB.exists():
        ref = O.ref_measure(n, want, 1000, [0, n - 1], 3, "shim-measure")
        for i, c in enumerate(ref):
            key = format(i, "02b")
            assert counts.get(key, {"count": 0})["count"] == int(c), key
    probs = O.port_marginal(n, want, [0, n - 1])
    for i, pr in enumerate(probs):
        key = format(i, "02b")
        if pr > 0:
            assert abs(counts[key]["probability"] - pr) <= 1e-12


def _adjoint_rank(rank, world, uid, cir, data, q):
    try:
        os.environ["QSV_NCCL_LIB"] = str(SHIM)
        from paper_2512_18995_b200 import qsv as Q

        ctx = Q.Context(0, rank, world, uid)
        g = Q.adjoint_gradients(cir, None, data, ctx=ctx)
        q.put((rank, list(g.param_grads), list(g.data_grads)))
        ctx.close()
    except Exception:
        q.put((rank, traceback.format_exc(), None))


def run_adjoint(cir, world, data=()):
    uid = qsv.Context.nccl_unique_id()
    ctxm = mp.get_context("spawn")
    q = ctxm.Queue()
    procs = [ctxm.Process(target=_adjoint_rank, args=(r, world, uid, cir, list(data), q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    try:
        for _ in range(world):
            r, pg, dg = q.get(timeout=180)
            if dg is None:
                raise AssertionError(f"rank {r} failed:\n{pg}")
            res[r] = (pg, dg)
    finally:
        for p in procs:
            p.join(timeout=60)
            if p.is_alive():
                p.kill()
    return res


def test_adjoint_dist_matches_single_rank():  # tests/test_dist.cpp:224-276
    # (the reference's 1-qubit-on-2-ranks case leaves no local qubit; this
    # engine needs n >= log2(ranks) + 1 and says so: "more ranks than amplitudes")
    cir = qsv.Circuit(2)
    cir.ry(0, 1.1, trainable=True)
    cir.observable([0], "z")
    res = run_adjoint(cir, 2)  # wire 0 is the rank qubit
    for r in res:
        assert abs(res[r][0][0] + np.sin(1.1)) <= 1e-10
    rng = qsv.Rng(13, "shim-adj")
    for world in (2, 4):
        c = random_circuit(rng, 6, 14)
        for g in c.gates():
            g.trainable = bool(g.params)
        c.observable([0], "z")
        c.observable([2], "x")
        want = qsv.adjoint_gradients(c)
        res = run_adjoint(c, world)
        for r in res:
            assert np.max(np.abs(np.asarray(res[r][0]) - want.param_grads)) <= 1e-10
    c = qsv.Circuit(4)
    c.rylayer(encode=True)
    c.cnot_ring()
    c.observable([0], "z")
    c.observable([1], "x")
    data = [0.0, 1.0, 2.0, 3.0]
    want = qsv.adjoint_gradients(c, None, data)
    res = run_adjoint(c, 4, data)
    for r in res:
        assert np.max(np.abs(np.asarray(res[r][1]) - want.data_grads)) <= 1e-10


@pytest.mark.parametrize("world", [2, 4, 8])
def test_swaps_fused_into_passes_through_peer_memory(world):
    # the swaps after a pass are done by the pass itself: its last register
    # group stores every amplitude into the destination rank's scratch state
    # (CUDA IPC mappings of every rank's buffers), then the states flip; with
    # QSV_P2P_SWAP=0 the same plan runs its swaps as NCCL all-to-alls
    rng = qsv.Rng(29, f"shim-fused-{world}")
    for n, cir, dtype, tol in ((14, W.cfg4_circuit(14, layers=4), qsv.C128, 1e-12),
                               (13, W.cfg3_circuit(13), qsv.C128, 1e-12),
                               (14, W.cfg5_circuit(14, layers=3), qsv.C64, 1e-5)):
        sched = qsv.plan_schedule(n, cir.gates(), dtype=dtype, world=world)
        assert any(s["kind"] == "swap" and s["fused"] for s in sched["steps"]), n
        psi = random_state(rng, n)
        want = O.port_forward(n, cir.gates(), init=psi)[0]
        for env, mode in (({}, 1), ({"QSV_P2P_SWAP": "0"}, -1)):
            got, z, nrm, _, _ = run_ranks(n, cir.gates(), world, init=psi, dtype=dtype, env=env)
            assert all(v == mode for v in PEER_MEMORY.values()), (PEER_MEMORY, env)
            assert np.max(np.abs(got - want)) <= tol, (world, n, env)
            if dtype == qsv.C64:
                assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-6, (world, n, env)
            assert abs(nrm - 1.0) <= 10 * tol
