"""The multi-GPU path's host logic on CPU (torch.distributed "gloo").

The C++ planner's distributed schedule (qsv_plan_dry with world > 1: local
passes with their gates on physical bits, global<->local qubit swaps) is
executed by world_size 2 and 4 CPU processes, each holding its rank's slice
(the indices whose top log2(world) bits equal the rank). A
swap step performs the same pairwise half-slice exchange dist.cu issues with
NCCL send/recv, here with gloo. The gathered state must equal the
single-rank reference (the reference's own dist test strategy,
tests/test_dist.cpp:59-62, 128-174).
"""
import os
import socket

import numpy as np
import pytest

from oracle import oracle as O
from paper_2512_18995_b200 import qsv
from paper_2512_18995_b200 import workloads as W
from paper_2512_18995_b200.qsv import Circuit, Rng, make_gate
from tests.helpers import random_circuit, random_state


def apply_phys(sl, g, rank, nl):
    """One scheduled gate on a rank slice; bits are physical, rank bits fixed."""
    t, ctl = g["t"], g["c"]
    k = len(t)
    m = np.array([complex(a, b) for a, b in g["m"]]).reshape(1 << k, 1 << k)
    idx = np.arange(len(sl), dtype=np.int64)
    glob = (np.int64(rank) << nl) | idx
    ok = np.ones(len(sl), bool)
    for c in ctl:
        ok &= ((glob >> c) & 1) == 1
    if any(b >= nl for b in t):  # must be diagonal: no communication
        assert np.allclose(m, np.diag(np.diag(m))), "non-diagonal gate on a global bit"
        v = np.zeros(len(sl), dtype=np.int64)
        for b in t:
            v = (v << 1) | ((glob >> b) & 1)
        d = np.diag(m)
        sl[ok] *= d[v[ok]]
        return
    tmask = 0
    for b in t:
        tmask |= 1 << b
    base = idx[((idx & tmask) == 0) & ok]
    offs = []
    for j in range(1 << k):
        o = 0
        for i, b in enumerate(t):
            if (j >> (k - 1 - i)) & 1:
                o |= 1 << b
        offs.append(o)
    sub = np.stack([sl[base | o] for o in offs])
    new = m @ sub
    for j, o in enumerate(offs):
        sl[base | o] = new[j]


def permute_bits(sl, out_perm):
    idx = np.arange(len(sl), dtype=np.int64)
    dst = np.zeros_like(idx)
    for b, q in enumerate(out_perm):
        dst |= ((idx >> b) & 1) << q
    out = np.empty_like(sl)
    out[dst] = sl
    return out


def global_permute(sl, gperm, rank, world, nl):
    """The swaps fused into a pass (PassHost::gperm): every amplitude goes
    straight to the rank and local index the global bit permutation puts it
    at -- what the pass kernel's peer-memory stores do -- here as index/value
    messages over gloo."""
    import torch
    import torch.distributed as dist

    idx = np.arange(len(sl), dtype=np.int64)
    glob = (np.int64(rank) << nl) | idx
    out = np.zeros_like(glob)
    for b, q in enumerate(gperm):
        out |= ((glob >> b) & 1) << q
    dest, dloc = out >> nl, out & ((1 << nl) - 1)
    new = np.empty_like(sl)
    mine = dest == rank
    new[dloc[mine]] = sl[mine]
    ops, bufs = [], []
    for peer in range(world):
        if peer == rank:
            continue
        m = dest == peer
        msg = np.concatenate([dloc[m].astype(np.float64), sl[m].view(np.float64)])
        send = torch.from_numpy(msg)
        recv = torch.empty_like(send)  # the exchange is symmetric in size
        ops += [dist.P2POp(dist.isend, send, peer), dist.P2POp(dist.irecv, recv, peer)]
        bufs.append(recv)
    if ops:
        for q in dist.batch_isend_irecv(ops):
            q.wait()
    for recv in bufs:
        r = recv.numpy()
        k = len(r) // 3
        new[r[:k].astype(np.int64)] = r[k:].view(np.complex128)
    return new


def run_schedule(rank, world, sched, init_full, fused=False):
    import torch
    import torch.distributed as dist

    nl = sched["nlocal"]
    sl = init_full[rank << nl:(rank + 1) << nl].copy()
    idx = np.arange(len(sl), dtype=np.int64)
    sent = 0
    fused_done = False
    for step in sched["steps"]:
        if step["kind"] == "pass":
            if step["fused"] and fused_done:
                continue
            for g in step["gates"]:
                assert g["enc"] < 0
                apply_phys(sl, g, rank, nl)
            if step["out_perm"]:
                sl = permute_bits(sl, step["out_perm"])
            fused_done = fused and bool(step["gperm"])
            if fused_done:
                sl = global_permute(sl, step["gperm"], rank, world, nl)
            continue
        if step["fused"] and fused_done:
            continue
        fused_done = False
        for gb, lb in step["pairs"]:
            r = gb - nl
            partner = rank ^ (1 << r)
            my = (rank >> r) & 1
            mask = ((idx >> lb) & 1) == (1 - my)
            send = torch.from_numpy(np.ascontiguousarray(sl[mask]).view(np.float64).copy())
            recv = torch.empty_like(send)
            reqs = dist.batch_isend_irecv([dist.P2POp(dist.isend, send, partner), dist.P2POp(dist.irecv, recv, partner)])
            for q in reqs:
                q.wait()
            sl[mask] = recv.numpy().view(np.complex128)
            sent += send.numel() * 8
    return sl, sent


def _worker(rank, world, port, sched, init_full, out_dir, fused=False):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sl, sent = run_schedule(rank, world, sched, init_full, fused)
        np.save(os.path.join(out_dir, f"r{rank}.npy"), sl)
        np.save(os.path.join(out_dir, f"s{rank}.npy"), np.array([sent]))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_distributed(n, gates, world, init_full, tmp_path, opts=None, fused=False):
    import torch.multiprocessing as mp

    sched = qsv.plan_schedule(n, gates, world=world, opts=opts)
    mp.spawn(_worker, args=(world, free_port(), sched, init_full, str(tmp_path), fused), nprocs=world, join=True)
    got = np.concatenate([np.load(tmp_path / f"r{r}.npy") for r in range(world)])
    sent = sum(int(np.load(tmp_path / f"s{r}.npy")[0]) for r in range(world))
    return got, sched, sent


@pytest.mark.parametrize("world", [2, 4])
def test_random_circuits_across_world_sizes(world, tmp_path):  # test_dist.cpp:128-145
    rng = Rng(7, "dist-equiv")
    for trial in range(3):
        n = 5 + rng.next_below(4)
        cir = random_circuit(rng, n, 18)
        psi = random_state(rng, n)
        want = O.port_forward(n, cir.gates(), init=psi)[0]
        got, sched, _ = run_distributed(n, cir.gates(), world, psi, tmp_path)
        assert np.max(np.abs(got - want)) < 1e-12, (world, trial)


def test_qft_matches_single_rank(tmp_path):  # test_dist.cpp:147-160
    n = 10
    cir = qsv.qft_circuit(n)
    init = np.zeros(1 << n, complex)
    init[0] = 1
    got, _, _ = run_distributed(n, cir.gates(), 4, init, tmp_path)
    want = O.port_forward(n, cir.gates())[0]
    assert np.max(np.abs(got - want)) < 1e-12
    assert np.max(np.abs(np.abs(got) - 2.0 ** -5)) < 1e-12


def test_cfg_families_distributed(tmp_path):
    for cir, n, world in ((W.cfg4_circuit(8, layers=3), 8, 2), (W.cfg5_circuit(8, layers=2), 8, 4),
                          (W.cfg3_circuit(9), 9, 2)):
        psi = random_state(Rng(1, "dist-cfg"), n)
        want = O.port_forward(n, cir.gates(), init=psi)[0]
        got, _, _ = run_distributed(n, cir.gates(), world, psi, tmp_path)
        assert np.max(np.abs(got - want)) < 1e-12


def test_local_and_diagonal_gates_send_nothing():  # test_dist.cpp:96-110
    gates = [make_gate("h", [3]), make_gate("x", [2]), make_gate("rzz", [4, 5], [], [0.7]),
             make_gate("rz", [0], [], [0.3]), make_gate("p", [1], [0], [0.9])]
    info, _ = qsv.plan_dry(6, gates, world=4)
    assert info["nswaps"] == 0 and info["comm_bytes_per_exec"] == 0


def test_global_target_needs_one_exchange():  # test_dist.cpp:112-126
    info, _ = qsv.plan_dry(3, [make_gate("h", [0])], world=2)
    # one swap to bring wire 0 local, one to restore the canonical layout;
    # each moves half a slice (the reference moves the whole slice per gate)
    assert info["nswaps"] == 2
    assert info["comm_bytes_per_exec"] == 2 * 16 * 2  # 2 swaps x half of a 4-amplitude slice


def test_rejects_non_power_of_two_world():  # test_dist.cpp:90-94
    with pytest.raises(qsv.InvalidInput):
        qsv.plan_dry(4, [make_gate("h", [0])], world=3)


@pytest.mark.parametrize("world", [2, 4])
def test_swaps_fused_into_passes(world, tmp_path):
    # with specialised kernels the swaps after a pass are fused into it (its
    # stores go straight to the destination rank through peer memory); the
    # fused schedule and the NCCL-swap schedule must both equal the reference
    rng = Rng(17, "dist-fused")
    cases = [(W.cfg4_circuit(9, layers=3), 9), (W.cfg3_circuit(9), 9), (random_circuit(rng, 8, 30), 8)]
    nfused = 0
    for cir, n in cases:
        psi = random_state(rng, n)
        want = O.port_forward(n, cir.gates(), init=psi)[0]
        sched = qsv.plan_schedule(n, cir.gates(), world=world, opts={"jit": 1})
        nfused += sum(1 for s in sched["steps"] if s["kind"] == "swap" and s["fused"])
        for fused in (False, True):
            got, _, _ = run_distributed(n, cir.gates(), world, psi, tmp_path, opts={"jit": 1}, fused=fused)
            assert np.max(np.abs(got - want)) < 1e-12, (world, n, fused)
    assert nfused > 0
