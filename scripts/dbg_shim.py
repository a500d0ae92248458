"""Debug: per-rank view of the multi-rank path through the NCCL shim."""
import multiprocessing as mp
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np


def rank_main(rank, world, uid, gname, q):
    os.environ["QSV_NCCL_LIB"] = os.path.abspath("tests/fake_nccl/_build/libnccl_fake.so")
    from paper_2512_18995_b200 import qsv as Q
    ctx = Q.Context(0, rank, world, uid)
    n = 10
    c = Q.Circuit(n)
    if gname == "h": c.h(0)
    elif gname == "x": c.x(0)
    else: c.ry(0, 0.3)
    st = Q.QubitState(n, ctx=ctx)
    p = Q.Plan(n, c.gates(), ctx=ctx)
    p.execute(st)
    loc = st.amplitudes()
    z = st.expect_z_all()[0]
    nrm = float(st.norm2()[0])
    q.put((rank, float(np.vdot(loc, loc).real), np.nonzero(np.abs(loc) > 1e-9)[0][:4].tolist(), z[:3].tolist(), nrm))
    del p, st
    ctx.close()


def main():
    os.environ["QSV_NCCL_LIB"] = os.path.abspath("tests/fake_nccl/_build/libnccl_fake.so")
    from paper_2512_18995_b200 import qsv
    for g in ("h", "x", "ry"):
        uid = qsv.Context.nccl_unique_id()
        cm = mp.get_context("spawn")
        q = cm.Queue()
        ps = [cm.Process(target=rank_main, args=(r, 2, uid, g, q)) for r in range(2)]
        for p in ps: p.start()
        for _ in range(2): print(g, q.get(timeout=120), flush=True)
        for p in ps: p.join(30)


if __name__ == "__main__":
    main()
