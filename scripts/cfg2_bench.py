"""cfg2 timing: 4096 x 12-qubit c64 batched VQC, encoded Ry + 6 x (U3 + ring CZ), <Z_i> per row."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2512_18995_b200 import qsv, workloads as W
cir, data = W.cfg2_circuit()
ctx = qsv.default_context()
for opts in ({"jit": 1}, {"jit": -1}, {"jit": 1, "reg_slots": 3}, {"jit": 1, "tile_bits": 12, "reg_slots": 4}):
    p = qsv.Plan(12, cir.gates(), dtype=qsv.C64, opts=opts)
    st = qsv.QubitState(12, batch=4096, dtype=qsv.C64)
    s = torch.cuda.ExternalStream(ctx.stream())
    for _ in range(3):
        qsv.check(qsv.lib().qsv_state_set_basis(st.h, 0)); p.execute(st, data); z = st.expect_z_all()
    ctx.sync()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    K = 20
    e0.record(s)
    for _ in range(K):
        p.execute(st, data)
    e1.record(s); e1.synchronize()
    t_exec = e0.elapsed_time(e1) / K
    t0 = time.perf_counter()
    for _ in range(K):
        qsv.check(qsv.lib().qsv_state_set_basis(st.h, 0)); p.execute(st, data); z = st.expect_z_all()
    t_full = (time.perf_counter() - t0) / K * 1e3
    print(f"opts={opts} passes={p.info['npasses']} execute={t_exec:.3f} ms  basis+execute+<Z>={t_full:.3f} ms  "
          f"circuits/s={4096/(t_full/1e3):.0f}", flush=True)
