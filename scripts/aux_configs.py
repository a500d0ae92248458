"""Timing of the non-headline configs on one GPU (device-resident, CUDA events):
cfg1 (20q c128 forward + all <Z_i>), cfg2 (4096 x 12q c64 batched forward +
<Z_i> per row), and the cfg4/cfg5 families at the largest single-GPU n."""
import sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2512_18995_b200 import qsv, workloads as W

ctx = qsv.default_context()
s = torch.cuda.ExternalStream(ctx.stream())
L = qsv.lib()


def timed(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    ctx.sync()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s); e1.synchronize()
    return e0.elapsed_time(e1) / reps


cir = W.cfg1_circuit()
p = qsv.Plan(20, cir.gates(), dtype=qsv.C128)
st = qsv.QubitState(20, dtype=qsv.C128)
def f1():
    qsv.check(L.qsv_state_set_basis(st.h, 0)); p.execute(st)
ms = timed(f1)
ms_z = timed(lambda: (f1(), st.expect_z_all()), reps=10)
print(f"cfg1 20q c128 {p.info['ngates']} gates passes={p.info['npasses']}: forward {ms:.3f} ms "
      f"({p.info['ngates'] / ms * 1e3:.0f} gates/s); forward + <Z_i> (host sync) {ms_z:.3f} ms", flush=True)
pg = qsv.Plan(20, cir.gates(), dtype=qsv.C128, opts={"use_graph": 1})
def f1g():
    qsv.check(L.qsv_state_set_basis(st.h, 0)); pg.execute(st)
ms = timed(f1g)
print(f"cfg1 20q c128 as a CUDA graph (opts.use_graph): forward {ms:.3f} ms ({p.info['ngates'] / ms * 1e3:.0f} gates/s)",
      flush=True)

cir, data = W.cfg2_circuit()
p = qsv.Plan(12, cir.gates(), dtype=qsv.C64)
st = qsv.QubitState(12, batch=4096, dtype=qsv.C64)
def f2():
    qsv.check(L.qsv_state_set_basis(st.h, 0)); p.execute(st, data)
ms = timed(f2)
ms_z = timed(lambda: (f2(), st.expect_z_all()), reps=10)
def f2z():
    qsv.check(L.qsv_state_set_basis(st.h, 0)); return p.execute_expect_z(st, data)
ms_fz = timed(f2z, reps=10)
print(f"cfg2 fused forward + <Z_i> (qsv_plan_execute_expect_z, host sync) {ms_fz:.3f} ms "
      f"({4096 / ms_fz * 1e3:.0f} circuits/s)", flush=True)
pz = qsv.Plan(12, cir.gates(), dtype=qsv.C64, opts={"from_zero": 1})
ms_pz = timed(lambda: pz.execute(st, data))
ms_pzz = timed(lambda: pz.execute_expect_z(st, data), reps=10)
print(f"cfg2 from-|0> plan (product-state prefix synthesised in the pass): forward {ms_pz:.3f} ms "
      f"({4096 / ms_pz * 1e3:.0f} circuits/s); forward + <Z_i> {ms_pzz:.3f} ms ({4096 / ms_pzz * 1e3:.0f} circuits/s)",
      flush=True)
print(f"cfg2 4096x12q c64 {p.info['ngates']} gates passes={p.info['npasses']}: forward {ms:.3f} ms "
      f"({4096 / ms * 1e3:.0f} circuits/s); forward + <Z_i> (host sync) {ms_z:.3f} ms "
      f"({4096 / ms_z * 1e3:.0f} circuits/s)", flush=True)

for name, n, cir, dt in (("cfg4", 32, W.cfg4_circuit(32), qsv.C128), ("cfg5", 33, W.cfg5_circuit(33), qsv.C64)):
    p = qsv.Plan(n, cir.gates(), dtype=dt)
    st = qsv.QubitState(n, dtype=dt)
    ms = p.profile(st)[: p.info["npasses"]]
    amp = 8 if dt == qsv.C64 else 16
    print(f"{name} n={n} {p.info['ngates']} gates passes={p.info['npasses']}: {ms.sum():.1f} ms "
          f"({p.info['ngates'] / ms.sum() * 1e3:.0f} gates/s, avg pass {2 * amp * (1 << n) / (ms.mean() / 1e3) / 1e9:.0f} GB/s)",
          flush=True)
