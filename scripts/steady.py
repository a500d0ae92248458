"""Per-step pass times over a long back-to-back run (power/clock behaviour)."""
import sys, subprocess, threading, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import numpy as np
import torch
from paper_2512_18995_b200 import qsv, workloads as W
n = int(sys.argv[1]) if len(sys.argv) > 1 else 30
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 30
cir = W.cfg3_circuit(n)
p = qsv.Plan(n, cir.gates(), dtype=qsv.C128)
st = qsv.QubitState(n, dtype=qsv.C128)
st.upload(W.cfg3_slice(0, 1 << n) / np.sqrt(1 << n))
for _ in range(3):
    p.execute(st)
p.ctx.sync()
clk = []
stop = False
def poll():
    while not stop:
        r = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,clocks.mem", "--format=csv,noheader,nounits"],
                           capture_output=True, text=True).stdout.strip()
        clk.append(r)
        time.sleep(0.1)
th = threading.Thread(target=poll); th.start()
for s in range(steps):
    ms = p.profile(st)
    print(f"step {s:2d} total {ms.sum():.3f} ms  {np.round(ms, 3).tolist()}", flush=True)
s = torch.cuda.ExternalStream(p.ctx.stream())
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
e0.record(s)
for _ in range(steps):
    p.execute(st)
e1.record(s); e1.synchronize()
print(f"execute-only: {e0.elapsed_time(e1) / steps:.3f} ms/step")
stop = True; th.join()
print("clocks(sm MHz, W, mem MHz):", clk)
