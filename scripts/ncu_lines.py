"""Summarise an ncu report: top CUDA source lines by instructions and stall samples."""
import csv, subprocess, sys
from collections import defaultdict
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
cur_file = None; hdr = None
agg = defaultdict(lambda: [0.0, 0.0, ""])
tot_i = tot_s = 0.0
for r in rows:
    if not r: continue
    if r[0] == "File Path": cur_file = r[1].split("/")[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    try:
        line = int(r[0])
    except ValueError:
        continue
    ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)")
    try:
        i = float(r[ie] or 0); s = float(r[ss] or 0)
    except ValueError:
        continue
    k = (cur_file, line)
    agg[k][0] += i; agg[k][1] += s; agg[k][2] = r[1][:90]
    tot_i += i; tot_s += s
print(f"total warp-instr {tot_i:.3e}, stall samples {tot_s:.0f}")
for k, (i, s, src) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:top]:
    print(f"{k[0]}:{k[1]:<5d} inst {100*i/tot_i:5.1f}%  stall {100*s/tot_s:5.1f}%  {src.strip()}")
