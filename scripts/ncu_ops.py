"""Opcode mix of the first kernel in an ncu report."""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out)); hdr = None; c = Counter(); s = Counter(); tot = 0
for r in rows:
    if r and r[0] == "Address": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    ie = hdr.index("Instructions Executed"); ss = hdr.index("Warp Stall Sampling (All Samples)")
    txt = r[1].strip().split()
    if not txt: continue
    op = txt[1] if txt[0].startswith("@") else txt[0]
    op = op.split(".")[0]
    v = float(r[ie] or 0); c[op] += v; s[op] += float(r[ss] or 0); tot += v
for op, v in c.most_common(int(sys.argv[2]) if len(sys.argv) > 2 else 20):
    print(f"{op:10s} {100*v/tot:6.2f}%  stall {s[op]:.0f}")
