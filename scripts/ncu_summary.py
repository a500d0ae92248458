"""Key metrics of every kernel in an ncu report (one line each)."""
import csv, subprocess, sys
rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out)); hdr = rows[0]
want = {
    "dur_ms": "gpu__time_duration.sum", "dram_rd": "dram__bytes_read.sum", "dram_wr": "dram__bytes_write.sum",
    "dram%": "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "issue%": "sm__issue_active.avg.pct_of_peak_sustained_elapsed",
    "fp64%": "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fma%": "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "lsu%": "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "occ%": "sm__warps_active.avg.pct_of_peak_sustained_active",
    "regs": "launch__registers_per_thread", "inst": "smsp__inst_executed.sum", "shm_conf": "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
}
stalls = [k for k in hdr if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
units = rows[1]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get("Kernel Name", "?")[:40]
    parts = []
    for k, m in want.items():
        v = d.get(m, "")
        parts.append(f"{k}={v}")
    top = sorted(((float(d[k] or 0), k.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', '')) for k in stalls), reverse=True)[:6]
    print(name, " ".join(parts))
    print("   stalls:", ", ".join(f"{n}={v:.2f}" for v, n in top))
