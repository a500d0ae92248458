"""DRAM traffic per launch of the qsv_pass kernels in an ncu --set full report -> JSON (profiles/)."""
import csv, json, subprocess, sys
rep, out, workload = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout.splitlines()))
hdr = rows[0]
launches = []
for r in rows[2:]:
    d = dict(zip(hdr, r))
    if "qsv_pass" not in d.get("Kernel Name", ""):
        continue
    launches.append({"kernel": "qsv_pass", "duration_ms": float(d["gpu__time_duration.sum"]) / (1e6 if "gpu__time_duration.sum" in d and float(d["gpu__time_duration.sum"]) > 1e5 else 1),
                     "dram_read_GB": float(d["dram__bytes_read.sum"]), "dram_write_GB": float(d["dram__bytes_write.sum"])})
units = dict(zip(hdr, rows[1]))
scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}
us = scale.get(units.get("dram__bytes_read.sum", "byte"), 1.0)
tu = units.get("gpu__time_duration.sum", "ns")
for l in launches:
    l["duration_ms"] = l["duration_ms"]
traffic = sum((l["dram_read_GB"] + l["dram_write_GB"]) * us for l in launches) / max(1, len(launches))
json.dump({"workload": workload, "source": f"ncu --set full ({rep})", "units": {"dram": units.get("dram__bytes_read.sum"), "time": tu},
           "launches": launches, "traffic_per_launch_bytes": traffic}, open(out, "w"), indent=1)
print(json.dumps({"traffic_per_launch_bytes": traffic, "n": len(launches)}))
