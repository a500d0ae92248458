python -c "from paper_2512_18995_b200 import build; build.build()"
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qsv_pass -c 4 -o gpurun_out/r2_cfg3_30q python scripts/prof_one.py cfg3 30 > gpurun_out/r2_ncu_cfg3.log 2>&1; echo ncu rc=$?
python scripts/ncu_traffic.py gpurun_out/r2_cfg3_30q.ncu-rep gpurun_out/r2_traffic_cfg3_30q.json "cfg3 30q QFT+swaps, 4 passes (round-2 codegen: tile search, sign flushes)"
python scripts/ncu_summary.py gpurun_out/r2_cfg3_30q.ncu-rep | tee gpurun_out/r2_ncu_cfg3_summary.txt
