python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qsv_pass -c 5 -o gpurun_out/r2_cfg5f_28q python scripts/prof_one.py cfg5f 28 > gpurun_out/r2_ncu_cfg5f.log 2>&1; echo ncu rc=$?
python scripts/ncu_summary.py gpurun_out/r2_cfg5f_28q.ncu-rep | tee gpurun_out/r2_ncu_cfg5f_summary.txt
