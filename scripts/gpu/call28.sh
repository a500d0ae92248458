python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python bench.py > gpurun_out/bench_r2v3.json 2> gpurun_out/bench_r2v3.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_r2v3.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qsv_pass -c 6 -o gpurun_out/r2_cfg4f_28q python scripts/prof_one.py cfg4f 28 > gpurun_out/r2_ncu_cfg4f.log 2>&1; echo ncu rc=$?
python scripts/ncu_summary.py gpurun_out/r2_cfg4f_28q.ncu-rep | tee gpurun_out/r2_ncu_cfg4f_summary.txt
