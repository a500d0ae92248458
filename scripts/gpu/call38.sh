python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python bench.py > gpurun_out/bench_r2v4.json 2> gpurun_out/bench_r2v4.err; echo bench rc=$?
tail -c 400 gpurun_out/bench_r2v4.json
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qsv_pass -c 6 -o gpurun_out/r2_cfg4f_28q_p1 python scripts/prof_one.py cfg4f 28 > gpurun_out/r2_ncu_cfg4f_p1.log 2>&1; echo ncu rc=$?
python scripts/ncu_summary.py gpurun_out/r2_cfg4f_28q_p1.ncu-rep | tee gpurun_out/r2_ncu_cfg4f_p1_summary.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k passenger 2>&1 | tail -1
