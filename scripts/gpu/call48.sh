python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python bench.py > gpurun_out/bench_r2v5.json 2> gpurun_out/bench_r2v5.err; echo bench rc=$?
tail -c 300 gpurun_out/bench_r2v5.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_v5.csv python bench.py --steps 2 --warmup 1 --no-aux --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_launch_v5.log 2>&1; echo ncu rc=$?
