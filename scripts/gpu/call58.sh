bash scripts/gpu/call8.sh
timeout 900 python bench.py > gpurun_out/bench_r2v6.json 2> gpurun_out/bench_r2v6.err; echo bench rc=$?
tail -c 300 gpurun_out/bench_r2v6.json
