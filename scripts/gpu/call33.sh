python -c "import __graft_entry__ as g; g.build()" > /dev/null
bash scripts/bench_shim2.sh
tail -3 gpurun_out/bench2_1.log; tail -3 gpurun_out/bench2_0.log
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 2>/dev/null | tail -c 600
