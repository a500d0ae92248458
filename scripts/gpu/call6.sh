python -c "from paper_2512_18995_b200 import build; build.build()"
nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -lineinfo -I paper_2512_18995_b200/csrc scripts/micro/swap_copy.cu -o /tmp/swap_copy && { timeout 300 /tmp/swap_copy 32 16; timeout 300 /tmp/swap_copy 33 8; } > gpurun_out/r2_swap_copy.txt 2>&1; cat gpurun_out/r2_swap_copy.txt
timeout 600 ncu --set full --clock-control none -k regex:block_copy -c 4 -o gpurun_out/r2_swap_copy_33q /tmp/swap_copy 33 8 > /dev/null 2>&1; python scripts/ncu_summary.py gpurun_out/r2_swap_copy_33q.ncu-rep > gpurun_out/r2_ncu_swap_copy.txt 2>&1; cat gpurun_out/r2_ncu_swap_copy.txt
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench2.json 2> gpurun_out/r2_bench2.err; echo bench rc=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-aux --e2e-steps 2 > gpurun_out/r2_ncu_launch.log 2>&1; echo ncu rc=$?
tail -c 1500 gpurun_out/r2_bench2.json
