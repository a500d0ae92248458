# micro-benchmarks, codegen A/B, ncu of the c64 pass
python -c "from paper_2512_18995_b200 import build; build.build()"
nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -lineinfo -I paper_2512_18995_b200/csrc scripts/micro/swap_copy.cu -o /tmp/swap_copy && { timeout 300 /tmp/swap_copy 32 16; timeout 300 /tmp/swap_copy 33 8; } > gpurun_out/r2_swap_copy.txt 2>&1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo scripts/micro/tc_dense5.cu -o /tmp/tc_dense5 && timeout 300 /tmp/tc_dense5 30 > gpurun_out/r2_tc_chain.txt 2>&1
cat gpurun_out/r2_swap_copy.txt gpurun_out/r2_tc_chain.txt
AB_REPS=10 timeout 900 python scripts/ab.py 28 cfg5 '' 'QSV_X_NOSIGN=1' 'QSV_X_NOSIGN=1,QSV_X_NOPAIR=1' 'QSV_X_NOSIGN=1,QSV_X_NOPAIR=1,QSV_X_OLDSWZ=1' 2>&1 | tail -4 | tee gpurun_out/r2_ab_cfg5.txt
AB_REPS=10 timeout 900 python scripts/ab.py 28 cfg4 '' 'QSV_X_NOSIGN=1' 2>&1 | tail -2 | tee gpurun_out/r2_ab_cfg4.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qsv_pass -c 3 -o gpurun_out/r2_cfg5_28q python scripts/prof_one.py cfg5 28 > gpurun_out/r2_ncu_cfg5.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2_cfg5_28q.ncu-rep 2>&1 | tee gpurun_out/r2_ncu_cfg5_summary.txt
