python -c "from paper_2512_18995_b200 import build; build.build()"
nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/fp_peaks scripts/micro/fp_peaks.cu && timeout 120 /tmp/fp_peaks | tee gpurun_out/r2_fp_peaks.txt
timeout 900 ncu --set full --import-source on --clock-control none -k regex:qsv_pass -c 5 -o gpurun_out/r2_cfg4_28q python scripts/prof_one.py cfg4 28 > gpurun_out/r2_ncu_cfg4.log 2>&1
python scripts/ncu_summary.py gpurun_out/r2_cfg4_28q.ncu-rep 2>&1 | tee gpurun_out/r2_ncu_cfg4_summary.txt
