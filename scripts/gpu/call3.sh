# c64 swizzle / pair A/B, swap gather-scatter micro, TC chain micro, parity of the c64 paths
python -c "from paper_2512_18995_b200 import build; build.build()"
make -C tests/fake_nccl >/dev/null
nvcc -O3 -std=c++20 -gencode arch=compute_100a,code=sm_100a -lineinfo -I paper_2512_18995_b200/csrc scripts/micro/swap_copy.cu -o /tmp/swap_copy && timeout 300 /tmp/swap_copy 32 16 > gpurun_out/r2_swap_copy.txt 2>&1; timeout 300 /tmp/swap_copy 33 8 >> gpurun_out/r2_swap_copy.txt 2>&1
nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo scripts/micro/tc_dense5.cu -o /tmp/tc_dense5 && timeout 300 /tmp/tc_dense5 30 > gpurun_out/r2_tc_chain.txt 2>&1
cat gpurun_out/r2_swap_copy.txt gpurun_out/r2_tc_chain.txt
AB_REPS=10 timeout 900 python scripts/ab.py 28 cfg5 '' 'QSV_X_NOPAIR=1' 'QSV_X_OLDSWZ=1,QSV_X_NOPAIR=1' 2>&1 | tail -4
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x 2>&1 | tail -5
