set -x
nvidia-smi --query-gpu=name,memory.total --format=csv
nproc; free -g | head -2
python -c "from paper_2512_18995_b200 import build; build.build()"
timeout 900 python -m pytest tests/test_gpu_fullsize.py -k "26q" -q -s -x 2>&1 | tail -20
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench1.json 2> gpurun_out/r2_bench1.err; echo bench rc=$?
tail -c 3000 gpurun_out/r2_bench1.json
