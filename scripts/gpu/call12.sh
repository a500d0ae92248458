python -c "import __graft_entry__ as g; g.build()"
for f in tests/test_gpu_dense_blocks.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py; do
  echo "=== $f"; timeout 1200 python -m pytest $f -q -m gpu 2>&1 | tail -3
done
timeout 1500 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench3.json 2> gpurun_out/r2_bench3.err; echo bench rc=$?
python -c "
import json; d=json.loads(open('gpurun_out/r2_bench3.json').read().strip().splitlines()[-1])
print(d['value'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])
for k in ('dense_local_30q','dense_brickwork_30q'): print(k, json.dumps(d['aux'][k]))
"
