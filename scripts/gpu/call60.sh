python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "measure" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_circuit_file.py tests/test_bridge_cpp.py -q -x -m gpu 2>&1 | tail -1
timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/bench_aux_check2.json 2> gpurun_out/bench_aux_check2.err; echo bench rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_aux_check2.json').read().strip().splitlines()[-1])
for k in ('measure_24q','density_10q'): print(k, json.dumps(d['aux'][k])[:500])
PY
