python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/value_apply_time.py 14 20 24
bash scripts/gpu/call8.sh
timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/bench_aux_check3.json 2> gpurun_out/bench_aux_check3.err; echo bench rc=$?
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_aux_check3.json').read().strip().splitlines()[-1])
for k in ('measure_24q','density_10q'): print(k, json.dumps(d['aux'][k])[:300])
PY
