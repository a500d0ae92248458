python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python bench.py --steps 3 --warmup 3 --e2e-steps 2 > gpurun_out/bench_aux_check.json 2> gpurun_out/bench_aux_check.err; echo bench rc=$?
tail -5 gpurun_out/bench_aux_check.err
python - <<'PY'
import json
d=json.loads(open('gpurun_out/bench_aux_check.json').read().strip().splitlines()[-1])
for k in ('adjoint_20q','measure_24q','density_10q'): print(k, json.dumps(d['aux'][k])[:600])
PY
