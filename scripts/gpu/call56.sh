python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/forward_time.py 12 20 24
QSV_NO_PLAN_CACHE=1 timeout 600 python scripts/forward_time.py 12 20 24
for f in tests/test_gpu_parity.py tests/test_gpu_mixed.py tests/test_bridge_cpp.py tests/test_circuit_file.py tests/test_gpu_adjoint.py; do timeout 900 python -m pytest $f -q -x -m gpu 2>&1 | tail -1; done
