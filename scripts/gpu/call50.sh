python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_adjoint.py -q -x -m gpu 2>&1 | tail -3
timeout 900 python scripts/adjoint_time.py 14 16 18 20 22
