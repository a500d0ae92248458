python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python -m pytest tests/test_gpu_adjoint.py -q -x -m gpu 2>&1 | tail -3
make -C tests/fake_nccl >/dev/null; timeout 900 python -m pytest tests/test_gpu_dist_shim.py -q -x -m gpu -k adj 2>&1 | tail -2
timeout 900 python scripts/adjoint_time.py 16 20 22 24
