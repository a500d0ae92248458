python -c "import __graft_entry__ as g; g.build()" > /dev/null
make -C tests/fake_nccl >/dev/null
timeout 900 python -m pytest tests/test_gpu_multi.py -q -x -m gpu 2>&1 | tail -15
timeout 600 python scripts/value_apply_time.py 20
