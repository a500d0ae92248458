python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=3
timeout 900 python scripts/ab.py 32 cfg4f "" "QSV_PASSENGERS=0" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg3 "" "QSV_PASSENGERS=0" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg5f "" "QSV_PASSENGERS=0" 2>&1 | grep median
for f in tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_adjoint.py tests/test_gpu_mixed.py; do timeout 900 python -m pytest $f -q -x -m gpu 2>&1 | tail -1; done
make -C tests/fake_nccl >/dev/null; timeout 900 python -m pytest tests/test_gpu_dist_shim.py tests/test_gpu_multi.py -q -x -m gpu 2>&1 | tail -1
