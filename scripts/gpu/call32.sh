python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=5
timeout 900 python scripts/ab.py 30 cfg3c64 "" "QSV_X_NODEFER=1" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg3 "" "QSV_X_DEFER=1" 2>&1 | grep median
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_mixed.py tests/test_gpu_adjoint.py -q -x -m gpu 2>&1 | tail -2
make -C tests/fake_nccl >/dev/null; timeout 900 python -m pytest tests/test_gpu_dist_shim.py tests/test_gpu_multi.py -q -x -m gpu 2>&1 | tail -2
