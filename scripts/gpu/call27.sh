python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=3
timeout 900 python scripts/ab.py 30 cfg3c64 "" "QSV_X_NOLIGHT=1" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 brick "OPT_dense_blocks=-1" "OPT_dense_blocks=-1,QSV_X_NOLIGHT=1" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg5f "" "QSV_X_NOLIGHT=1" 2>&1 | grep median
for f in tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_dense_blocks.py tests/test_circuit_file.py; do
  echo "=== $f"; timeout 1500 python -m pytest $f -q -x -m gpu 2>&1 | tail -2
done
