python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=5
timeout 900 python scripts/ab.py 28 cfg4f "" "QSV_X_CPOOL=1" "QSV_X_CPOOL=1,QSV_X_NOSCALE=1" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg4f "" "QSV_X_CPOOL=1" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg3 "" "QSV_X_CPOOL=1" 2>&1 | grep median
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "variants" 2>&1 | tail -2
QSV_X_CPOOL=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "variants or random or family" 2>&1 | tail -2
