python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=3
timeout 900 python scripts/ab.py 28 cfg4f "" "QSV_PASSENGERS=1" "QSV_PASSENGERS=2" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg4f "" "QSV_PASSENGERS=1" "QSV_PASSENGERS=2" 2>&1 | grep median
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "family or mirror or random" 2>&1 | tail -2
QSV_PASSENGERS=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "family or mirror or random" 2>&1 | tail -2
