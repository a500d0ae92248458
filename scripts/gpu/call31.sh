python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=7
timeout 900 python scripts/ab.py 30 cfg3 "" "QSV_X_NODEFER_PASS=1" "QSV_X_NODEFER=1" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg3c64 "" "QSV_X_NODEFER_PASS=1" "QSV_X_NODEFER=1" 2>&1 | grep median
export AB_REPS=3
timeout 900 python scripts/ab.py 30 cfg4f "" "QSV_X_NODEFER_PASS=1" "QSV_X_NODEFER=1" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg5f "" "QSV_X_NODEFER_PASS=1" "QSV_X_NODEFER=1" 2>&1 | grep median
