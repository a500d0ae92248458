python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=3
timeout 900 python scripts/ab.py 30 cfg4f "" "QSV_PREFETCH=0" 2>&1 | grep median
timeout 900 python scripts/ab.py 32 cfg4f "" "QSV_PREFETCH=0" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg3 "" "QSV_PREFETCH=0" 2>&1 | grep median
