python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=3
timeout 900 python scripts/ab.py 30 cfg5f "" "QSV_X_UNROLL=1" 2>&1 | grep median
