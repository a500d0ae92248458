python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=3
timeout 900 python scripts/ab.py 30 cfg5f "" "QSV_MAX_THREADS=256" "QSV_MAX_THREADS=128" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg4f "" "QSV_MAX_THREADS=128" 2>&1 | grep median
