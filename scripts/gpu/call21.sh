python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=3
timeout 900 python scripts/ab.py 28 cfg4f "" "QSV_MAX_GROUPS=8" "QSV_MAX_GROUPS=6" "QSV_MAX_GROUPS=5" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg4f "" "QSV_MAX_GROUPS=8" "QSV_MAX_GROUPS=6" "QSV_MAX_GROUPS=5" 2>&1 | grep median
timeout 900 python scripts/ab.py 32 cfg4f "" "QSV_MAX_GROUPS=8" "QSV_MAX_GROUPS=6" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg5f "" "QSV_MAX_GROUPS=8" "QSV_MAX_GROUPS=6" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 brick "OPT_dense_blocks=-1" "OPT_dense_blocks=-1,QSV_MAX_GROUPS=8" "OPT_dense_blocks=-1,QSV_MAX_GROUPS=6" 2>&1 | grep median
