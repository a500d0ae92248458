python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python scripts/cfg2_bench.py 2>&1 | head -4
export AB_REPS=3
timeout 900 python scripts/ab.py 28 cfg5f "" "OPT_reg_slots=4" 2>&1 | grep median
timeout 900 python scripts/ab.py 32 cfg5f "" "OPT_reg_slots=4" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg5f "" "OPT_reg_slots=4" "OPT_reg_slots=4,QSV_MAX_THREADS=512" 2>&1 | grep median
