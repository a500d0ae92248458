python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=5
timeout 900 python scripts/ab.py 30 cfg3 "" "OPT_reg_slots=3" "OPT_tile_bits=12" "QSV_MAX_THREADS=64" 2>&1 | grep median
