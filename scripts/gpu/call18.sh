python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=5
timeout 900 python scripts/ab.py 28 cfg4f "" "QSV_PREFETCH=0" "OPT_tile_bits=12" "OPT_reg_slots=3" "OPT_reg_slots=3,QSV_PREFETCH=0" "QSV_X_NOSCALE=1" "OPT_tile_bits=10" 2>&1 | grep median
timeout 900 python scripts/ab.py 28 cfg5f "" "OPT_tile_bits=12" "OPT_reg_slots=4" "OPT_tile_bits=12,OPT_reg_slots=4" "OPT_tile_bits=14" "QSV_X_NOSCALE=1" 2>&1 | grep median
