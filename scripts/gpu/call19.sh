python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=3
timeout 900 python scripts/ab.py 30 cfg4f "" "OPT_tile_bits=12" "OPT_tile_bits=13" "OPT_tile_bits=12,OPT_reg_slots=3" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg5f "" "OPT_tile_bits=12,OPT_reg_slots=4" "OPT_tile_bits=11,OPT_reg_slots=4" "OPT_tile_bits=12,OPT_reg_slots=4,QSV_PREFETCH=0" "OPT_tile_bits=13,OPT_reg_slots=4" "OPT_tile_bits=12,OPT_reg_slots=3" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 brick "OPT_dense_blocks=-1" "OPT_dense_blocks=-1,OPT_tile_bits=12,OPT_reg_slots=4" "OPT_dense_blocks=-1,OPT_tile_bits=12" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 cfg3c64 "" "OPT_tile_bits=12,OPT_reg_slots=4" 2>&1 | grep median
