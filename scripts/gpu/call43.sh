python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=3
timeout 900 python scripts/ab.py 30 cfg5f "" "OPT_tile_bits=12,OPT_reg_slots=3" "OPT_tile_bits=12,OPT_reg_slots=3,QSV_PREFETCH=0" "OPT_tile_bits=12,OPT_reg_slots=4,QSV_MAX_THREADS=128" "OPT_tile_bits=13,OPT_reg_slots=4" 2>&1 | grep median
