python -c "import __graft_entry__ as g; g.build()" > /dev/null
export AB_REPS=3
for n in 28 30 32; do
timeout 900 python scripts/ab.py $n cfg3c64 "" "OPT_tile_bits=12,OPT_reg_slots=4" "OPT_tile_bits=12" "OPT_tile_bits=11,OPT_reg_slots=4" "OPT_tile_bits=13,OPT_reg_slots=4" 2>&1 | grep median
done
timeout 900 python scripts/ab.py 33 cfg5f "" "OPT_tile_bits=12,OPT_reg_slots=4" 2>&1 | grep median
