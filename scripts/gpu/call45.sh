python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 300 python scripts/cfg2_bench.py 2>&1 | head -1
timeout 900 python scripts/tile_search_ab.py cfg5 33
export AB_REPS=3
timeout 900 python scripts/ab.py 30 cfg3c64 "" "OPT_reg_slots=3" 2>&1 | grep median
timeout 900 python scripts/ab.py 30 brick "OPT_dense_blocks=-1" "OPT_dense_blocks=-1,OPT_reg_slots=3" 2>&1 | grep median
bash scripts/gpu/call8.sh
