python -c "from paper_2512_18995_b200 import build; build.build()"
timeout 900 python scripts/scatter_check.py 2>&1 | tail -40
AB_REPS=12 timeout 900 python scripts/ab.py 30 cfg3 '' 'OPT_tile_bits=12' 'OPT_tile_bits=12,QSV_SCATTER_OUT=0' 2>&1 | tail -3
