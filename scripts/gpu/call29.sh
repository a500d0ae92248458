python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/tile_search_ab.py cfg5 30
QSV_PF_MAXKB=128 QSV_PREFETCH=1 timeout 600 python scripts/tile_search_ab.py cfg5 30
QSV_PF_MAXKB=128 QSV_PREFETCH=1 QSV_MAX_THREADS=1024 timeout 600 python scripts/tile_search_ab.py cfg5 30
QSV_MAX_THREADS=1024 timeout 600 python scripts/tile_search_ab.py cfg5 30
QSV_PF_MAXKB=128 QSV_PREFETCH=1 QSV_MAX_THREADS=1024 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "cfg5 or random or variants" 2>&1 | tail -2
