python -c "from paper_2512_18995_b200 import build; build.build()"
for w in "cfg4 32" "cfg5 33" "brick 30" "cfg3 30"; do
  for v in 0 1; do echo -n "search=$v "; QSV_TILE_SEARCH=$v timeout 600 python scripts/tile_search_ab.py $w 2>&1 | tail -1; done
done
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x 2>&1 | tail -3
