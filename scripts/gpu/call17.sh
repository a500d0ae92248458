python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu 2>&1 | tail -3
export AB_REPS=7
for c in "28 cfg4f" "28 cfg5f"; do
  timeout 600 python scripts/ab.py $c "" "QSV_X_NOXPERM=1" "QSV_X_NOHOIST=1" "QSV_X_NOHOIST=1,QSV_X_NOXPERM=1" 2>&1 | grep median
done
timeout 300 python scripts/ab.py 30 cfg3 "" "QSV_X_NOHOIST=1,QSV_X_NOXPERM=1" 2>&1 | grep median
timeout 600 python scripts/tile_search_ab.py cfg4 32
timeout 600 python scripts/tile_search_ab.py cfg5 33
