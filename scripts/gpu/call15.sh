python -c "from paper_2512_18995_b200 import build; build.build()"
timeout 300 python -m pytest tests/test_gpu_dense_blocks.py -q -x 2>&1 | tail -4
for v in 0 1; do echo "QSV_DENSE_V2=$v"; QSV_DENSE_V2=$v timeout 300 python scripts/dense_ab.py 28 20 local 2>&1 | tail -1; QSV_DENSE_V2=$v timeout 300 python scripts/dense_ab.py 28 20 dense 2>&1 | tail -1; done
