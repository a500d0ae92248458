python -c "from paper_2512_18995_b200 import build; build.build()"
timeout 600 python -m pytest tests/test_gpu_dense_blocks.py -q -s 2>&1 | grep -E "Error|passed|failed|assert|max abs" | head -30
timeout 600 python scripts/dense_ab.py 28 20 dense
timeout 600 python scripts/dense_ab.py 28 4 cfg5
