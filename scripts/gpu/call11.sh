python -c "from paper_2512_18995_b200 import build; build.build()"
timeout 600 python scripts/dense_ab.py 28 20 local
timeout 600 python scripts/dense_ab.py 28 40 local
timeout 600 python scripts/dense_ab.py 30 20 local
