python -c "import __graft_entry__ as g; g.build()" > /dev/null
QSV_PASSENGERS=2 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "family or mirror or random" 2>&1 | grep -E "Error|error|assert|FAILED|def test|^E " | head -30
QSV_PASSENGERS=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu 2>&1 | tail -5
