python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/apply_gate_time.py 14 20 24 28
QSV_X_NODIRECT=1 timeout 600 python scripts/apply_gate_time.py 20
bash scripts/gpu/call8.sh
