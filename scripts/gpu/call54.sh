python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/apply_gate_time.py 14 20 24
