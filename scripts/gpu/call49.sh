python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 900 python scripts/adjoint_time.py 14 16 18 20
