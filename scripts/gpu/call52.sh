python -c "import __graft_entry__ as g; g.build()" > /dev/null
timeout 600 python scripts/adjoint_parts.py 20
timeout 600 python scripts/adjoint_parts.py 18
