python -c "import __graft_entry__ as g; g.build()" > /dev/null
for b in 2 4 8 1; do echo "bps=$b"; QSV_ADJ_BLOCKS_PER_SM=$b timeout 600 python scripts/adjoint_parts.py 20 | tail -2; QSV_ADJ_BLOCKS_PER_SM=$b timeout 600 python scripts/adjoint_parts.py 24 | tail -2; done
