python -c "import __graft_entry__ as g; g.build()"
make -C tests/fake_nccl >/dev/null
for f in tests/test_gpu_parity.py tests/test_gpu_dense_blocks.py tests/test_gpu_multi.py tests/test_bridge_cpp.py tests/test_gpu_fullsize.py tests/test_gpu_adjoint.py tests/test_gpu_mixed.py tests/test_gpu_dist_shim.py tests/test_circuit_file.py; do
  echo "=== $f"; timeout 1500 python -m pytest $f -q -m gpu 2>&1 | tail -4
done
timeout 600 python -c "import __graft_entry__ as g; g.smoke()"
