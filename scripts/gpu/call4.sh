python -c "from paper_2512_18995_b200 import build; build.build()"
make -C tests/fake_nccl >/dev/null
for f in tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_adjoint.py tests/test_gpu_mixed.py tests/test_gpu_dist_shim.py tests/test_circuit_file.py; do
  echo "=== $f"; timeout 1500 python -m pytest $f -q -m gpu --durations=8 2>&1 | tail -22
done
