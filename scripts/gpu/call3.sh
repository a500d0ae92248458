python -c "from paper_2512_18995_b200 import build; build.build()"
make -C tests/fake_nccl >/dev/null
timeout 900 python -m pytest tests/test_gpu_multi.py tests/test_bridge_cpp.py -v -x --timeout 180 2>&1 | tail -30
