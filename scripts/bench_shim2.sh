export QSV_BENCH_SHARE_GPU=1 QSV_NCCL_LIB=$PWD/tests/fake_nccl/_build/libnccl_fake.so QSV_SWAP_STAGE_BYTES=4194304
make -C tests/fake_nccl > /dev/null 2>&1
for mode in 1 0; do
QSV_P2P_SWAP=$mode timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2953$mode bench.py --gpus 2 --steps 2 --warmup 1 --qubits 22 --e2e-steps 2 > gpurun_out/bench2_$mode.log 2>&1; echo rc=$? >> gpurun_out/bench2_$mode.log
done
