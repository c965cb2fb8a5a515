set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest15_parity.log 2>&1; echo pytest_parity=$?; tail -n 3 gpurun_out/pytest15_parity.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "p2p" > gpurun_out/pytest15_p2p.log 2>&1; echo pytest_p2p=$?
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "nccl" > gpurun_out/pytest15_nccl.log 2>&1; echo pytest_nccl=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench15_n2_p2p.log 2>&1; echo bench_p2p=$?
AMG_TRANSPORT=nccl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
    bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench15_n2_nccl.log 2>&1; echo bench_nccl=$?
tail -n 5 gpurun_out/pytest15_p2p.log; tail -n 3 gpurun_out/pytest15_nccl.log
tail -n 1 gpurun_out/bench15_n2_p2p.log | cut -c 1-300; tail -n 1 gpurun_out/bench15_n2_nccl.log | cut -c 1-300
