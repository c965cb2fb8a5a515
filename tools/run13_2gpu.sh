set -x
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/topo13.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest13_multi.log 2>&1; echo pytest_multi=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 \
    bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench13_n2.log 2>&1; echo bench_n2=$?
tail -n 3 gpurun_out/pytest13_multi.log; tail -n 1 gpurun_out/bench13_n2.log | cut -c 1-400
