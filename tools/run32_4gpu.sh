set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest32_multi.log 2>&1; echo pytest_multi=$?; tail -2 gpurun_out/pytest32_multi.log; grep -E "^E  " gpurun_out/pytest32_multi.log | head -3
for T in p2p nccl; do
AMG_TRANSPORT=$T timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench32_n4_$T.log 2>&1; echo bench_n4_$T=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 \
    bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench32_n2_p2p.log 2>&1; echo bench_n2=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench32_n1.log 2>&1; echo bench_n1=$?
AMG_TUNE_CACHE=$PWD/gpurun_out/tune_R3.txt timeout 1200 python bench.py --config R3 --steps 3 --warmup 3 > gpurun_out/bench32_r3.log 2>&1; echo bench_r3=$?
for f in bench32_n4_p2p bench32_n4_nccl bench32_n2_p2p bench32_n1 bench32_r3; do tail -n 1 gpurun_out/$f.log | cut -c 1-160; done
