set -x
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest26_multi.log 2>&1; echo pytest_multi=$?
for T in p2p nccl; do
AMG_TRANSPORT=$T timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 \
    bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench26_n4_$T.log 2>&1; echo bench_n4_$T=$?
done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 \
    bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench26_n2_p2p.log 2>&1; echo bench_n2=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench26_n1.log 2>&1; echo bench_n1=$?
tail -n 3 gpurun_out/pytest26_multi.log
for f in bench26_n4_p2p bench26_n4_nccl bench26_n2_p2p bench26_n1; do tail -n 1 gpurun_out/$f.log | cut -c 1-200; done
for T in p2p nccl; do
AMG_TRANSPORT=$T timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29518 \
    tools/level_breakdown.py --gpus 4 > gpurun_out/levels26_n4_$T.log 2>&1; echo lev_n4_$T=$?
done
timeout 600 python tools/level_breakdown.py > gpurun_out/levels26_n1.log 2>&1; echo lev_n1=$?
grep total_ms gpurun_out/levels26_*.log | cut -c 1-300
