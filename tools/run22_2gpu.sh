set -x
mkdir -p gpurun_out
for T in nccl p2p; do
AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=$T timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 \
    tools/debug/dist_vcycle.py > gpurun_out/dbg22_$T.log 2>&1; echo dbg_$T=$?
done
grep max_levels gpurun_out/dbg22_*.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest22_multi.log 2>&1; echo pytest_multi=$?
tail -n 3 gpurun_out/pytest22_multi.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 \
    bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench22_n2_p2p.log 2>&1; echo bench_n2=$?
AMG_TRANSPORT=nccl timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29517 \
    bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench22_n2_nccl.log 2>&1; echo bench_n2_nccl=$?
for f in bench22_n2_p2p bench22_n2_nccl; do tail -n 1 gpurun_out/$f.log | cut -c 1-200; done
