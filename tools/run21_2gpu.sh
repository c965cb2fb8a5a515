set -x
mkdir -p gpurun_out
for T in nccl p2p; do
AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=$T timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29515 \
    tools/debug/dist_vcycle.py > gpurun_out/dbg21_$T.log 2>&1; echo dbg_$T=$?
AMG_REPLICATE_NNZ=1000000000000 AMG_TRANSPORT=$T timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29516 \
    tools/debug/dist_vcycle.py > gpurun_out/dbg21_${T}_rep.log 2>&1; echo dbg_rep_$T=$?
done
grep max_levels gpurun_out/dbg21_*.log
