set -x
mkdir -p gpurun_out
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 tools/debug/dist_pcg.py > gpurun_out/dbg31_$2.log 2>&1; echo $2=$?; }
DBG_GATHER=1 AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=nccl run 29531 nccl_g
DBG_GATHER=1 AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=p2p run 29532 p2p_g
grep -h "iters\|rank" gpurun_out/dbg31_*.log
timeout 600 python -m pytest tests/test_gpu_multi.py -x -q -k "case0 and 2-nccl" > gpurun_out/pytest31.log 2>&1; echo pt=$?; grep -E "^E  " gpurun_out/pytest31.log | head -3
