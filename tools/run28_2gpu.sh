set -x
mkdir -p gpurun_out
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 tools/debug/dist_pcg.py > gpurun_out/dbg28_$2.log 2>&1; echo $2=$?; }
AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=nccl run 29521 nccl
AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=p2p run 29522 p2p
AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=p2p AMG_P2P_INTERIOR=0 run 29523 p2p_noorder
AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=p2p AMG_GRAPHS=0 run 29524 p2p_nograph
AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=nccl AMG_GRAPHS=0 run 29525 nccl_nograph
grep -h "iters" gpurun_out/dbg28_*.log
