set -x
mkdir -p gpurun_out
run() { timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port $1 tools/debug/dist_pcg.py > gpurun_out/dbg29_$2.log 2>&1; echo $2=$?; }
DBG_VCYCLE_FIRST=1 AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=nccl run 29521 nccl_vf
DBG_VCYCLE_FIRST=1 AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=p2p run 29522 p2p_vf
DBG_VCYCLE_FIRST=1 AMG_REPLICATE_NNZ=100000 AMG_TRANSPORT=p2p AMG_P2P_INTERIOR=0 run 29523 p2p_vf_noorder
grep -h "iters" gpurun_out/dbg29_*.log
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "world-2 or paper" > gpurun_out/pytest29.log 2>&1; echo pytest=$?; tail -3 gpurun_out/pytest29.log
