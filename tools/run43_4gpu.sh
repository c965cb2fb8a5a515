# 4-GPU C3 level-1 regression diagnosis: shared vs per-rank setup, SELL-VI off, NCCL transport
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build43.log 2>&1; echo build=$?
timeout 600 python -m pytest tests/test_gpu_parity.py -q -k "sellvi" > gpurun_out/parity43.log 2>&1; echo parity=$?; tail -2 gpurun_out/parity43.log
export AMG_TUNE_CACHE=$PWD/gpurun_out/tune43.txt
run() {  # name, extra env..., then args
  name=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29521 tools/level_breakdown.py --gpus 4 $LBARGS > gpurun_out/lev43_$name.log 2>&1; echo $name=$?
  grep rank gpurun_out/lev43_$name.log | cut -c1-400
}
LBARGS="" run shared X=1
LBARGS="--per-rank-setup" run perrank X=1
LBARGS="" run nosellvi AMG_SELLVI=0
LBARGS="" run nccl AMG_TRANSPORT=nccl
