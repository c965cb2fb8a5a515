# 4-GPU: L-shape (NEXT-4) multi-GPU parity (2 and 4 GPUs, P2P and NCCL) and L3 benches at 2 and 4 GPUs
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build53.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -k "case3-100000 or paper_experiment" > gpurun_out/pytest53.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest53.log
for n in 2 4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2954$n bench.py --gpus $n --config L3 --steps 5 --warmup 3 > gpurun_out/bench53_L3_n$n.log 2>&1; echo L3n$n=$?
  tail -n 1 gpurun_out/bench53_L3_n$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('L3 n$n', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['roofline']['frac'], d['clocks'])"
done
