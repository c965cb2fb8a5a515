# 4-GPU: L3 at 2 and 4 GPUs after the P2P split-slice fix
set -x
mkdir -p gpurun_out
for n in 4 2; do
  timeout 420 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2959$n bench.py --gpus $n --config L3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench58_L3_n$n.log 2>&1; echo L3n$n=$?
  tail -n 1 gpurun_out/bench58_L3_n$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('L3 n$n', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['roofline']['frac'], d['clocks'])"
done
