# 4-GPU, final tree: every multi-GPU test (2 and 4 GPUs, P2P and NCCL), C3 at 2 and 4 GPUs, C5s weak at 2 and 4
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build56.log 2>&1; echo build=$?
timeout 1800 python -m pytest tests/test_gpu_multi.py -q > gpurun_out/pytest56.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest56.log
for n in 2 4; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2956$n bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench56_c3_n$n.log 2>&1; echo c3n$n=$?
  tail -n 1 gpurun_out/bench56_c3_n$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 n$n', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
done
for n in 2 4; do
  timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2957$n bench.py --gpus $n --config C5s --steps 5 --warmup 3 > gpurun_out/bench56_c5s_n$n.log 2>&1; echo c5sn$n=$?
  tail -n 1 gpurun_out/bench56_c5s_n$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5s n$n', d['value'], d['iters'], d['s_per_iter'], d['config']['dofs'], d['clocks'])"
done
