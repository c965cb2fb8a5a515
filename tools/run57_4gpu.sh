# 4-GPU: P2P fix for split SELL-VI slices (warps with boundary items wait) — P2P multi-GPU tests, C3 at 2 and 4 GPUs
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build57.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_multi.py -q -k "p2p or shared" > gpurun_out/pytest57.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest57.log
grep FAILED gpurun_out/pytest57.log | head
for n in 2 4; do
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2958$n bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench57_c3_n$n.log 2>&1; echo c3n$n=$?
  tail -n 1 gpurun_out/bench57_c3_n$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 n$n', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['roofline']['frac'], d['e2e']['value'], d['clocks'])"
done
