# 4-GPU: C3 after the SELL-VI rule fix (long rows need a shared-memory table), 2/4-GPU benches, C5s weak
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build45.log 2>&1; echo build=$?
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29531 tools/level_breakdown.py --gpus 4 > gpurun_out/lev45_n4.log 2>&1; echo lev4=$?
grep rank gpurun_out/lev45_n4.log | cut -c1-330
for n in 4 2; do
  timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port 2953$n bench.py --gpus $n --steps 5 --warmup 3 > gpurun_out/bench45_c3_n$n.log 2>&1; echo c3n$n=$?
  tail -n 1 gpurun_out/bench45_c3_n$n.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 n$n', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['roofline']['frac'], d['clocks'])"
done
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29535 bench.py --gpus 4 --config C5s --steps 5 --warmup 3 > gpurun_out/bench45_c5s_n4.log 2>&1; echo c5s4=$?
tail -n 1 gpurun_out/bench45_c5s_n4.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5s n4', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['config']['dofs'], d['clocks'])"
timeout 1800 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest45.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest45.log
