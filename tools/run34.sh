set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build34.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_multi.py -x -q -k "shared or (p2p and 2 and case1)" > gpurun_out/multi34.log 2>&1; echo multi=$?
tail -3 gpurun_out/multi34.log
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench34_c3_n2.log 2>&1; echo c3n2=$?
timeout 900 python bench.py --config C5s --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench34_c5s_n1.log 2>&1; echo c5s1=$?
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --config C5s --steps 5 --warmup 3 > gpurun_out/bench34_c5s_n2.log 2>&1; echo c5s2=$?
for f in bench34_c3_n2 bench34_c5s_n1 bench34_c5s_n2; do tail -n 1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['config']['dofs'], d['clocks'])"; done
free -g
