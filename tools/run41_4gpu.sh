set -x
mkdir -p gpurun_out
export AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C3.txt
cp profiles/tune_C3.txt $AMG_TUNE_CACHE
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build41.log 2>&1; echo build=$?
for k in 0 120; do AMG_L2_KEEP_MB=$k timeout 600 python tools/level_breakdown.py > gpurun_out/levels41_keep$k.log 2>&1; echo lev$k=$?; tail -1 gpurun_out/levels41_keep$k.log; done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/bench41_c3_n4.log 2>&1; echo c3n4=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench41_c3_n2.log 2>&1; echo c3n2=$?
for f in bench41_c3_n4 bench41_c3_n2; do tail -n 1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d.get('setup_phases'), d['roofline']['frac'], d['clocks'])"; done
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29513 tools/level_breakdown.py --gpus 4 > gpurun_out/levels41_n4.log 2>&1; echo lev4=$?
cat gpurun_out/levels41_n4.log | grep rank
unset AMG_TUNE_CACHE
export AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C5s.txt
timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29514 bench.py --gpus 2 --config C5s --steps 5 --warmup 3 > gpurun_out/bench41_c5s_n2.log 2>&1; echo c5s2=$?
timeout 1500 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29515 bench.py --gpus 4 --config C5s --steps 5 --warmup 3 > gpurun_out/bench41_c5s_n4.log 2>&1; echo c5s4=$?
timeout 900 python bench.py --config C5s --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench41_c5s_n1.log 2>&1; echo c5s1=$?
for f in bench41_c5s_n1 bench41_c5s_n2 bench41_c5s_n4; do tail -n 1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d.get('setup_phases'), d['config']['dofs'], d['clocks'])"; done
unset AMG_TUNE_CACHE
timeout 1800 python -m pytest tests/test_gpu_multi.py -x -q -k "4" > gpurun_out/pytest41.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest41.log
free -g | head -2
