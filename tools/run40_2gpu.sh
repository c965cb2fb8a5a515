set -x
mkdir -p gpurun_out
export AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C3.txt
rm -f $AMG_TUNE_CACHE
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build40.log 2>&1; echo build=$?
tail -1 gpurun_out/build40.log
timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench40_c3_n1.log 2>&1; echo c3n1=$?
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/bench40_c3_n2.log 2>&1; echo c3n2=$?
for f in bench40_c3_n1 bench40_c3_n2; do tail -n 1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d.get('setup_phases'), d['roofline']['frac'], d['clocks'])"; done
unset AMG_TUNE_CACHE
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/pytest40.log 2>&1; echo pytest=$?
tail -3 gpurun_out/pytest40.log
