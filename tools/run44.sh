set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build44.log 2>&1; echo build=$?
tail -1 gpurun_out/build44.log
timeout 1800 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/parity44.log 2>&1; echo parity=$?
tail -3 gpurun_out/parity44.log
for cfg in C4 C3; do
  extra="--no-cpu-baseline"
  AMG_TUNE_CACHE=$PWD/gpurun_out/tune_$cfg.txt timeout 1500 python bench.py --config $cfg --steps 5 --warmup 3 $extra > gpurun_out/bench44_$cfg.log 2>&1; echo $cfg=$?
  tail -n 1 gpurun_out/bench44_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['vcycle_GBps'], d['roofline']['kernel'][:60], d['roofline']['achieved'], d['roofline']['frac'], d['clocks'])"
done
