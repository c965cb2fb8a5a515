set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build42.log 2>&1; echo build=$?
tail -1 gpurun_out/build42.log
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity42.log 2>&1; echo parity=$?
tail -3 gpurun_out/parity42.log
for cfg in C3 C4 C5 R3 R4; do
  rm -f gpurun_out/tune_$cfg.txt
  extra="--no-cpu-baseline"; [ $cfg = C3 ] && extra=""
  AMG_TUNE_CACHE=$PWD/gpurun_out/tune_$cfg.txt timeout 1500 python bench.py --config $cfg --steps 5 --warmup 3 $extra > gpurun_out/bench42_$cfg.log 2>&1; echo $cfg=$?
  tail -n 1 gpurun_out/bench42_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['vcycle_GBps'], d.get('vcycle_GBps_plain_csr_equivalent'), d['roofline']['kernel'][:40], d['roofline']['frac'], d.get('cpu_baseline',{}).get('value'), d['clocks'])"
done
