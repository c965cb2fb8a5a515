# 1 GPU: tail-split SELL-VI parity + level-0 timing (default rule vs no split), C3 and C4 benches
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build48.log 2>&1; echo build=$?
tail -n 1 gpurun_out/build48.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/parity48.log 2>&1; echo parity=$?
tail -n 3 gpurun_out/parity48.log
for lp in def 0; do
  if [ $lp = def ]; then unset AMG_SELLVI_PARTS; else export AMG_SELLVI_PARTS=$lp; fi
  timeout 600 python tools/op_sweep.py --config C3 --levels 0 --ops 0 --reps 10 > gpurun_out/sweep48_$lp.jsonl 2> gpurun_out/sweep48_$lp.err; echo sweep$lp=$?
  python tools/sweep_summary.py gpurun_out/sweep48_$lp.jsonl | head -3
done
unset AMG_SELLVI_PARTS
for cfg in C3 C4; do
  timeout 1500 python bench.py --config $cfg --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench48_$cfg.log 2>&1; echo $cfg=$?
  tail -n 1 gpurun_out/bench48_$cfg.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$cfg', d['value'], d['iters'], d['s_per_iter'], d['vcycle_GBps'], d['roofline']['achieved'], d['roofline']['frac'], d['config']['level_kernels'][0].get('sellvi_parts'), d['clocks'])"
done
