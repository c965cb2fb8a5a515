# 1 GPU: tail split on multi-GPU-share-sized cubes (p=3, n=60 ≈ a 4-GPU share of C3, n=76 ≈ a 2-GPU share)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build49.log 2>&1; echo build=$?
for n in 60 76; do
for lp in def 0; do
  if [ $lp = def ]; then unset AMG_SELLVI_PARTS; else export AMG_SELLVI_PARTS=$lp; fi
  timeout 600 python tools/op_sweep.py --config C3 --n $n --levels 0 --ops 0 --reps 20 > gpurun_out/sweep49_n${n}_$lp.jsonl 2> gpurun_out/sweep49_n${n}_$lp.err; echo sweep_n${n}_$lp=$?
  python tools/sweep_summary.py gpurun_out/sweep49_n${n}_$lp.jsonl | head -3
done
done
unset AMG_SELLVI_PARTS
timeout 1500 python bench.py --config C3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench49_C3.log 2>&1; echo C3=$?
tail -n 1 gpurun_out/bench49_C3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('C3', d['value'], d['iters'], d['s_per_iter'], d['vcycle_GBps'], d['roofline']['achieved'], d['roofline']['frac'], d['config']['level_kernels'][0].get('sellvi_parts'), d['clocks'])"
