set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build38.log 2>&1; echo build=$?
timeout 900 python tools/op_sweep.py --config C3 --levels 0 --ops 0 --reps 10 > gpurun_out/sweep38.jsonl 2> gpurun_out/sweep38.err; echo sweep=$?
tail -4 gpurun_out/sweep38.jsonl; tail -3 gpurun_out/sweep38.err
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "sellvi or 6 or kernel_configs" > gpurun_out/parity38.log 2>&1; echo parity=$?
tail -3 gpurun_out/parity38.log
rm -f gpurun_out/tune_C3_38.txt
AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C3_38.txt timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench38_c3.log 2>&1; echo c3=$?
AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C3_38.txt timeout 900 python tools/level_breakdown.py > gpurun_out/levels38.log 2>&1; echo lev=$?
tail -n 1 gpurun_out/bench38_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['iters'], d['s_per_iter'], d['vcycle_GBps'], d['roofline']['launch_ms'], d['roofline']['frac'], d['clocks'])"
tail -1 gpurun_out/levels38.log
