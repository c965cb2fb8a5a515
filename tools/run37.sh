set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build37.log 2>&1; echo build=$?
tail -2 gpurun_out/build37.log
timeout 900 python tools/op_sweep.py --config C3 --levels 0 --ops 0 --reps 10 > gpurun_out/sweep37.jsonl 2> gpurun_out/sweep37.err; echo sweep=$?
tail -4 gpurun_out/sweep37.jsonl; tail -3 gpurun_out/sweep37.err
rm -f gpurun_out/tune_C3_37.txt
AMG_VERBOSE=1 AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C3_37.txt timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench37_c3.log 2>&1; echo c3=$?
AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C3_37.txt timeout 900 python tools/level_breakdown.py > gpurun_out/levels37.log 2>&1; echo lev=$?
tail -n 1 gpurun_out/bench37_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['vcycle_GBps'], d['roofline'], [ (k['layout'], k['kernel'],k['G'],k['U'],k['tuned_us']) for k in d['config']['level_kernels']], d['clocks'])"
tail -2 gpurun_out/levels37.log
timeout 1800 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/parity37.log 2>&1; echo parity=$?
tail -5 gpurun_out/parity37.log
