set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build35.log 2>&1; echo build=$?
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "kernel_configs or d16 or vcycle" > gpurun_out/parity35.log 2>&1; echo parity=$?
tail -3 gpurun_out/parity35.log
timeout 900 python tools/op_sweep.py --config C3 --levels 0,1 --ops 0 --reps 10 > gpurun_out/sweep35.jsonl 2> gpurun_out/sweep35.err; echo sweep=$?
rm -f gpurun_out/tune_C3_35.txt
AMG_VERBOSE=1 AMG_TUNE_CACHE=gpurun_out/tune_C3_35.txt timeout 900 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench35_c3.log 2>&1; echo c3=$?
AMG_VERBOSE=1 AMG_TUNE_CACHE=gpurun_out/tune_C3_35.txt timeout 900 python tools/level_breakdown.py > gpurun_out/levels35.log 2>&1; echo lev=$?
tail -n 1 gpurun_out/bench35_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['iters'], d['s_per_iter'], d['setup_s'], d['roofline'], [ (k['kernel'],k['G'],k['U'],k['tuned_us']) for k in d['config']['level_kernels']], d['clocks'])"
cat gpurun_out/levels35.log | tail -2
python tools/sweep_summary.py gpurun_out/sweep35.jsonl | head -30
