# 1 GPU: L-shape with the paper's data (library rhs = 2): smoke, all GPU tests, L3 bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke52.log 2>&1; echo smoke=$?
tail -n 1 gpurun_out/smoke52.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest52.log 2>&1; echo pytest=$?
tail -n 3 gpurun_out/pytest52.log
cp gpurun_out/tune_L3.txt profiles/tune_L3.txt 2>/dev/null
timeout 1800 python bench.py --config L3 --steps 5 --warmup 3 > gpurun_out/bench52_L3.log 2>&1; echo L3=$?
tail -n 1 gpurun_out/bench52_L3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('L3', d['value'], d['iters'], d['s_per_iter'], d['vcycle_GBps'], d['roofline']['achieved'], d['roofline']['frac'], d['cpu_baseline']['value'], d['e2e'], d['config']['opc'], d['config']['levels'], d['clocks'], d['config'].get('t_gen_s'), d['config'].get('t_setup_s'))"
grep -i "Traceback" -A5 gpurun_out/bench52_L3.log | head -8
