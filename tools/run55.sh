# 1 GPU, round-end check of the final tree: smoke, every -m gpu test, default bench (C3, + reference arm), L3 bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke55.log 2>&1; echo smoke=$?
tail -n 1 gpurun_out/smoke55.log
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/pytest55.log 2>&1; echo pytest=$?
tail -n 3 gpurun_out/pytest55.log
timeout 900 python bench.py > gpurun_out/bench55_default.log 2>&1; echo bench=$?
tail -n 1 gpurun_out/bench55_default.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('default', d['config']['workload'][:40], d['value'], d['iters'], d['steps'], d['warmup'], d['vcycle_GBps'], d['roofline']['frac'], d['roofline']['traffic'], d['e2e']['value'], d['cpu_baseline']['value'], d['clocks'], d['gpu_launches'])"
timeout 1800 python bench.py --config L3 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench55_L3.log 2>&1; echo L3=$?
tail -n 1 gpurun_out/bench55_L3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('L3', d['value'], d['iters'], d['vcycle_GBps'], d['roofline']['achieved'], d['roofline']['frac'], d['roofline']['traffic'], d['clocks'])"
