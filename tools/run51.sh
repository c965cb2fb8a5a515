# 1 GPU: NEXT-4 L-shape — GPU parity tests, L3 bench (the paper's GPU multipatch case k=96 p=3)
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build51.log 2>&1; echo build=$?
timeout 900 python -m pytest tests/test_gpu_parity.py -q -k lshape > gpurun_out/parity51.log 2>&1; echo parity=$?
tail -n 3 gpurun_out/parity51.log
export AMG_TUNE_CACHE=$PWD/gpurun_out/tune_L3.txt
timeout 1800 python bench.py --config L3 --steps 5 --warmup 3 > gpurun_out/bench51_L3.log 2>&1; echo L3=$?
tail -n 1 gpurun_out/bench51_L3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('L3', d['value'], d['iters'], d['s_per_iter'], d['vcycle_GBps'], d['roofline']['kernel'], d['roofline']['achieved'], d['roofline']['frac'], d['cpu_baseline']['value'], d['config']['opc'], d['config']['levels'], d['clocks'])"
grep -i "error\|Traceback" gpurun_out/bench51_L3.log | head -5
