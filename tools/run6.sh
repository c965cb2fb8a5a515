set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke6.log 2>&1; echo smoke=$?
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest6.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench6.log 2>&1; echo bench=$?
AMG_GRAPHS=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench6_nograph.log 2>&1; echo bench_ng=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config C2 --no-cpu-baseline > gpurun_out/bench6_c2.log 2>&1; echo bench_c2=$?
AMG_GRAPHS=0 timeout 600 python bench.py --steps 5 --warmup 3 --config C2 --no-cpu-baseline > gpurun_out/bench6_c2_ng.log 2>&1; echo bench_c2ng=$?
tail -n 3 gpurun_out/pytest6.log; tail -n 2 gpurun_out/smoke6.log
