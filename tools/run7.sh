set -x
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke7.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest7.log 2>&1; echo pytest=$?
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench7.log 2>&1; echo bench=$?
timeout 600 python bench.py --steps 5 --warmup 3 --config C2 --no-cpu-baseline > gpurun_out/bench7_c2.log 2>&1; echo bench_c2=$?
tail -n 3 gpurun_out/pytest7.log; tail -n 2 gpurun_out/smoke7.log
