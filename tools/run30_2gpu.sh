set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "ring or paper or fcg or coarse_cg" > gpurun_out/pytest30_new.log 2>&1; echo pytest_new=$?; tail -3 gpurun_out/pytest30_new.log
timeout 1200 python -m pytest tests/test_gpu_multi.py -x -q > gpurun_out/pytest30_multi.log 2>&1; echo pytest_multi=$?; tail -3 gpurun_out/pytest30_multi.log; grep -E "^E  " gpurun_out/pytest30_multi.log | head -5
AMG_TUNE_CACHE=$PWD/gpurun_out/tune_R3.txt timeout 1200 python bench.py --config R3 --steps 3 --warmup 3 > gpurun_out/bench30_r3.log 2>&1; echo bench_r3=$?; tail -1 gpurun_out/bench30_r3.log | cut -c 1-300
