set -x
mkdir -p gpurun_out
free -g | head -2
AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C4.txt timeout 2400 python bench.py --config C4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench24_c4.log 2>&1; echo c4=$?
AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C5.txt timeout 2400 python bench.py --config C5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench24_c5.log 2>&1; echo c5=$?
tail -n 2 gpurun_out/bench24_c4.log | cut -c 1-400; tail -n 2 gpurun_out/bench24_c5.log | cut -c 1-400
