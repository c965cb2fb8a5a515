set -x
mkdir -p gpurun_out
export AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C3.txt
rm -f $AMG_TUNE_CACHE
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke25.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest25.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench25_paper.log 2>&1; echo bench=$?
timeout 900 python bench.py --steps 5 --warmup 3 --problem manufactured --no-cpu-baseline > gpurun_out/bench25_manu.log 2>&1; echo bench_manu=$?
AMG_GRAPHS=0 timeout 600 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/prof25_plain.log 2>&1 && \
AMG_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "solve/" \
   --kernel-name-base demangled -k 'regex:EpiCheb<\(bool\)0>' -c 3 \
   -o gpurun_out/prof25 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/ncu25_full.log 2>&1; echo ncu_full=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "solve/" --csv --log-file gpurun_out/launches25.csv \
   python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/ncu25_list.log 2>&1; echo ncu_list=$?
tail -n 3 gpurun_out/pytest25.log; tail -n 2 gpurun_out/smoke25.log; tail -n 1 gpurun_out/bench25_paper.log | cut -c 1-300; cat $AMG_TUNE_CACHE
