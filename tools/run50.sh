# 1 GPU, round-end evidence after the SELL-VI tail split: smoke, all -m gpu tests, C3 bench (+ reference arm), launch list and
# ncu --set full of the level-0 SELL-VI step, C4 ncu of its SELL-VI step
set -x
mkdir -p gpurun_out
export AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C3.txt
rm -f $AMG_TUNE_CACHE
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke50.log 2>&1; echo smoke=$?
tail -n 1 gpurun_out/smoke50.log
timeout 2400 python -m pytest tests -m gpu -q > gpurun_out/pytest50.log 2>&1; echo pytest=$?
tail -n 3 gpurun_out/pytest50.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench50_c3.log 2>&1; echo bench=$?
tail -n 1 gpurun_out/bench50_c3.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3', d['value'], d['iters'], d['s_per_iter'], d['vcycle_GBps'], d['roofline'], d['e2e'], d['cpu_baseline'], d['clocks'], d['gpu_launches'])"
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench50_ref.log 2>&1; echo ref=$?
tail -n 1 gpurun_out/bench50_ref.log | cut -c 1-400
AMG_GRAPHS=0 timeout 600 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/prof50_plain.log 2>&1; echo plain=$?
AMG_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "solve/" \
   --kernel-name-base demangled -k 'regex:k_sellvi.*EpiCheb<\(bool\)0>' -c 2 \
   -o gpurun_out/prof50 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/ncu50_full.log 2>&1; echo ncu_full=$?
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "solve/" --csv --log-file gpurun_out/launches50.csv \
   python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/ncu50_list.log 2>&1; echo ncu_list=$?
python tools/summarize_launches.py gpurun_out/launches50.csv --solve-only | head -12
