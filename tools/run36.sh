set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build36.log 2>&1; echo build=$?
timeout 900 python tools/op_sweep.py --config C3 --levels 0 --ops 0 --reps 10 > gpurun_out/sweep36.jsonl 2> gpurun_out/sweep36.err; echo sweep=$?
python tools/sweep_summary.py gpurun_out/sweep36.jsonl | head -12
export AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C3_36.txt
cp tools/tune_vi_seed.txt $AMG_TUNE_CACHE
AMG_GRAPHS=0 timeout 600 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/prof36_plain.log 2>&1; echo plain=$?
AMG_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "solve/" \
   --kernel-name-base demangled -k 'regex:EpiCheb<\(bool\)0>' -c 2 \
   -o gpurun_out/prof36 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/ncu36_full.log 2>&1; echo ncu_full=$?
ncu -i gpurun_out/prof36.ncu-rep --page details --csv > gpurun_out/prof36_details.csv 2>&1; echo det=$?
