set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build39.log 2>&1; echo build=$?
timeout 900 python tools/op_sweep.py --config C3 --format 6 --levels 0,1 --ops 0,1,2 --reps 10 > gpurun_out/sweep39_f6.jsonl 2> gpurun_out/sweep39_f6.err; echo sweep6=$?
timeout 900 python tools/op_sweep.py --config C3 --format 0 --levels 0 --ops 0,1,2 --reps 10 > gpurun_out/sweep39_f0.jsonl 2> gpurun_out/sweep39_f0.err; echo sweep0=$?
grep autotuned gpurun_out/sweep39_f6.jsonl gpurun_out/sweep39_f0.jsonl | cut -c 1-300
export AMG_TUNE_CACHE=$PWD/gpurun_out/tune_C3_39.txt
cp tools/tune_C3_38.txt $AMG_TUNE_CACHE
AMG_GRAPHS=0 timeout 600 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/prof39_plain.log 2>&1; echo plain=$?
AMG_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "solve/" \
   --kernel-name-base demangled -k 'regex:EpiCheb<\(bool\)0>' -c 2 \
   -o gpurun_out/prof39 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/ncu39_full.log 2>&1; echo ncu_full=$?
