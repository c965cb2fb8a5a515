# 1 GPU: ncu --set full of the L3 level-0 SELL-VI step (roofline traffic for the L3 bench line) and launch list
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build54.log 2>&1; echo build=$?
AMG_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "solve/" \
   --kernel-name-base demangled -k 'regex:k_sellvi.*EpiCheb<\(bool\)0>' -c 2 \
   -o gpurun_out/prof54 python tools/profile_solve.py --config L3 --warm 1 --solves 1 > gpurun_out/ncu54_full.log 2>&1; echo ncu_full=$?
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "solve/" --csv --log-file gpurun_out/launches54.csv \
   python tools/profile_solve.py --config L3 --warm 1 --solves 1 > gpurun_out/ncu54_list.log 2>&1; echo ncu_list=$?
python tools/summarize_launches.py gpurun_out/launches54.csv --solve-only > gpurun_out/launches54_summary.txt 2>&1
head -8 gpurun_out/launches54_summary.txt
