set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke9.log 2>&1; echo smoke=$?
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest9.log 2>&1; echo pytest=$?
timeout 900 python tools/op_sweep.py --config C3 --levels 0,1,2 --ops 0,1,2 > gpurun_out/opsweep9.jsonl 2>&1; echo sweep=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench9.log 2>&1; echo bench=$?
AMG_GRAPHS=0 timeout 600 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/prof9_plain.log 2>&1 && \
AMG_GRAPHS=0 timeout 900 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "solve/" \
   --kernel-name-base demangled -k regex:"EpiCheb<0>" -c 3 \
   -o gpurun_out/prof9 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/ncu9_full.log 2>&1; echo ncu_full=$?
tail -n 3 gpurun_out/pytest9.log; tail -n 2 gpurun_out/smoke9.log; tail -n 1 gpurun_out/bench9.log | cut -c 1-600
