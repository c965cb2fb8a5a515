set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/smoke8.log 2>&1; echo smoke=$?
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest8.log 2>&1; echo pytest=$?
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench8.log 2>&1; echo bench=$?
timeout 600 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/prof8_plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches8.csv \
   python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/ncu8_list.log 2>&1; echo ncu_list=$?
timeout 900 ncu --set full --clock-control none --import-source on -k regex:EpiCheb -s 40 -c 6 \
   -o gpurun_out/prof8 python tools/profile_solve.py --config C3 --warm 1 --solves 1 > gpurun_out/ncu8_full.log 2>&1; echo ncu_full=$?
tail -n 3 gpurun_out/pytest8.log; tail -n 2 gpurun_out/smoke8.log; tail -n 1 gpurun_out/bench8.log
