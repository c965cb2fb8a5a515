set -x
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench33_graph.log 2>&1; echo g=$?
AMG_GRAPHS=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench33_nograph.log 2>&1; echo ng=$?
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench33_graph2.log 2>&1; echo g2=$?
timeout 600 python tools/level_breakdown.py > gpurun_out/levels33_n1.log 2>&1; echo lev=$?
for f in bench33_graph bench33_nograph bench33_graph2; do tail -n 1 gpurun_out/$f.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$f', d['value'], d['s_per_iter'], d['roofline']['launch_ms'], d['clocks'])"; done
cat gpurun_out/levels33_n1.log
