# GPU-box task runner (one script instead of one per gpurun call).
#
#   gpurun --timeout S -- 'bash tools/gpu.sh TAG TASK [TASK ...]'
#
# Every task writes gpurun_out/<TAG>_<task>.log (merged back by gpurun) and prints a one-line summary.
# Tasks:
#   build            build the library + oracle (in-tree)
#   smoke            __graft_entry__.smoke()
#   pytest           every -m gpu test (1 GPU; multi-GPU tests skip themselves)
#   pytest_multi     tests/test_gpu_multi.py (needs >= 2 GPUs)
#   bench[:CFG]      bench.py at 1 GPU (default workload C3), 5 steps, 3 warm-up
#   benchN:N[:CFG]   bench.py under torchrun at N GPUs
#   ref              bench.py --impl reference --steps 2 --warmup 1
#   launches[:CFG]   ncu launch list (gpu__time_duration.sum) of one solve
#   ncu[:CFG[:RE]]   ncu --set full of the kernels matching RE (default: the level-0 Chebyshev step)
#   kmetrics[:CFG]   ncu per-kernel DRAM bytes / duration / L1 / occupancy over one solve (tools/ncu_kernels.py)
#   sanitize         compute-sanitizer memcheck / racecheck / synccheck on C1 and C2 solves
#   sweep[:CFG]      tools/op_sweep.py kernel sweep of the level operators
set -x
mkdir -p gpurun_out
TAG=$1; shift
# the bench reads the committed tuning cache (profiles/tune_<cfg>.txt) and never writes it
summ() { python - "$@" <<'EOF'
import json, sys
try:
    d = json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
except Exception as e:  # noqa: BLE001
    print("no json:", e); sys.exit(0)
keys = ["impl", "value", "unit", "iters", "s_per_iter", "solve_s", "setup_s", "vcycle_GBps", "gpu_launches"]
print({k: d.get(k) for k in keys if k in d})
for k in ("roofline", "e2e", "cpu_baseline", "clocks"):
    if k in d:
        print(k, json.dumps(d[k])[:400])
EOF
}
for T in "$@"; do
  IFS=: read -r name a1 a2 <<< "$T"
  log=gpurun_out/${TAG}_${name}${a1:+_$a1}${a2:+_$a2}.log
  case $name in
    build) python -c "import __graft_entry__ as g; g.build()" > $log 2>&1; echo build=$? ;;
    smoke) python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $log 2>&1; echo smoke=$?; tail -n 1 $log ;;
    pytest) timeout 2400 python -m pytest tests -m gpu -q -rs > $log 2>&1; echo pytest=$?; tail -n 3 $log; grep -E "FAILED|Error" $log | head ;;
    pytest_multi) timeout 2400 python -m pytest tests/test_gpu_multi.py -q -rs ${a1:+-k $a1} > $log 2>&1; echo pytest_multi=$?; tail -n 3 $log; grep FAILED $log | head ;;
    bench) timeout 1200 python bench.py --config ${a1:-C3} --steps 5 --warmup 3 > $log 2>&1; echo bench=$?; summ $log ;;
    benchN) timeout 1200 python -m torch.distributed.run --nnodes=1 --nproc-per-node $a1 --master-addr 127.0.0.1 --master-port 2960$a1 \
              bench.py --gpus $a1 --config ${a2:-C3} --steps 5 --warmup 3 --no-cpu-baseline > $log 2>&1; echo benchN=$?; summ $log ;;
    ref) timeout 1800 python bench.py --impl reference --steps 2 --warmup 1 > $log 2>&1; echo ref=$?; summ $log ;;
    launches) timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --nvtx --nvtx-include "solve/" --csv \
                --log-file gpurun_out/${TAG}_launches_${a1:-C3}.csv python tools/profile_solve.py --config ${a1:-C3} --warm 1 --solves 1 > $log 2>&1
              echo launches=$?; python tools/summarize_launches.py gpurun_out/${TAG}_launches_${a1:-C3}.csv --solve-only | head -16 ;;
    ncu) AMG_GRAPHS=0 timeout 1200 ncu --set full --clock-control none --import-source on --nvtx --nvtx-include "solve/" \
           --kernel-name-base demangled -k "regex:${a2:-k_sellvi.*EpiCheb<\(bool\)0>}" -c 2 \
           -o gpurun_out/${TAG}_${a1:-C3} python tools/profile_solve.py --config ${a1:-C3} --warm 1 --solves 1 > $log 2>&1; echo ncu=$? ;;
    kmetrics) timeout 1500 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__throughput.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread,launch__grid_size \
                --clock-control none --nvtx --nvtx-include "solve/" --csv --log-file gpurun_out/${TAG}_kmetrics_${a1:-C3}.csv \
                python tools/profile_solve.py --config ${a1:-C3} --warm 1 --solves 1 > $log 2>&1; echo kmetrics=$?
              python tools/ncu_kernels.py gpurun_out/${TAG}_kmetrics_${a1:-C3}.csv --md gpurun_out/${TAG}_kmetrics_${a1:-C3}.md | head -24 ;;
    sanitize) for cfg in C1 C2; do for tool in memcheck racecheck synccheck; do
                timeout 1200 compute-sanitizer --tool $tool --error-exitcode 7 python tools/profile_solve.py --config $cfg --warm 0 --solves 1 \
                  > gpurun_out/${TAG}_san_${cfg}_${tool}.log 2>&1; echo san_${cfg}_${tool}=$?; tail -n 2 gpurun_out/${TAG}_san_${cfg}_${tool}.log; done; done ;;
    sweep) timeout 1200 python tools/op_sweep.py --config ${a1:-C3} > $log 2>&1; echo sweep=$?; tail -n 30 $log ;;
    *) echo "unknown task $name" ;;
  esac
done
