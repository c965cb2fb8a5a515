# 1 GPU: split-slice SELL-VI (parts) parity, level-0 K0 timing per parts, C3 bench
set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/build47.log 2>&1; echo build=$?
tail -n 1 gpurun_out/build47.log
timeout 1500 python -m pytest tests/test_gpu_parity.py -q > gpurun_out/parity47.log 2>&1; echo parity=$?
tail -n 3 gpurun_out/parity47.log
for lp in 0 1 2; do
  AMG_SELLVI_PARTS=$lp timeout 600 python tools/op_sweep.py --config C3 --levels 0 --ops 0 --reps 10 > gpurun_out/sweep47_lp$lp.jsonl 2> gpurun_out/sweep47_lp$lp.err; echo sweep$lp=$?
  python tools/sweep_summary.py gpurun_out/sweep47_lp$lp.jsonl | head -5
done
