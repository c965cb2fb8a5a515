set -x
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build3.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu3.log 2>&1; echo pytest=$?
for f in 1 2 0; do timeout 600 python bench.py --steps 5 --warmup 3 --format $f --no-cpu-baseline > gpurun_out/bench3_f$f.log 2>&1; echo bench_f$f=$?; done
python tools/profile_solve.py --config C3 --warm 0 --solves 1 --format 1 > gpurun_out/p3_plain1.log 2>&1 && ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled -k "regex:EpiCheb<false>" -s 2 -c 1 -o gpurun_out/prof_cheb_csr2 python tools/profile_solve.py --config C3 --warm 0 --solves 1 --format 1 > gpurun_out/ncu3a.log 2>&1; echo ncu_a=$?
python tools/profile_solve.py --config C3 --warm 0 --solves 1 --format 2 > gpurun_out/p3_plain2.log 2>&1 && ncu --set full --clock-control none --cache-control none --import-source on --kernel-name-base demangled -k "regex:EpiCheb<false>" -s 2 -c 1 -o gpurun_out/prof_cheb_sell2 python tools/profile_solve.py --config C3 --warm 0 --solves 1 --format 2 > gpurun_out/ncu3b.log 2>&1; echo ncu_b=$?
tail -n 3 gpurun_out/pytest_gpu3.log
for f in 1 2 0; do tail -c 600 gpurun_out/bench3_f$f.log; echo; done
