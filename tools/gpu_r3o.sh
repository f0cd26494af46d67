# shape-keyed priors (arena mean, look-ahead fraction): full GPU suite, bench lines of all configs,
# the reference arm on c5, launch list of the c5 bench command
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/o_test_all.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/o_test_all.log
timeout 900 python bench.py --impl reference > gpurun_out/o_bench_ref_c5.log 2>&1
for c in c5 c4 c2 c3 c1; do timeout 1200 python bench.py --config $c > gpurun_out/o_bench_$c.log 2>&1; tail -1 gpurun_out/o_bench_$c.log | cut -c1-330; done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/o_launches_c5_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/o_ncu_bench_c5.log 2>&1
