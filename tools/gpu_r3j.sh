# look-ahead first guess (pilot / remembered fraction): tests, the c5 reference golden on the
# device, A/B of the c5 and c4 bench lines
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lookahead.py -x -q -m gpu > gpurun_out/j_test_la.log 2>&1; echo "la rc=$?"; tail -3 gpurun_out/j_test_la.log
timeout 1800 python -m pytest tests/test_gpu_configs.py -x -q -m gpu -k c5 > gpurun_out/j_test_c5.log 2>&1; echo "c5 rc=$?"; tail -3 gpurun_out/j_test_c5.log
for c in c5 c4 c2; do
  timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/j_bench_$c.log 2>&1; tail -1 gpurun_out/j_bench_$c.log | cut -c1-330
  IMMX_LA_PILOT=0 timeout 900 python bench.py --config $c --no-cpu-baseline > gpurun_out/j_bench_${c}_nopilot.log 2>&1; tail -1 gpurun_out/j_bench_${c}_nopilot.log | cut -c1-330
done
IMMX_DEBUG_TIERS=1 timeout 600 python tools/run_config.py --config c5 --reps 2 > gpurun_out/j_tiers_c5.log 2>&1
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/j_test_all.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/j_test_all.log
