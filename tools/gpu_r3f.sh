# look-ahead sampling + LUT 16/12 default: tests, then per-config runs (look-ahead on / off)
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_select_filter.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_integration.py tests/test_gpu_hybrid.py tests/test_gpu_lt.py -m gpu -x -q > gpurun_out/f_tests.log 2>&1; echo "rc=$?" >> gpurun_out/f_tests.log
tail -3 gpurun_out/f_tests.log
for c in c5 c4 c2 c3 c1; do
for la in 0 1.25; do
IMMX_LOOKAHEAD=$la IMMX_DEBUG_TIERS=0 timeout 600 python tools/run_config.py --config $c --reps 3 > gpurun_out/f_${c}_la$la.log 2>&1
echo "$c lookahead=$la: $(grep 'rep 2' gpurun_out/f_${c}_la$la.log | sed -e 's/ ratio.*edges/ edges/' -e 's/ seeds.*//')"
done
done
