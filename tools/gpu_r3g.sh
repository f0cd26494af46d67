# min chunk 32 + vectorised argmax / clears: tests, then select phase main vs chunk1 variant
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_lookahead.py tests/test_gpu_select_filter.py tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_hybrid.py tests/test_gpu_lt.py tests/test_cli.py -m gpu -x -q > gpurun_out/g_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g_tests.log
tail -3 gpurun_out/g_tests.log
run() { # name config env...
  local name=$1 cfg=$2; shift 2
  env "$@" IMMX_DEBUG_PHASES=1 timeout 600 python tools/run_config.py --config $cfg --reps 3 > gpurun_out/g_${cfg}_$name.log 2>&1
  echo "$cfg $name: $(grep 'rep 2' gpurun_out/g_${cfg}_$name.log | sed -e "s/.*'estimate': \([0-9.]*\).*'select': \([0-9.]*\).*/estimate \1 select \2/") | $(grep 'rounds:' gpurun_out/g_${cfg}_$name.log | tail -1 | sed 's/.*rounds: //')"
}
for c in c3 c1 c2 c4 c5; do
run main $c A=1
run chunk1 $c IMMX_B200_LIB=$PWD/variants/var_chunk1.so
done
