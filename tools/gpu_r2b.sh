# long-row path: correctness (oracle parity incl. forced-low thresholds, reference goldens),
# then the A/B of full IMM runs against the previous build (variants/var_base.so)
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_longrow.py tests/test_gpu_parity.py tests/test_gpu_integration.py tests/test_gpu_configs.py tests/test_gpu_fullsize.py tests/test_gpu_golden.py -x -q > gpurun_out/b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/b_tests.log
for c in c5 c4 c2; do
  echo "== base $c"; IMMX_B200_LIB=$PWD/variants/var_base.so timeout 600 python tools/run_config.py --config $c --reps 2 2>&1 | grep "rep 1" | sed 's/ seeds.*//; s/phases.*ratio/ratio/'
  for L in 0 1024 2048 4096 8192; do
    echo "== L=$L $c"; IMMX_LONG_MIN=$L timeout 600 python tools/run_config.py --config $c --reps 2 2>&1 | grep "rep 1" | sed 's/ seeds.*//; s/phases.*ratio/ratio/'
  done
  for L in 1024 2048; do
    echo "== lr8 L=$L $c"; IMMX_B200_LIB=$PWD/variants/var_lr8.so IMMX_LONG_MIN=$L timeout 600 python tools/run_config.py --config $c --reps 2 2>&1 | grep "rep 1" | sed 's/ seeds.*//; s/phases.*ratio/ratio/'
  done
done > gpurun_out/b_ab.log 2>&1
