mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_longrow.py tests/test_gpu_parity.py -x -q > gpurun_out/g4_tests.log 2>&1; echo "rc=$?" >> gpurun_out/g4_tests.log
for L in 0 512 2048 8192; do
  for c in c2 c4 c5; do
    echo "== L=$L $c"; IMMX_LONG_MIN=$L timeout 600 python tools/run_config.py --config $c --reps 3 2>&1 | grep "rep 2" | sed 's/ seeds.*//'
  done
done > gpurun_out/g4_sweep.log 2>&1
