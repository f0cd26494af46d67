# short-slab long-row variant for rows in [IMMX_MID_MIN, IMMX_LONG_MIN): tests, sweep of the threshold
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_longrow.py -x -q -m gpu > gpurun_out/t_test_lr.log 2>&1; echo "lr rc=$?"; tail -3 gpurun_out/t_test_lr.log
for c in c4 c5; do
for m in 0 2048 1024 512 256 0 1024; do
  echo "== $c mid_min=$m: $(IMMX_MID_MIN=$m timeout 600 python tools/run_config.py --config $c --reps 3 2>&1 | grep 'rep 2' | sed -e 's/.*edges \([0-9.e+]*\) sample_ms/edges \1 sample_ms/' -e 's/ seeds.*//')"
done; done 2>&1 | tee gpurun_out/t_mid_sweep.log
