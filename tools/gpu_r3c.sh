# signature filter: its own tests; launch lists of the c4 / c3 runs (select kernels only)
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_select_filter.py -m gpu -x -q > gpurun_out/c_tests.log 2>&1; echo "rc=$?" >> gpurun_out/c_tests.log
tail -3 gpurun_out/c_tests.log
for c in c4 c3; do
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_huff|k_sig|k_argmax_pick|k_dense' --csv \
  --log-file gpurun_out/c_launches_$c.csv python tools/run_config.py --config $c --reps 1 > gpurun_out/c_ncu_$c.log 2>&1
done
