# filter with one instruction less per test + funnel-shift mask (filt); the same + max-only coin loop (filtmax)
mkdir -p gpurun_out
for c in c5 c4; do bash tools/ab_run.sh $c main filt filtmax main filt filtmax 2>&1 | tee gpurun_out/p_ab_$c.log | cut -c1-60,150-330; done
export IMMX_B200_LIB=$PWD/variants/var_filtmax.so
timeout 1200 python -m pytest tests/test_gpu_longrow.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/p_test_a.log 2>&1; echo "a rc=$?"; tail -3 gpurun_out/p_test_a.log
timeout 1800 python -m pytest tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/p_test_cfg.log 2>&1; echo "cfg rc=$?"; tail -3 gpurun_out/p_test_cfg.log
