# chained long rows in every tier (hash tiers with the capacity guard): A/B, then tests on the variant
mkdir -p gpurun_out
for c in c5 c4; do bash tools/ab_run.sh $c main chain main chain 2>&1 | tee gpurun_out/v_ab_$c.log | cut -c1-60,150-330; done
export IMMX_B200_LIB=$PWD/variants/var_chain.so
timeout 1500 python -m pytest tests/test_gpu_longrow.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_lookahead.py -x -q -m gpu > gpurun_out/v_test_a.log 2>&1; echo "a rc=$?"; tail -n 3 gpurun_out/v_test_a.log
timeout 1800 python -m pytest tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/v_test_cfg.log 2>&1; echo "cfg rc=$?"; tail -n 3 gpurun_out/v_test_cfg.log
