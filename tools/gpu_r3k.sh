# chained long rows: long-row / parity / config tests, then A/B against the un-chained build
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_longrow.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -m gpu > gpurun_out/k_test_a.log 2>&1; echo "a rc=$?"; tail -3 gpurun_out/k_test_a.log
timeout 1800 python -m pytest tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/k_test_cfg.log 2>&1; echo "cfg rc=$?"; tail -3 gpurun_out/k_test_cfg.log
for c in c5 c4; do bash tools/ab_run.sh $c main nochain main nochain 2>&1 | tee gpurun_out/k_ab_$c.log | cut -c1-330; done
