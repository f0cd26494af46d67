# split slab barrier (arrive / next filter / wait): tests, then A/B against the plain barrier
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_longrow.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_lookahead.py -x -q -m gpu > gpurun_out/n_test_a.log 2>&1; echo "a rc=$?"; tail -3 gpurun_out/n_test_a.log
for c in c5 c4; do bash tools/ab_run.sh $c main nosplit main nosplit 2>&1 | tee gpurun_out/n_ab_$c.log | cut -c1-60,150-330; done
timeout 1800 python -m pytest tests/test_gpu_configs.py -x -q -m gpu > gpurun_out/n_test_cfg.log 2>&1; echo "cfg rc=$?"; tail -3 gpurun_out/n_test_cfg.log
