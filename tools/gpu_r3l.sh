mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_longrow.py -x -q -m gpu > gpurun_out/l_test_a.log 2>&1; echo "a rc=$?"; tail -2 gpurun_out/l_test_a.log
for c in c5 c4; do bash tools/ab_run.sh $c main pf nochain pf 2>&1 | tee gpurun_out/l_ab_$c.log | cut -c1-330; done
