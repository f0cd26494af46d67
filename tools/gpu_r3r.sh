# coin-loop unroll sweep on the max-only loop (main = 4), then the GPU suite on main
mkdir -p gpurun_out
bash tools/ab_run.sh c5 main u2 u8 u16 main u8 2>&1 | tee gpurun_out/r_ab_c5.log | cut -c1-60,150-330
bash tools/ab_run.sh c4 main u8 u16 2>&1 | tee gpurun_out/r_ab_c4.log | cut -c1-60,150-330
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/r_test_all.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/r_test_all.log
