# long-row path v2: parity (forced-low thresholds + exact coins), timings, one ncu capture
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_longrow.py tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q > gpurun_out/d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/d_tests.log
run() { timeout 600 python tools/run_config.py --config $1 --reps 2 2>&1 | grep "rep 1" | sed 's/ seeds.*//'; }
for c in c5 c4 c2; do echo "== $c"; run $c; done > gpurun_out/d_ab.log 2>&1
timeout 300 python tools/prof_sample.py --config c5 --count 400000 --reps 1 > gpurun_out/d_plain_c5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rrr_block -s 1 -c 1 -o gpurun_out/samp_c5_r2b \
  python tools/prof_sample.py --config c5 --count 400000 --reps 1 > gpurun_out/d_ncu_c5.log 2>&1
