# selection: length-sorted lock-step find pass -- parity + timings
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_golden.py tests/test_gpu_hybrid.py tests/test_gpu_configs.py tests/test_gpu_parity.py tests/test_cli.py tests/test_gpu_fullsize.py -x -q > gpurun_out/i_tests.log 2>&1; echo "rc=$?" >> gpurun_out/i_tests.log
run() { timeout 600 python tools/run_config.py --config $1 --reps 2 2>&1 | grep "rep 1" | sed 's/ seeds.*//; s/ratio.*sample_ms/sample_ms/'; }
for c in c4 c3 c5 c2; do echo "== $c"; run $c; done > gpurun_out/i_ab.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/i_launches_c4.csv \
    python tools/run_config.py --config c4 --reps 1 > gpurun_out/i_ncu_c4.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_huff_find -s 10 -c 1 -o gpurun_out/find_c4_r2b \
  python tools/run_config.py --config c4 --reps 1 > gpurun_out/i_ncu_find.log 2>&1
