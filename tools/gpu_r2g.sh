mkdir -p gpurun_out
IMMX_DEBUG_SELECT=1 timeout 300 python tools/run_config.py --config c4 --reps 1 > gpurun_out/g_sel_c4.log 2>&1
IMMX_DEBUG_SELECT=1 timeout 300 python tools/run_config.py --config c3 --reps 1 > gpurun_out/g_sel_c3.log 2>&1
timeout 300 python tools/prof_sample.py --config c3 --count 100000 --reps 1 > gpurun_out/g_plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rrr_kernel -s 1 -c 1 -o gpurun_out/lt_c3_r2 \
  python tools/prof_sample.py --config c3 --count 100000 --reps 1 > gpurun_out/g_ncu_c3.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_huff_find -s 10 -c 1 -o gpurun_out/find_c4_r2 \
  python tools/run_config.py --config c4 --reps 1 > gpurun_out/g_ncu_find.log 2>&1
