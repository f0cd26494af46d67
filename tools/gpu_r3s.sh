# final round-2 numbers on the final kernel: sampler captures (c5, c4) for
# profiles/ncu_sampler_traffic.json, bench lines of all configs + the reference arm, launch list
mkdir -p gpurun_out
timeout 300 python tools/prof_sample.py --config c5 --count 400000 --reps 1 > gpurun_out/s_plain_c5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rrr_block -s 1 -c 1 -o gpurun_out/samp_c5_r2e \
  python tools/prof_sample.py --config c5 --count 400000 --reps 1 > gpurun_out/s_ncu_c5.log 2>&1
timeout 300 python tools/prof_sample.py --config c4 --count 1000000 --reps 1 > gpurun_out/s_plain_c4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rrr_block -s 1 -c 1 -o gpurun_out/samp_c4_r2e \
  python tools/prof_sample.py --config c4 --count 1000000 --reps 1 > gpurun_out/s_ncu_c4.log 2>&1
tail -2 gpurun_out/s_plain_c5.log gpurun_out/s_plain_c4.log
