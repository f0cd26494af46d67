# c5 sampler capture (un-chained build = the round-2 kernel), source-level stalls
mkdir -p gpurun_out
export IMMX_B200_LIB=$PWD/variants/var_nochain.so
timeout 600 python tools/prof_sample.py --config c5 --count 400000 --reps 1 > gpurun_out/m_plain_c5.log 2>&1; tail -2 gpurun_out/m_plain_c5.log
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:rrr_block -s 1 -c 1 -o gpurun_out/samp_c5_r2d \
  python tools/prof_sample.py --config c5 --count 400000 --reps 1 > gpurun_out/m_ncu_c5.log 2>&1; tail -2 gpurun_out/m_ncu_c5.log
ls -la gpurun_out/samp_c5_r2d.ncu-rep
