# long-row slab width A/B, tier debug of one c5 run, ncu capture of a c5 / c4 sampler launch
mkdir -p gpurun_out
run() { timeout 600 python tools/run_config.py --config $1 --reps 2 2>&1 | grep "rep 1" | sed 's/ seeds.*//'; }
for c in c5 c4; do
  for L in 2048 4096; do echo "== lr16 L=$L $c"; IMMX_LONG_MIN=$L run $c; done
  for L in 2048 4096; do echo "== lr8 L=$L $c"; IMMX_B200_LIB=$PWD/variants/var_lr8.so IMMX_LONG_MIN=$L run $c; done
  for L in 4096 8192; do echo "== lr32 L=$L $c"; IMMX_B200_LIB=$PWD/variants/var_lr32.so IMMX_LONG_MIN=$L run $c; done
done > gpurun_out/c_ab.log 2>&1
IMMX_DEBUG_TIERS=1 timeout 300 python tools/run_config.py --config c5 --reps 1 > gpurun_out/c_tiers_c5.log 2>&1
IMMX_DEBUG_TIERS=1 timeout 300 python tools/run_config.py --config c4 --reps 1 > gpurun_out/c_tiers_c4.log 2>&1
timeout 300 python tools/prof_sample.py --config c5 --count 50000 --reps 1 > gpurun_out/c_plain_c5.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rrr_block -s 1 -c 1 -o gpurun_out/samp_c5_r2a \
  python tools/prof_sample.py --config c5 --count 50000 --reps 1 > gpurun_out/c_ncu_c5.log 2>&1
timeout 300 python tools/prof_sample.py --config c4 --count 200000 --reps 1 > gpurun_out/c_plain_c4.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rrr_block -s 1 -c 1 -o gpurun_out/samp_c4_r2a \
  python tools/prof_sample.py --config c4 --count 200000 --reps 1 > gpurun_out/c_ncu_c4.log 2>&1
