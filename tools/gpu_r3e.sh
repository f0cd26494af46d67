# LUT sizes per width choice (c4, c5, c3); c2 per-round launch list
mkdir -p gpurun_out
for c in c4 c5 c3; do
for w in "12 8" "16 8" "16 12" "14 10"; do
set -- $w
IMMX_DEBUG_CODEBOOK=1 IMMX_LUT_ROOT=$1 IMMX_LUT_SUB=$2 timeout 600 python tools/run_config.py --config $c --reps 1 2>&1 | grep -E "decode table|lut" | sed "s/^/$c $1-$2: /"
done
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_huff|k_sig|k_argmax_pick|k_dense' --csv \
  --log-file gpurun_out/e_launches_c2.csv python tools/run_config.py --config c2 --reps 1 > gpurun_out/e_ncu_c2.log 2>&1
