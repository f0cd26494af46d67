# IMMX_LONG_MIN sweep on the final kernel
mkdir -p gpurun_out
for c in c4 c5; do
for m in 4096 2048 3072 6144 8192; do
  echo "== $c long_min=$m: $(IMMX_LONG_MIN=$m timeout 600 python tools/run_config.py --config $c --reps 3 2>&1 | grep 'rep 2' | sed -e 's/.*edges \([0-9.e+]*\) sample_ms/edges \1 sample_ms/' -e 's/ seeds.*//')"
done; done 2>&1 | tee gpurun_out/x_long_sweep.log
