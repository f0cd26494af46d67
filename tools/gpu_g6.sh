mkdir -p gpurun_out
for c in c5 c4 c2; do
for r in 1 2; do
  echo "== base $c"; IMMX_B200_LIB=$PWD/variants/var_base.so timeout 600 python tools/run_config.py --config $c --reps 2 2>&1 | grep "rep 1" | sed 's/ seeds.*//; s/phases.*ratio/ratio/'
  for L in 0 2048 16384; do
    echo "== L=$L $c"; IMMX_LONG_MIN=$L timeout 600 python tools/run_config.py --config $c --reps 2 2>&1 | grep "rep 1" | sed 's/ seeds.*//; s/phases.*ratio/ratio/'
  done
done; done > gpurun_out/g6_ab.log 2>&1
