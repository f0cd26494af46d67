# c2 sampler regression hunt: current vs session-start sampler vs no long path in the bitmap tiers
mkdir -p gpurun_out
for r in 1 2; do for v in main r1samp nolongbm; do
  if [ $v = main ]; then lib=""; else lib=$PWD/variants/var_$v.so; fi
  echo "== $v c2"; IMMX_B200_LIB=$lib timeout 300 python tools/prof_sample.py --config c2 --count 60000 --reps 2 2>&1 | grep "rep 1"
  echo "== $v c2 run"; IMMX_B200_LIB=$lib timeout 300 python tools/run_config.py --config c2 --reps 2 2>&1 | grep "rep 1" | grep -o "wall [0-9.]*s\|sample_ms.*"
  echo "== $v c1 run"; IMMX_B200_LIB=$lib timeout 300 python tools/run_config.py --config c1 --reps 3 2>&1 | grep "rep 2" | grep -o "wall [0-9.]*s\|sample_ms.*"
done; done > gpurun_out/l_ab.log 2>&1
