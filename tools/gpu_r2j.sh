# selection A/B: windowed lock-step find (main) at 5/6/8 CTAs per SM vs the refill find (oldsel)
mkdir -p gpurun_out
run() { timeout 600 python tools/run_config.py --config $1 --reps 2 2>&1 | grep "rep 1" | grep -o "'select': [0-9.]*"; }
for r in 1 2; do
for c in c4 c3 c2 c5; do
  for x in 5 6 8; do echo "== main ctas=$x $c $(IMMX_FIND_CTAS=$x run $c)"; done
  echo "== oldsel $c $(IMMX_B200_LIB=$PWD/variants/var_oldsel.so run $c)"
done; done > gpurun_out/j_ab.log 2>&1
