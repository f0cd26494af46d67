# select: CTA-aggregated filter; LUT widths; segment length variants; per-kernel event timing
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_select_filter.py tests/test_gpu_hybrid.py tests/test_gpu_golden.py -m gpu -x -q > gpurun_out/d_tests.log 2>&1; echo "rc=$?" >> gpurun_out/d_tests.log
tail -2 gpurun_out/d_tests.log
run() { # name config env...
  local name=$1 cfg=$2; shift 2
  env "$@" IMMX_DEBUG_PHASES=1 timeout 600 python tools/run_config.py --config $cfg --reps 2 > gpurun_out/d_${cfg}_$name.log 2>&1
  echo "$cfg $name: $(grep 'rep 1' gpurun_out/d_${cfg}_$name.log | sed -e "s/.*'select': \([0-9.]*\).*store \([0-9.]* GB\).*/select \1 s store \2/") | $(grep 'rounds:' gpurun_out/d_${cfg}_$name.log | tail -1 | sed 's/.*rounds: //')"
}
for c in c3 c4 c2 c5; do
run base $c A=1
run r16s8 $c IMMX_LUT_ROOT=16 IMMX_LUT_SUB=8
run r16s12 $c IMMX_LUT_ROOT=16 IMMX_LUT_SUB=12
run r14s10 $c IMMX_LUT_ROOT=14 IMMX_LUT_SUB=10
run seg32 $c IMMX_B200_LIB=$PWD/variants/var_seg32.so
run seg16 $c IMMX_B200_LIB=$PWD/variants/var_seg16.so
run seg16r16s12 $c IMMX_B200_LIB=$PWD/variants/var_seg16.so IMMX_LUT_ROOT=16 IMMX_LUT_SUB=12
done
