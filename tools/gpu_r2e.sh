# A/B: coin shift on the FMA pipe (main) vs all-ALU (nofma) vs 3 CTAs/SM at 80 registers (minb3)
mkdir -p gpurun_out
for r in 1 2; do
for v in main nofma minb3; do
  if [ $v = main ]; then lib=""; else lib=$PWD/variants/var_$v.so; fi
  echo "== $v c5"; IMMX_B200_LIB=$lib timeout 300 python tools/prof_sample.py --config c5 --count 400000 --reps 2 2>&1 | grep "rep 1"
  echo "== $v c4"; IMMX_B200_LIB=$lib timeout 300 python tools/prof_sample.py --config c4 --count 1000000 --reps 2 2>&1 | grep "rep 1"
done; done > gpurun_out/e_ab.log 2>&1
timeout 600 python -m pytest tests/test_gpu_longrow.py tests/test_gpu_parity.py -x -q > gpurun_out/e_tests.log 2>&1; echo "rc=$?" >> gpurun_out/e_tests.log
