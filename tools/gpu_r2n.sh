# next-row L2 prefetch A/B; bench c2 with NVML clock polling vs the nvidia-smi child
mkdir -p gpurun_out
for r in 1 2; do for v in main nopf; do
  if [ $v = main ]; then lib=""; else lib=$PWD/variants/var_$v.so; fi
  echo "== $v c5 $(IMMX_B200_LIB=$lib timeout 300 python tools/prof_sample.py --config c5 --count 400000 --reps 2 2>&1 | grep 'rep 1' | grep -o '[0-9.]* Gedges/s')"
  echo "== $v c4 $(IMMX_B200_LIB=$lib timeout 300 python tools/prof_sample.py --config c4 --count 1000000 --reps 2 2>&1 | grep 'rep 1' | grep -o '[0-9.]* Gedges/s')"
done; done > gpurun_out/n_ab.log 2>&1
timeout 900 python bench.py --config c2 > gpurun_out/n_bench_c2_nvml.log 2>&1
BENCH_CLOCKS=smi timeout 900 python bench.py --config c2 > gpurun_out/n_bench_c2_smi.log 2>&1
timeout 900 python bench.py --config c1 > gpurun_out/n_bench_c1_nvml.log 2>&1
timeout 600 python -m pytest tests/test_gpu_longrow.py tests/test_gpu_parity.py -x -q > gpurun_out/n_tests.log 2>&1; echo "rc=$?" >> gpurun_out/n_tests.log
