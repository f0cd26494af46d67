# selection: decode table persisting in L2 + evict-first stream loads, A/B
mkdir -p gpurun_out
run() { timeout 600 python tools/run_config.py --config $1 --reps 2 2>&1 | grep "rep 1" | sed 's/ seeds.*//; s/ratio.*sample_ms/sample_ms/'; }
for r in 1 2; do
for c in c4 c3 c5; do
  echo "== main $c"; run $c
  echo "== nopersist $c"; IMMX_NO_L2_PERSIST=1 run $c
  echo "== ldg $c"; IMMX_B200_LIB=$PWD/variants/var_ldg.so run $c
  echo "== ldg+nopersist $c"; IMMX_NO_L2_PERSIST=1 IMMX_B200_LIB=$PWD/variants/var_ldg.so run $c
done; done > gpurun_out/h_ab.log 2>&1
IMMX_DEBUG_CODEBOOK=1 timeout 300 python tools/run_config.py --config c4 --reps 1 2>&1 | grep codebook > gpurun_out/h_cb.log
IMMX_DEBUG_CODEBOOK=1 timeout 300 python tools/run_config.py --config c3 --reps 1 2>&1 | grep codebook >> gpurun_out/h_cb.log
IMMX_DEBUG_CODEBOOK=1 timeout 300 python tools/run_config.py --config c5 --reps 1 2>&1 | grep codebook >> gpurun_out/h_cb.log
timeout 900 python -m pytest tests/test_gpu_golden.py tests/test_gpu_hybrid.py tests/test_gpu_configs.py -x -q > gpurun_out/h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/h_tests.log
