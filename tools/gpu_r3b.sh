# signature filter in select_huffman: parity (store / select / hybrid / config tests), then the
# select phase per config with IMMX_SIG_K = 0 (no filter) / 1 / 2 / 3
mkdir -p gpurun_out
timeout 1800 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hybrid.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_lt.py tests/test_gpu_integration.py tests/test_cli.py -m gpu -x -q > gpurun_out/b_tests.log 2>&1; echo "rc=$?" >> gpurun_out/b_tests.log
tail -3 gpurun_out/b_tests.log
for c in c3 c2 c5 c4; do
for k in 0 1 2 3; do
IMMX_SIG_K=$k timeout 600 python tools/run_config.py --config $c --reps 2 > gpurun_out/b_${c}_k$k.log 2>&1
grep "rep 1" gpurun_out/b_${c}_k$k.log | sed -e 's/.*phases/phases/' -e 's/edges .*//' | sed -e "s/^/$c k=$k /"
done
done
IMMX_DEBUG_SELECT=1 IMMX_SIG_K=2 timeout 600 python tools/run_config.py --config c4 --reps 1 > gpurun_out/b_c4_dbg.log 2>&1
IMMX_DEBUG_SELECT=1 IMMX_SIG_K=2 timeout 600 python tools/run_config.py --config c3 --reps 1 > gpurun_out/b_c3_dbg.log 2>&1
