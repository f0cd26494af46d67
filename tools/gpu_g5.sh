mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_integration.py -x -q > gpurun_out/g5_integ.log 2>&1; echo "rc=$?" >> gpurun_out/g5_integ.log
for r in 1 2; do for L in 0 2048; do
  echo "== L=$L"; IMMX_LONG_MIN=$L timeout 300 python tools/prof_sample.py --config c5 --count 20000 --reps 2 2>&1 | grep "rep 1"
done; done > gpurun_out/g5_ab.log 2>&1
IMMX_LONG_MIN=2048 timeout 300 python tools/prof_sample.py --config c5 --count 20000 --reps 1 > gpurun_out/g5_plain.log 2>&1 && \
IMMX_LONG_MIN=2048 ncu --set full --clock-control none --import-source on -k regex:rrr_block -c 5 -o gpurun_out/g5_long python tools/prof_sample.py --config c5 --count 20000 --reps 1 > gpurun_out/g5_ncu.log 2>&1
