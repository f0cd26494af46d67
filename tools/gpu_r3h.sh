# device-built decode table: tests, full suite, then c5 / c4 / c2 / c3 runs host vs device table
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_lut.py -m gpu -x -q > gpurun_out/h_lut.log 2>&1; echo "rc=$?" >> gpurun_out/h_lut.log
tail -3 gpurun_out/h_lut.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/h_tests.log 2>&1; echo "rc=$?" >> gpurun_out/h_tests.log
tail -3 gpurun_out/h_tests.log
for c in c5 c4 c2 c3 c1; do
for h in 1 0; do
IMMX_LUT_HOST=$h IMMX_DEBUG_CODEBOOK=1 timeout 600 python tools/run_config.py --config $c --reps 3 > gpurun_out/h_${c}_host$h.log 2>&1
echo "$c lut_host=$h: $(grep 'rep 2' gpurun_out/h_${c}_host$h.log | sed -e 's/ ratio.*edges/ edges/' -e 's/ seeds.*//' -e 's/.*phases//')"
grep "immx codebook" gpurun_out/h_${c}_host$h.log | tail -2
done
done
