# model-weighted upload tests; bench lines (e2e through the model upload); LT walk capture (c3);
# final sampler captures (c5, c4) for profiles/ncu_sampler_traffic.json
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_upload_model.py -x -q > gpurun_out/t_tests.log 2>&1; echo "rc=$?" >> gpurun_out/t_tests.log
for c in c5 c1 c3; do timeout 900 python bench.py --config $c > gpurun_out/t_bench_$c.log 2>&1; done
timeout 300 python tools/prof_sample.py --config c3 --count 100000 --reps 1 > gpurun_out/t_plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rrr_kernel -s 1 -c 1 -o gpurun_out/lt_c3_r2 \
  python tools/prof_sample.py --config c3 --count 100000 --reps 1 > gpurun_out/t_ncu_c3.log 2>&1
timeout 300 python tools/prof_sample.py --config c5 --count 400000 --reps 1 > gpurun_out/t_plain_c5.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rrr_block -s 1 -c 1 -o gpurun_out/samp_c5_r2c \
  python tools/prof_sample.py --config c5 --count 400000 --reps 1 > gpurun_out/t_ncu_c5.log 2>&1
timeout 300 python tools/prof_sample.py --config c4 --count 1000000 --reps 1 > gpurun_out/t_plain_c4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:rrr_block -s 1 -c 1 -o gpurun_out/samp_c4_r2c \
  python tools/prof_sample.py --config c4 --count 1000000 --reps 1 > gpurun_out/t_ncu_c4.log 2>&1
