# final round-2 numbers: bench lines of all five configs (+ the reference arm on c5), launch
# list of the c5 bench command, ncu --set full of the select kernels on c4 (round 10)
mkdir -p gpurun_out
timeout 900 python bench.py --impl reference > gpurun_out/i_bench_ref_c5.log 2>&1
for c in c5 c4 c2 c3 c1; do timeout 1200 python bench.py --config $c > gpurun_out/i_bench_$c.log 2>&1; tail -1 gpurun_out/i_bench_$c.log | cut -c1-400; done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/i_launches_c5_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/i_ncu_bench_c5.log 2>&1
timeout 600 python tools/run_config.py --config c4 --reps 1 > gpurun_out/i_plain_c4.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_huff_find -s 10 -c 1 -o gpurun_out/find_c4_r2s4 \
  python tools/run_config.py --config c4 --reps 1 > gpurun_out/i_ncu_find.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_sig_filter -s 10 -c 1 -o gpurun_out/filter_c4_r2s4 \
  python tools/run_config.py --config c4 --reps 1 > gpurun_out/i_ncu_filter.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_huff_apply -s 10 -c 1 -o gpurun_out/apply_c4_r2s4 \
  python tools/run_config.py --config c4 --reps 1 > gpurun_out/i_ncu_apply.log 2>&1
ls -la gpurun_out/*.ncu-rep
