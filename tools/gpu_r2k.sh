# round-2 bench lines (all configs, both arms for c5) + the c5 launch list of the bench command
mkdir -p gpurun_out
(nproc; lscpu | grep -E "Model name|Socket|Core|Thread"; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > gpurun_out/k_host.txt 2>&1
timeout 900 python bench.py > gpurun_out/k_bench_c5.log 2>&1; echo rc=$? >> gpurun_out/k_bench_c5.log
timeout 900 python bench.py --impl reference > gpurun_out/k_bench_c5_ref.log 2>&1; echo rc=$? >> gpurun_out/k_bench_c5_ref.log
for c in c4 c2 c3 c1; do timeout 900 python bench.py --config $c > gpurun_out/k_bench_$c.log 2>&1; echo rc=$? >> gpurun_out/k_bench_$c.log; done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 5000 --csv --log-file gpurun_out/k_launches_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/k_ncu_c5.log 2>&1; echo rc=$? >> gpurun_out/k_ncu_c5.log
