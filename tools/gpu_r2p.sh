mkdir -p gpurun_out
BENCH_CLOCKS=off timeout 900 python bench.py --config c2 --steps 10 --no-cpu-baseline > gpurun_out/p_c2_off.log 2>&1
timeout 900 python tools/run_config.py --config c2 --reps 8 > gpurun_out/p_c2_run.log 2>&1
