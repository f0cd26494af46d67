mkdir -p gpurun_out
/usr/bin/time -f "wall %e s" python -c "import paper_2208_00613_b200 as im; im.default_device()" > gpurun_out/s_init.log 2>&1
IMMX_DEBUG_PHASES=1 timeout 900 python tools/run_config.py --config c2 --reps 8 > gpurun_out/s_c2.log 2>&1
IMMX_DEBUG_PHASES=1 timeout 900 python tools/run_config.py --config c4 --reps 4 > gpurun_out/s_c4.log 2>&1
IMMX_DEBUG_PHASES=1 timeout 900 python tools/run_config.py --config c5 --reps 4 > gpurun_out/s_c5.log 2>&1
timeout 900 python bench.py --config c2 > gpurun_out/s_bench_c2.log 2>&1
