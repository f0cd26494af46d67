mkdir -p gpurun_out
IMMX_DEBUG_PHASES=1 timeout 900 python tools/run_config.py --config c2 --reps 8 > gpurun_out/r_c2.log 2>&1
IMMX_DEBUG_PHASES=1 IMMX_SYNC_ALLOC=1 timeout 900 python tools/run_config.py --config c2 --reps 8 > gpurun_out/r_c2_sync.log 2>&1
