mkdir -p gpurun_out
IMMX_DEBUG_TIERS=1 timeout 900 python tools/run_config.py --config c2 --reps 8 > gpurun_out/q_c2_run.log 2>&1
