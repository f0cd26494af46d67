mkdir -p gpurun_out
python tools/mem_probe.py 16 > gpurun_out/g3_mem.log 2>&1
python tools/mem_probe.py 22 >> gpurun_out/g3_mem.log 2>&1
bash tools/ab_run.sh c5 main base main base > gpurun_out/g3_ab_c5.log 2>&1
bash tools/ab_run.sh c4 main base > gpurun_out/g3_ab_c4.log 2>&1
