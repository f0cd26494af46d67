set -x
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -25; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > gpurun_out/host_info.txt 2>&1
timeout 900 python bench.py --config c5 --steps 5 --warmup 3 > gpurun_out/g1_c5.log 2>&1; echo rc=$? >> gpurun_out/g1_c5.log
timeout 900 python bench.py --impl reference --config c5 --steps 3 --warmup 3 > gpurun_out/g1_c5_ref.log 2>&1; echo rc=$? >> gpurun_out/g1_c5_ref.log
