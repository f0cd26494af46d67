# round 2 session 2: first box call -- full GPU suite + smoke, c5 bench (both arms), c5 launch list
set -x
mkdir -p gpurun_out
(nproc; free -g; lscpu | head -25; nvidia-smi --query-gpu=name,memory.total,clocks.max.sm --format=csv) > gpurun_out/host_info.txt 2>&1
timeout 2400 python -m pytest tests -m gpu -x -q --durations=30 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench_c5.log 2>&1; echo rc=$? >> gpurun_out/bench_c5.log
timeout 900 python bench.py --impl reference > gpurun_out/bench_c5_ref.log 2>&1; echo rc=$? >> gpurun_out/bench_c5_ref.log
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/launches_c5.csv \
  python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ncu_c5.log 2>&1; echo rc=$? >> gpurun_out/ncu_c5.log
