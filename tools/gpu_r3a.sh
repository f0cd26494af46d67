# re-entry check: full GPU suite + smoke, then the driver's two bench commands on the default config
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/a_bench_ref.log 2>&1
timeout 900 python bench.py > gpurun_out/a_bench.log 2>&1
tail -3 gpurun_out/gpu_tests.log; tail -2 gpurun_out/smoke.log; tail -1 gpurun_out/a_bench_ref.log; tail -1 gpurun_out/a_bench.log
