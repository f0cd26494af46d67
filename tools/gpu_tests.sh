# full GPU test suite + smoke on the box; logs under gpurun_out/
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "rc=$?" >> gpurun_out/smoke.log
