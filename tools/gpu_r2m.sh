# full GPU suite + smoke after the sampler / selection changes; c2 bench line
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -x -q --durations=15 > gpurun_out/m_tests.log 2>&1; echo "rc=$?" >> gpurun_out/m_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/m_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/m_smoke.log
timeout 900 python bench.py --config c2 > gpurun_out/m_bench_c2.log 2>&1; echo rc=$? >> gpurun_out/m_bench_c2.log
