# final round-2 lines on the final kernel: GPU suite, reference arm, bench of all configs, launch list
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -x -q -m gpu > gpurun_out/u_test_all.log 2>&1; echo "all rc=$?"; tail -3 gpurun_out/u_test_all.log
timeout 900 python bench.py --impl reference > gpurun_out/u_bench_ref_c5.log 2>&1
for c in c5 c4 c2 c3 c1; do timeout 1200 python bench.py --config $c > gpurun_out/u_bench_$c.log 2>&1; tail -n 1 gpurun_out/u_bench_$c.log | cut -c1-330; done
timeout 1500 ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/u_launches_c5_bench.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/u_ncu_bench_c5.log 2>&1
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -n 2
