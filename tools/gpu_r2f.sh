# launch lists (one IMM run per config) + an ncu capture of the LT walk (c3)
mkdir -p gpurun_out
for c in c4 c3 c5 c2; do
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 20000 --csv --log-file gpurun_out/f_launches_$c.csv \
    python tools/run_config.py --config $c --reps 1 > gpurun_out/f_ncu_$c.log 2>&1
done
timeout 300 python tools/prof_sample.py --config c3 --count 100000 --reps 1 > gpurun_out/f_plain_c3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:rrr_kernel -s 1 -c 1 -o gpurun_out/lt_c3_r2 \
  python tools/prof_sample.py --config c3 --count 100000 --reps 1 > gpurun_out/f_ncu_c3.log 2>&1
