# what the clock sampling costs the timed region (c2, 10 steps): off / nvml / smi at 1 s, nvml at 250 ms
mkdir -p gpurun_out
for r in 1 2; do
for m in off nvml smi; do BENCH_CLOCKS=$m timeout 900 python bench.py --config c2 --steps 10 --no-cpu-baseline > gpurun_out/o_c2_$m.$r.log 2>&1; done
BENCH_CLOCKS=nvml BENCH_CLOCK_MS=250 timeout 900 python bench.py --config c2 --steps 10 --no-cpu-baseline > gpurun_out/o_c2_nvml250.$r.log 2>&1
done
