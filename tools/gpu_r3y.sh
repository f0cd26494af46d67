# 5 CTAs per SM: first hash tier of 2^12 slots (20 KB) and 48 registers
mkdir -p gpurun_out
for c in c5 c4; do bash tools/ab_run.sh $c main h12b5 h12b4 h13b5 main h12b5 2>&1 | tee gpurun_out/y_ab_$c.log | cut -c1-60,150-330; done
