# filter bit index from the product's high half (filt2), + max-only coin loop (filt2max)
mkdir -p gpurun_out
for c in c5 c4; do bash tools/ab_run.sh $c main filt2 filt2max main filt2 filt2max 2>&1 | tee gpurun_out/q_ab_$c.log | cut -c1-60,150-330; done
