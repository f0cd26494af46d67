#!/bin/bash
# Sampler throughput against the number of resident CTAs (IMMX_SAMPLER_CTAS; dev tooling).
# usage: tools/cta_sweep.sh <config> <samples>
for c in 148 296 444 592 740; do echo "== ctas $c"; IMMX_SAMPLER_CTAS=$c timeout 300 python tools/prof_sample.py --config $1 --count $2 --reps 2 2>&1 | grep "rep 1"; done
