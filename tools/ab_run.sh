#!/bin/bash
# A/B of library builds on full IMM runs (dev tooling): phases of the third run of each.
# usage: tools/ab_run.sh <config> main|<name>...   (<name> -> variants/var_<name>.so)
cfg=$1; shift
for v in "$@"; do
  if [ "$v" = main ]; then lib=""; else lib=$PWD/variants/var_$v.so; fi
  echo "== $v"; IMMX_B200_LIB=$lib timeout 600 python tools/run_config.py --config $cfg --reps 3 2>&1 | grep "rep 2" | sed 's/ seeds.*//'
done
